"""Install this package under the reference's import name ``spamm``.

Code written against the reference package (``import spamm``,
``from spamm.multiply import spamm, SpammConfig``, ``from spamm.quadtree
import from_dense``, ...) runs unchanged on the B200 after::

    from paper_1011_3534_b200 import compat
    compat.install()

``install`` aliases the top-level package and the submodules the reference
exposes (``spamm/__init__.py:12-98``): ``quadtree``, ``multiply``,
``generators``, ``purification``, ``ordering``, ``matrixmarket``.  The CLI
(``spamm.cli``) is outside this build's scope and is not
aliased.  ``uninstall`` restores whatever was registered before.
"""

from __future__ import annotations

import importlib
import sys

SUBMODULES = ("quadtree", "multiply", "generators", "purification", "ordering", "matrixmarket")

_saved = None


def install(name="spamm"):
    """Register this package as ``name`` (and ``name.<submodule>``) in
    ``sys.modules``; returns the aliased top-level module."""
    global _saved
    pkg = importlib.import_module(__package__)
    keys = [name] + [f"{name}.{m}" for m in SUBMODULES]
    if _saved is None:
        _saved = {k: sys.modules.get(k) for k in keys}
    sys.modules[name] = pkg
    for m in SUBMODULES:
        mod = importlib.import_module(f"{__package__}.{m}")
        sys.modules[f"{name}.{m}"] = mod
        setattr(pkg, m, mod)
    return pkg


def uninstall():
    """Undo :func:`install`."""
    global _saved
    if _saved is None:
        return
    for k, v in _saved.items():
        if v is None:
            sys.modules.pop(k, None)
        else:
            sys.modules[k] = v
    _saved = None
