"""MatrixMarket exchange for quadtree matrices (the reference's matrixmarket.py:1-103).

Same files byte for byte: ``matrix array real general`` (dense, column-major)
or ``matrix coordinate real general`` (1-based triples in column-major order),
values printed with 17 significant digits so float64 survives a round trip.
Reading accepts array or coordinate, real or integer, general or symmetric,
with the reference's validation and error messages.  Host text I/O only:
trees go through ``to_dense`` / ``from_dense`` (the GPU path) on either side.
"""

from __future__ import annotations

import numpy as np

_BANNER = "%%MatrixMarket"


def _as_dense(mat):
    dense = mat.to_dense() if hasattr(mat, "to_dense") else np.asarray(mat)
    if dense.ndim != 2:
        raise ValueError(f"expected a 2-D matrix, got shape {dense.shape}")
    return dense


def write_matrix_market(mat, path, fmt="array"):
    """Write ``mat`` (an ndarray or anything with to_dense()) as a MatrixMarket
    file (matrixmarket.py:12-36)."""
    dense = _as_dense(mat)
    rows, cols = dense.shape
    if fmt not in ("array", "coordinate"):
        raise ValueError(f"fmt must be 'array' or 'coordinate', got {fmt!r}")
    with open(path, "w") as fh:
        fh.write(f"{_BANNER} matrix {fmt} real general\n")
        if fmt == "array":
            fh.write(f"{rows} {cols}\n")
            if dense.size:
                np.savetxt(fh, dense.T.reshape(-1, 1), fmt="%.17g")
        else:
            col, row = np.nonzero(dense.T)          # column-major order
            fh.write(f"{rows} {cols} {col.size}\n")
            if col.size:
                table = np.empty((col.size, 3), dtype=object)
                table[:, 0] = row + 1
                table[:, 1] = col + 1
                table[:, 2] = dense[row, col]
                np.savetxt(fh, table, fmt=("%d", "%d", "%.17g"))


def _payload(fh):
    for line in fh:
        if line.strip() and not line.lstrip().startswith("%"):
            yield line


def read_matrix_market(path):
    """Read a real MatrixMarket file into a dense float64 array
    (matrixmarket.py:39-103)."""
    with open(path) as fh:
        header = fh.readline()
        if not header.startswith(_BANNER):
            raise ValueError(f"not a MatrixMarket file: {path}")
        words = header.split()
        if len(words) != 5:
            raise ValueError(f"malformed MatrixMarket header: {header.strip()!r}")
        obj, fmt, field, symmetry = (w.lower() for w in words[1:])
        for name, value, allowed in (("object", obj, ("matrix",)),
                                     ("format", fmt, ("array", "coordinate")),
                                     ("field", field, ("real", "integer")),
                                     ("symmetry", symmetry, ("general", "symmetric"))):
            if value not in allowed:
                raise ValueError(f"unsupported MatrixMarket {name} {value!r}")
        lines = _payload(fh)
        size = next(lines, None)
        if size is None:
            raise ValueError(f"missing size line in {path}")
        if fmt == "array":
            rows, cols = (int(t) for t in size.split())
            vals = np.array([float(t) for line in lines for t in line.split()], dtype=np.float64)
            if symmetry == "symmetric":
                # lower triangle column by column, diagonal included
                want = rows * (rows + 1) // 2
                if vals.size != want:
                    raise ValueError(f"expected {want} values, found {vals.size}")
                out = np.zeros((rows, cols))
                jj, ii = np.triu_indices(rows)      # (j <= i) pairs in column-major order
                out[ii, jj] = vals
                out[jj, ii] = vals
                return out
            if vals.size != rows * cols:
                raise ValueError(f"expected {rows * cols} values, found {vals.size}")
            return vals.reshape(cols, rows).T
        rows, cols, nnz = (int(t) for t in size.split())
        out = np.zeros((rows, cols))
        seen = 0
        for line in lines:
            i_s, j_s, v_s = line.split()
            i, j, v = int(i_s) - 1, int(j_s) - 1, float(v_s)
            out[i, j] += v
            if symmetry == "symmetric" and i != j:
                out[j, i] += v
            seen += 1
        if seen != nnz:
            raise ValueError(f"expected {nnz} entries, found {seen}")
        return out


__all__ = ["read_matrix_market", "write_matrix_market"]
