"""The distributed layout end to end on the GPU (paper_1011_3534_b200.
distributed): row-band ShardedTrees with gathered pyramids, the halo
exchange of operand blocks, spamm_sharded and purify_sharded -- against the
single-GPU library, bit for bit.

* world size 1 over NCCL (the production backend; one GPU here);
* world sizes 2 and 3 over gloo, every rank a separate process on cuda:0 --
  the ranks' kernels never wait on one another (the collectives are host
  side), so this is the multi-rank data flow, not a stand-in for NVLink
  timing.  (purification.py:105-227 for the driver.)"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _reference(tmp_path):
    """The single-GPU results the ranks are compared with, computed once here
    (not in every rank process) and handed to the workers through a file."""
    import pickle

    import paper_1011_3534_b200 as sp
    from paper_1011_3534_b200 import purification as P
    from paper_1011_3534_b200 import workloads

    ref = {}
    for tag, name, tau_i in (("c1", "c1", 0), ("c2", "c2", 2)):
        a, b, leaf, taus = workloads.make_config(name)
        a1 = sp.from_dense(a, leaf_size=leaf)
        b1 = a1 if name == "c2" else sp.from_dense(b, leaf_size=leaf)
        cfg = sp.SpammConfig(tau=taus[tau_i], collect_boxes=True)
        c1, st1 = sp.spamm(a1, b1, cfg)
        ref[tag] = dict(c=c1._padded.copy(), pyr=c1._pyramid()[2].copy(), occ=c1._pyramid()[3].copy(),
                        a_pyr=a1._pyramid()[2].copy(), norm=c1.norm(),
                        stats={k: getattr(st1, k) for k in
                               ("leaf_matmuls", "pruned_calls", "pruned_volume", "empty_skip_volume",
                                "max_depth_reached", "omitted_budget")},
                        boxes=st1.boxes)
    h = workloads.cubic_lattice_hamiltonian(16)
    r = P.purify(sp.from_dense(h, leaf_size=64), h.shape[0] // 2, P.SpammMode(1e-7), max_iter=12,
                 reference_energy=0.0)
    ref["purify"] = dict(density=r.density._padded.copy(), traces=r.trace_history,
                         counts=r.step_leaf_matmuls, energy=r.energy)
    path = tmp_path / "ref.pkl"
    with open(path, "wb") as fh:
        pickle.dump(ref, fh)
    return str(path)


def _check_multiply(spd, sp, comm, a_full, b_full, leaf, tau, ref, out, tag):
    import torch

    n = a_full.shape[0]
    at = torch.from_numpy(a_full).cuda() if comm.rank == 0 else None
    bt = torch.from_numpy(b_full).cuda() if comm.rank == 0 else None
    A = spd.ShardedTree.scatter(at, n, leaf, comm)
    B = A if b_full is a_full else spd.ShardedTree.scatter(bt, n, leaf, comm)
    cfg = sp.SpammConfig(tau=tau, collect_boxes=True)
    C, st, det = spd.spamm_sharded(A, B, cfg)
    got = C.gather_padded().cpu().numpy()
    u = np.uint64 if got.dtype == np.float64 else np.uint32
    ok = dict(
        c=np.array_equal(got.view(u), ref["c"].view(u)),
        pyramid=np.array_equal(C.tree._pyramid()[2].view(np.uint64), ref["pyr"].view(np.uint64))
        and np.array_equal(C.tree._pyramid()[3], ref["occ"]),
        a_pyramid=np.array_equal(A.tree._pyramid()[2].view(np.uint64), ref["a_pyr"].view(np.uint64)),
        stats=all(getattr(st, k) == ref["stats"][k] for k in
                  ("leaf_matmuls", "pruned_calls", "pruned_volume", "empty_skip_volume",
                   "max_depth_reached")),
        budget=st.omitted_budget == ref["stats"]["omitted_budget"],
        boxes=st.boxes == ref["boxes"],
        norm=C.norm() == ref["norm"],
        halo=det.halo_bytes if det is not None else 0,
    )
    out[tag] = ok


def _check_purify(spd, sp, comm, L, tau, sweeps, ref, out):
    import torch

    from paper_1011_3534_b200 import purification as P
    from paper_1011_3534_b200 import workloads

    h = workloads.cubic_lattice_hamiltonian(L)
    n = h.shape[0]
    F = spd.ShardedTree.scatter(torch.from_numpy(h).cuda() if comm.rank == 0 else None, n, 64, comm)
    res = spd.purify_sharded(F, n // 2, P.SpammMode(tau), max_iter=sweeps, reference_energy=0.0)
    got = res.density.gather_padded().cpu().numpy()
    out["purify"] = dict(
        density=np.array_equal(got.view(np.uint64), ref["density"].view(np.uint64)),
        traces=res.trace_history == ref["traces"],
        counts=res.step_leaf_matmuls == ref["counts"],
        energy=res.energy == ref["energy"],
    )
    # diagnostics (not asserted): first sweep whose trace differs
    diff = [q for q, (u, v) in enumerate(zip(res.trace_history, ref["traces"])) if u != v]
    out["purify_diag"] = dict(first_trace_diff=diff[:1])


def _worker(rank, world, port, out_dir, backend, ref_path):
    import pickle

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    kw = dict(device_id=torch.device("cuda", 0)) if backend == "nccl" else {}
    dist.init_process_group(backend, rank=rank, world_size=world, **kw)
    try:
        import paper_1011_3534_b200 as sp
        from paper_1011_3534_b200 import distributed as spd
        from paper_1011_3534_b200 import workloads

        sp.set_device(0)
        comm = spd.Comm()
        with open(ref_path, "rb") as fh:
            ref = pickle.load(fh)
        out = {}
        a, b, leaf, taus = workloads.make_config("c1")             # A != B, leaf 32
        _check_multiply(spd, sp, comm, a, b, leaf, taus[0], ref["c1"], out, "c1")
        a, _, leaf, taus = workloads.make_config("c2")             # B = A, leaf 64
        _check_multiply(spd, sp, comm, a, a, leaf, taus[2], ref["c2"], out, "c2")
        _check_purify(spd, sp, comm, 16, 1e-7, 12, ref["purify"], out)  # 16^3 lattice, n = 4096
        with open(os.path.join(out_dir, f"r{rank}.pkl"), "wb") as fh:
            pickle.dump(out, fh)
    finally:
        dist.destroy_process_group()


def _run(world, backend, tmp_path):
    import pickle

    import torch.multiprocessing as mp

    ref_path = _reference(tmp_path)
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path), backend, ref_path),
                       nprocs=world, start_method="spawn")
    outs = []
    for r in range(world):
        with open(tmp_path / f"r{r}.pkl", "rb") as fh:
            outs.append(pickle.load(fh))
    for r, out in enumerate(outs):
        for tag in ("c1", "c2"):
            o = dict(out[tag])
            halo = o.pop("halo")
            assert all(o.values()), (r, tag, o)
            if world > 1:
                assert halo > 0, (r, tag, "no operand blocks were fetched")
        assert all(out["purify"].values()), (r, out["purify"], out.get("purify_diag"))


def test_distributed_world1_nccl(tmp_path):
    _run(1, "nccl", tmp_path)


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_multirank_gloo(tmp_path, world):
    _run(world, "gloo", tmp_path)
