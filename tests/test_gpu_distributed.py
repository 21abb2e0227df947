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


def _check_multiply(spd, sp, comm, a_full, b_full, leaf, tau, out, tag):
    import torch

    n = a_full.shape[0]
    at = torch.from_numpy(a_full).cuda() if comm.rank == 0 else None
    bt = torch.from_numpy(b_full).cuda() if comm.rank == 0 else None
    A = spd.ShardedTree.scatter(at, n, leaf, comm)
    B = A if b_full is a_full else spd.ShardedTree.scatter(bt, n, leaf, comm)
    cfg = sp.SpammConfig(tau=tau, collect_boxes=True)
    C, st, det = spd.spamm_sharded(A, B, cfg)
    # the single-GPU product on the same inputs (every rank computes it)
    a1 = sp.from_dense(a_full, leaf_size=leaf)
    b1 = a1 if b_full is a_full else sp.from_dense(b_full, leaf_size=leaf)
    c1, st1 = sp.spamm(a1, b1, cfg)
    got = C.gather_padded().cpu().numpy()
    ok = dict(
        c=np.array_equal(got.view(np.uint64 if got.dtype == np.float64 else np.uint32),
                         c1._padded.view(np.uint64 if got.dtype == np.float64 else np.uint32)),
        pyramid=np.array_equal(C.tree._pyramid()[2].view(np.uint64), c1._pyramid()[2].view(np.uint64))
        and np.array_equal(C.tree._pyramid()[3], c1._pyramid()[3]),
        a_pyramid=np.array_equal(A.tree._pyramid()[2].view(np.uint64), a1._pyramid()[2].view(np.uint64)),
        stats=all(getattr(st, k) == getattr(st1, k) for k in
                  ("leaf_matmuls", "pruned_calls", "pruned_volume", "empty_skip_volume",
                   "max_depth_reached")),
        budget=st.omitted_budget == st1.omitted_budget,
        boxes=st.boxes == st1.boxes,
        norm=C.norm() == c1.norm(),
        halo=det.halo_bytes if det is not None else 0,
    )
    out[tag] = ok


def _check_purify(spd, sp, comm, L, tau, sweeps, out):
    import torch

    from paper_1011_3534_b200 import purification as P
    from paper_1011_3534_b200 import workloads

    h = workloads.cubic_lattice_hamiltonian(L)
    n = h.shape[0]
    F = spd.ShardedTree.scatter(torch.from_numpy(h).cuda() if comm.rank == 0 else None, n, 64, comm)
    res = spd.purify_sharded(F, n // 2, P.SpammMode(tau), max_iter=sweeps, reference_energy=0.0)
    ref = P.purify(sp.from_dense(h, leaf_size=64), n // 2, P.SpammMode(tau), max_iter=sweeps,
                   reference_energy=0.0)
    got = res.density.gather_padded().cpu().numpy()
    out["purify"] = dict(
        density=np.array_equal(got.view(np.uint64), ref.density._padded.view(np.uint64)),
        traces=res.trace_history == ref.trace_history,
        counts=res.step_leaf_matmuls == ref.step_leaf_matmuls,
        energy=res.energy == ref.energy,
    )


def _worker(rank, world, port, out_dir, backend):
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
        out = {}
        a, b, leaf, taus = workloads.make_config("c1")             # A != B, leaf 32
        _check_multiply(spd, sp, comm, a, b, leaf, taus[0], out, "c1")
        a, _, leaf, taus = workloads.make_config("c2")             # B = A, leaf 64
        _check_multiply(spd, sp, comm, a, a, leaf, taus[2], out, "c2")
        _check_purify(spd, sp, comm, 16, 1e-7, 12, out)            # 16^3 lattice, n = 4096
        with open(os.path.join(out_dir, f"r{rank}.pkl"), "wb") as fh:
            pickle.dump(out, fh)
    finally:
        dist.destroy_process_group()


def _run(world, backend, tmp_path):
    import pickle

    import torch.multiprocessing as mp

    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path), backend), nprocs=world,
                       start_method="spawn")
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
        assert all(out["purify"].values()), (r, out["purify"])


def test_distributed_world1_nccl(tmp_path):
    _run(1, "nccl", tmp_path)


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_multirank_gloo(tmp_path, world):
    _run(world, "gloo", tmp_path)
