"""Bytes each rank moves for one c5 multiply (n = 65536, leaf 64, tau = 1e-8)
in the distributed layout (paper_1011_3534_b200.distributed), from the
retained triples of the full-size product on one GPU: scatter of its rows
from one source, all-gather of the leaf level (pyramids), the halo of B
blocks its band's retained triples read from other ranks, and C's leaf-level
all-gather.  Prints one JSON line per world size."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1011_3534_b200 as sp  # noqa: E402
from paper_1011_3534_b200 import distributed as spd  # noqa: E402
from paper_1011_3534_b200 import workloads  # noqa: E402


def main():
    import torch

    at, _, leaf, taus = workloads.make_config_device("c5", "cuda:0")
    n = at.shape[0]
    a = sp.from_device_pointer(at.data_ptr(), n, leaf_size=leaf)
    del at
    torch.cuda.empty_cache()
    _, st, det = sp.spamm_detailed(a, a, sp.SpammConfig(tau=taus[0]), keep_triples=True,
                                   traverse_only=True)
    tr = det.triples.astype(np.int64)
    nb = a.block_grid
    blk = leaf * leaf * 8
    for world in (2, 4, 8):
        bands = [spd.row_shard(r, world, n, leaf) for r in range(world)]
        owner = np.zeros(nb, np.int64)
        for r, (lo, hi) in enumerate(bands):
            owner[lo:hi] = r
        per = []
        for r, (lo, hi) in enumerate(bands):
            mine = tr[(tr[:, 0] >= lo) & (tr[:, 0] < hi)]
            need = np.unique(mine[:, 2] * nb + mine[:, 1])
            halo = int((owner[need // nb] != r).sum())
            per.append(dict(rank=r, rows=hi - lo, retained=int(len(mine)),
                            scatter_bytes=int((hi - lo) * leaf * n * 8),
                            leaf_level_allgather_bytes=int(9 * nb * nb),
                            halo_blocks=halo, halo_bytes=halo * blk))
        print(json.dumps(dict(config="c5 n=65536 leaf=64 tau=1e-8", world=world,
                              retained_total=int(len(tr)), max_halo_bytes=max(p["halo_bytes"] for p in per),
                              per_rank=per)), flush=True)


if __name__ == "__main__":
    main()
