import sys; sys.path.insert(0,'.')
import torch, paper_1011_3534_b200 as sp
from paper_1011_3534_b200 import distributed as spd, workloads
at,_,leaf,taus = workloads.make_config_device("c5","cuda:0")
n = at.shape[0]
a = sp.from_device_pointer(at.data_ptr(), n, leaf_size=leaf); del at; torch.cuda.empty_cache()
for W in (1, 2):
    for r in range(W):
        rows = spd.row_shard(r, W, n, leaf)
        for rep in range(2):
            try:
                c, st, det = sp.spamm_detailed(a, a, sp.SpammConfig(tau=taus[0]), rows=rows)
                print(W, r, rep, "ok", det.ms_total, flush=True)
                del c
            except Exception as e:
                print(W, r, rep, "ERR", e, flush=True)
