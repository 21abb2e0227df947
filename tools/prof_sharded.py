import os, sys, time, cProfile, pstats
sys.path.insert(0, ".")
import torch, torch.distributed as dist
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", RANK="0", WORLD_SIZE="1")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import paper_1011_3534_b200 as sp
from paper_1011_3534_b200 import distributed as spd, workloads
at, _, leaf, taus = workloads.make_config_device("c5", "cuda:0")
n = at.shape[0]
A = spd.ShardedTree.scatter(at, n, leaf, spd.Comm())
del at; torch.cuda.empty_cache()
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    C, st, det = spd.spamm_sharded(A, A, sp.SpammConfig(tau=taus[0]))
    torch.cuda.synchronize(); print("spamm_sharded", (time.perf_counter()-t0)*1e3, "ms", flush=True)
    del C
pr = cProfile.Profile(); pr.enable()
C, st, det = spd.spamm_sharded(A, A, sp.SpammConfig(tau=taus[0]))
torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
