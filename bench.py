#!/usr/bin/env python
"""bench.py -- SpAMM on B200: retained-leaf FP64 TFLOP/s on BASELINE config 2.

Metric (BASELINE.json): "SpAMM time & retained-leaf FP64 TFLOP/s vs tau".
Workload (BASELINE.json configs[1]): n = 4096, leaf 64,
A = B = sym(u0 * 0.95^|i-j|) (seeded synthetic, numpy PCG64 seed 0), tau
swept over {1e-4, 1e-6, 1e-8, 1e-10}.  One step = one spamm() per tau on
device-resident trees (cull + leaf products + C's tree), i.e. the sweep.

* value      retained-leaf FLOP (2 b^3 per retained triple) / device time,
             TFLOP/s; each spamm timed with CUDA events on the library's own
             stream; L2 flushed (256 MiB write) before every multiply.
* e2e        the same metric through the public API with host buffers:
             from_dense(pinned A) -> spamm per tau -> each product's nonzero
             blocks + pyramid to pinned host memory (the block copy on a
             copy-out stream, overlapping the next call; the next step's A
             copied on a copy-in stream during this step's multiplies),
             host->device and device->host copies inside the timed region.
* roofline   the leaf-product kernel (K3) against the measured FP64 DMMA peak
             (profiles/fp64_peaks.json, measured on this pool's B200s).
* cpu_baseline / --impl reference: the C restatement of the reference
             algorithm (oracle/, OpenMP over all host cores) on the same inputs.

Launch: python bench.py [--gpus N --steps K --warmup W] [--impl reference];
N > 1 under torch.distributed.run (one process per GPU, NCCL).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD_DESC = {
    "c1": "A=u0*0.9^|i-j|, B=u1*0.9^|i-j|",
    "c2": "A=B=sym(u*0.95^|i-j|)",
    "c3_l2": "A=sym(u0/(|i-j|^2+1)), B=sym(u1/(|i-j|^2+1))",
    "c3_l3": "A=sym(u0/(|i-j|^3+1)), B=sym(u1/(|i-j|^3+1))",
    "c5": "A=B=sym(u*0.98^|i-j|)",
}
METRIC = "SpAMM time & retained-leaf FP64 TFLOP/s vs tau, n=4096-65536, 1/2/4/8 B200"


def workload_string(cfg_name, n, leaf, taus):
    """config.workload -- the same string on the B200 arm and the reference arm."""
    return (f"{cfg_name}: n={n} leaf={leaf} {WORKLOAD_DESC.get(cfg_name, '')}, "
            f"tau sweep {list(taus)}, one spamm per tau per step")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", default="c2", choices=["c1", "c2", "c3_l2", "c3_l3", "c5"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--profile", action="store_true", help="short run for ncu: no e2e/cpu/context")
    p.add_argument("--dtype", default="f64", choices=["f64", "f32"],
                   help="storage/compute precision (c5's FP32 variant: f32)")
    p.add_argument("--dist", action="store_true",
                   help="use the torch.distributed (NCCL) path even at world size 1")
    p.add_argument("--no-extra", action="store_true",
                   help="skip the per-config lines and the same-run FP64 peak")
    return p.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def leaf_flops(leaf, retained):
    return 2.0 * leaf ** 3 * retained


# ------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        rows = []
        if self.path and os.path.exists(self.path):
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) >= 9 and f[1].isdigit():
                    rows.append(f)
            os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [int(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        loaded = [x for x in sm if x > 600] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": int(rows[0][2]),
                "reasons": reasons, "samples": len(rows)}


# --------------------------------------------------------------- the oracle
def cpu_reference(a, leaf, taus, steps, warmup, b=None):
    """Time the oracle port (C restatement of the reference, OpenMP over all
    host cores) on the same workload: per tau cull + leaf stage + C's tree on
    prebuilt operand pyramids, like the GPU's value leg."""
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count()))
    from oracle import oracle

    pa = oracle.pad(a, leaf)
    na, oa = oracle.build_pyramid(pa, leaf)
    if b is None or b is a:
        pb, nb_, ob = pa, na, oa
    else:
        pb = oracle.pad(b, leaf)
        nb_, ob = oracle.build_pyramid(pb, leaf)
    N = pa.shape[0]
    depth = oracle.depth_for(N, leaf)
    times, flops = [], 0.0
    for step in range(warmup + steps):
        t0 = time.perf_counter()
        f = 0.0
        for tau in taus:
            st, trip, _, _ = oracle.cull(na, oa, nb_, ob, depth, N, tau, collect_boxes=False)
            c = oracle.leaf_stage(pa, pb, leaf, trip)
            oracle.build_pyramid(c, leaf)
            f += leaf_flops(leaf, st["leaf_matmuls"])
        dt = time.perf_counter() - t0
        if step >= warmup:
            times.append(dt)
            flops += f
    return flops / sum(times) / 1e12, sum(times) / len(times), int(os.environ["OMP_NUM_THREADS"])


def run_reference(args, cfg_name):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_1011_3534_b200 import workloads
    if cfg_name in workloads.DEVICE_CONFIGS:
        print(json.dumps({"impl": "reference", "unavailable":
                          f"{cfg_name} is generated on the GPU (> 100 GB of host staging); "
                          "the CPU port runs on c1-c3"}), flush=True)
        return
    a, b, leaf, taus = workloads.make_config(cfg_name)
    steps = max(1, args.steps)
    warm = max(0, args.warmup)
    value, sec_per_step, cores = cpu_reference(a, leaf, taus, steps, warm, b)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": steps, "warmup": warm,
        "ms_per_step": sec_per_step * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY §8(d))",
        "config": {"workload": workload_string(cfg_name, a.shape[0], leaf, taus),
                   "l2": "n/a (CPU)"},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "port",
                         "sample": f"full {cfg_name} tau sweep per step"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- the GPU
def fp64_peak():
    path = os.path.join(ROOT, "profiles", "fp64_peaks.json")
    with open(path) as fh:
        p = json.load(fh)
    peak = max(v for k, v in p.items() if k.startswith("dmma_") and k.endswith("_tflops"))
    return peak, "profiles/fp64_peaks.json (DMMA mma.sync f64 microbenchmark, this pool's B200)"


def fp32_peak():
    """FP32 FMA (CUDA-core) roofline for the f32 leaf kernels."""
    path = os.path.join(ROOT, "profiles", "fp64_peaks.json")
    if os.path.exists(path):
        with open(path) as fh:
            p = json.load(fh)
        if "ffma_tflops" in p:
            return p["ffma_tflops"], "profiles/fp64_peaks.json (FFMA microbenchmark, this pool's B200)"
    return 148 * 128 * 2 * 1.965e9 / 1e12, "nominal: 148 SMs x 128 FMA/clk x 2 x 1965 MHz"


def k3_traffic():
    path = os.path.join(ROOT, "profiles", "k3_traffic.json")
    if os.path.exists(path):
        with open(path) as fh:
            return json.load(fh)
    return None


E2E_REGIONS = 5  # timed e2e regions per run (median reported, all listed)


def fp64_peak_same_run():
    """The FP64 DMMA / DFMA microbenchmark (tools/fp64_peaks.cu, built by
    __graft_entry__.build()) run inside this bench run: the roofline
    denominator measured on this box, now."""
    exe = os.path.join(ROOT, "tools", "bin", "fp64_peaks")
    if not os.path.exists(exe):
        return None
    try:
        out = json.loads(subprocess.check_output([exe], timeout=120).decode())
    except Exception:
        return None
    dmma = max(v for k, v in out.items() if k.startswith("dmma_") and k.endswith("_tflops"))
    return {"dmma_tflops": dmma, "dfma_tflops": out.get("dfma_tflops"),
            "ffma_tflops": out.get("ffma_tflops"), "source": "tools/bin/fp64_peaks, this run"}


def measure_config(sp, cfg_name, dtype, flush, steps=3, warmup=1):
    """One BASELINE config device-timed exactly like `value` (L2 flushed,
    CUDA events on the library's stream around every multiply): retained-leaf
    TFLOP/s and the leaf-product kernel's roofline fraction."""
    import torch

    from paper_1011_3534_b200 import workloads

    tdt = torch.float32 if dtype == "f32" else torch.float64
    if cfg_name in workloads.DEVICE_CONFIGS:
        at, _, leaf, taus = workloads.make_config_device(cfg_name, "cuda", tdt)
        n = at.shape[0]
        a = sp.from_device_pointer(at.data_ptr(), n, leaf_size=leaf,
                                   dtype=np.float32 if dtype == "f32" else np.float64)
        del at
        torch.cuda.empty_cache()
        b = a
    else:
        ah, bh, leaf, taus = workloads.make_config(cfg_name)
        n = ah.shape[0]
        npdt = np.float32 if dtype == "f32" else np.float64
        a = sp.from_dense(ah, leaf_size=leaf, dtype=npdt)
        b = a if bh is ah else sp.from_dense(bh, leaf_size=leaf, dtype=npdt)
    f = ms = gemm = 0.0
    per_tau = {}
    for step in range(warmup + steps):
        for tau in taus:
            flush.zero_()
            torch.cuda.synchronize()
            c, st, det = sp.spamm_detailed(a, b, sp.SpammConfig(tau=tau))
            del c
            if step >= warmup:
                f += leaf_flops(leaf, st.leaf_matmuls)
                ms += det.ms_total
                gemm += det.ms_gemm
                per_tau[tau] = (st.leaf_matmuls, det.ms_total)
    del a, b
    torch.cuda.empty_cache()
    f64_tensor = dtype == "f64" and leaf >= 32
    peak, _ = fp64_peak() if f64_tensor else fp32_peak()
    k3 = f / (gemm * 1e-3) / 1e12 if gemm > 0 else 0.0
    return {"workload": workload_string(cfg_name, n, leaf, taus), "dtype": dtype,
            "value": f / (ms * 1e-3) / 1e12, "unit": "TFLOP/s",
            "ms_per_multiply": ms / (steps * len(taus)),
            "per_tau": [{"tau": t, "retained": r, "ms": m} for t, (r, m) in per_tau.items()],
            "roofline": {"kernel": "K3", "achieved": k3, "peak": peak,
                         "bound": "tensor" if f64_tensor else "fma", "frac": k3 / peak},
            "timing": "CUDA events per multiply, L2 flushed, inputs resident; "
                      f"{steps} steps after {warmup} warm-up"}


def run_b200(args, cfg_name):
    import torch
    import paper_1011_3534_b200 as sp
    from paper_1011_3534_b200 import workloads

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    sp.set_device(local)
    use_dist = world > 1 or args.dist
    if use_dist:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1011_3534_b200 import distributed as spd

    dev_cfg = cfg_name in workloads.DEVICE_CONFIGS
    tdtype = torch.float32 if args.dtype == "f32" else torch.float64
    # c5 (one multiply per step) under torchrun: the distributed layout --
    # rank 0 generates A, ShardedTree.scatter sends each rank its block rows
    # (NCCL), every multiply is spamm_sharded (plan, halo exchange of the
    # operand blocks other ranks hold, band products, merged statistics)
    sharded = dev_cfg and use_dist
    A_sh = None
    if sharded:
        cfgd = workloads.DEVICE_CONFIGS[cfg_name]
        n, leaf, taus = cfgd["n"], cfgd["leaf"], list(cfgd["taus"])
        at = (workloads.make_config_device(cfg_name, f"cuda:{local}", tdtype)[0]
              if rank == 0 else None)
        A_sh = spd.ShardedTree.scatter(at, n, leaf, spd.Comm(), dtype=tdtype)
        del at
        torch.cuda.empty_cache()
        a = b = A_sh.tree
        a_host = b_host = None
    elif dev_cfg:  # generated on the GPU (c5: > 100 GB of host staging otherwise)
        at, _, leaf, taus = workloads.make_config_device(cfg_name, f"cuda:{local}", tdtype)
        n = at.shape[0]
        a_host = b_host = None
        a = sp.from_device_pointer(at.data_ptr(), n, leaf_size=leaf,
                                   dtype=np.float32 if args.dtype == "f32" else np.float64)
        del at
        torch.cuda.empty_cache()
        b = a
    else:
        a_host, b_host, leaf, taus = workloads.make_config(cfg_name)
        if args.dtype == "f32":
            a_host = a_host.astype(np.float32)
            b_host = a_host if b_host is None or b_host is a_host else b_host.astype(np.float32)
        n = a_host.shape[0]
        a = sp.from_dense(a_host, leaf_size=leaf, dtype=a_host.dtype)
        b = a if b_host is a_host else sp.from_dense(b_host, leaf_size=leaf, dtype=b_host.dtype)
    shard = spd.row_shard(rank, world, n, leaf) if use_dist else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    nbk = spd.padded_blocks(n, leaf)
    # the step's multiplies (one per tau) as pieces: at N = 1 every tau whole;
    # at N > 1 the sweep is partitioned over the ranks -- a tau whole or split
    # into C block-row shards, balanced by retained triples per row (measured
    # by one planning multiply per tau; every rank computes the same plan, no
    # collective in the data path)
    pieces = [(q, None) for q in range(len(taus))]
    plan_desc = None
    if use_dist and not sharded:
        row_counts = []
        for tau in taus:
            _, _, det = sp.spamm_detailed(a, b, sp.SpammConfig(tau=tau), keep_triples=True)
            row_counts.append(np.bincount(det.triples[:, 0], minlength=nbk)[:nbk])
        plan, _ = spd.sweep_plan(world, n, leaf, row_counts)
        pieces = [(q, None if rows == (0, nbk) else rows) for q, rows in plan[rank]]
        plan_desc = [[(float(taus[q]), list(rows)) for q, rows in p] for p in plan]

    def one_step(collect=None):
        f, ms, gemm, launches = 0.0, 0.0, 0.0, 0
        per_tau = []
        for q, rows in pieces:
            tau = taus[q]
            flush.zero_()
            torch.cuda.synchronize()
            if sharded:  # the whole distributed multiply, timed on the device around the call
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                c, st, det = spd.spamm_sharded(A_sh, A_sh, sp.SpammConfig(tau=tau))
                e1.record()
                torch.cuda.synchronize()
                # (st: the global statistics; count each rank's share once in the sum below)
                f += leaf_flops(leaf, st.leaf_matmuls) / world
                ms += e0.elapsed_time(e1)
                gemm += det.ms_gemm if det is not None else 0.0
                launches += det.kernel_launches if det is not None else 0
                per_tau.append((tau, st.leaf_matmuls, e0.elapsed_time(e1),
                                det.ms_gemm if det is not None else 0.0,
                                det.ms_cull if det is not None else 0.0,
                                det.ms_ctree if det is not None else 0.0,
                                det.n_groups if det is not None else 0,
                                int(det.tier_survivors[-1]) if det is not None and det.tier_survivors
                                else 0))
                del c
                continue
            c, st, det = sp.spamm_detailed(a, b, sp.SpammConfig(tau=tau), rows=rows)
            f += leaf_flops(leaf, st.leaf_matmuls)
            ms += det.ms_total
            gemm += det.ms_gemm
            launches += det.kernel_launches
            per_tau.append((tau, st.leaf_matmuls, det.ms_total, det.ms_gemm, det.ms_cull,
                            det.ms_ctree, det.n_groups))
            del c
        return f, ms, gemm, launches, per_tau

    for _ in range(args.warmup):
        one_step()
    if use_dist:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    tot_f = tot_ms = tot_gemm = 0.0
    launches = 0
    per_tau_all = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            f, ms, gemm, la, per_tau = one_step()
            if use_dist:
                t = torch.tensor([ms], dtype=torch.float64, device="cuda")
                torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
                ms = float(t.item())
                fl = torch.tensor([f], dtype=torch.float64, device="cuda")
                torch.distributed.all_reduce(fl)
                f = float(fl.item())
            tot_f += f
            tot_ms += ms
            tot_gemm += gemm
            launches += la
            per_tau_all.append(per_tau)
    torch.cuda.synchronize()
    if use_dist:
        torch.distributed.barrier()
    clocks = clk.summary()
    value = tot_f / (tot_ms * 1e-3) / 1e12
    ms_per_step = tot_ms / args.steps

    # per-tau table from the last step
    table = [{"tau": t, "retained": r, "frac_of_nb3": r / (a.block_grid ** 3), "ms": m,
              "gemm_ms": g, "cull_ms": cu, "ctree_ms": ct, "c_blocks": ng,
              "tflops": leaf_flops(leaf, r) / (m * 1e-3) / 1e12}
             for (t, r, m, g, cu, ct, ng, *_) in per_tau_all[-1]]

    f64_tensor = args.dtype == "f64" and leaf >= 32
    peak, peak_src = fp64_peak() if f64_tensor else fp32_peak()
    # K3 roofline from this rank's own flops and K3 event time
    # (sharded: this rank's own retained triples, the last tier's survivors)
    local_f = sum(leaf_flops(leaf, x[7] if len(x) > 7 else x[1]) for step in per_tau_all for x in step)
    local_gemm = sum(x[3] for step in per_tau_all for x in step)
    achieved = local_f / (local_gemm * 1e-3) / 1e12 if local_gemm > 0 else 0.0
    traffic = k3_traffic()
    kname = ("leaf_dmma_ws_kernel<%d> (K3)" % min(leaf, 64) if f64_tensor
             else "leaf_sgemm_kernel (K3, FP32 FMA pipe)" if args.dtype == "f32" and leaf >= 64
             else "leaf_simt_kernel (K3, FMA pipe)")
    roofline = {"bound": "tensor" if f64_tensor else "fma", "kernel": kname, "achieved": achieved,
                "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "peak_source": peak_src,
                "traffic": (traffic.get("bytes_per_launch") if traffic and cfg_name == "c2"
                            and f64_tensor else None),
                "algorithmic": "2*b^3 flop per retained leaf triple / K3 event time"}

    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": args.dtype,
        "data": ("synthetic, generated on the GPU (torch Philox stream, the recipe's formula)"
                 if dev_cfg else "synthetic (seeded numpy PCG64, SURVEY §8(d))"),
        "config": {"workload": workload_string(cfg_name, n, leaf, taus),
                   "l2": "flushed (256 MiB write) before every multiply",
                   "parallelism": (f"row-distributed over {world} ranks (ShardedTree: rows scattered "
                                   f"from rank 0 over NCCL, per multiply a halo exchange of the "
                                   f"operand blocks other ranks hold, C kept as bands)"
                                   if sharded else
                                   f"tau sweep partitioned over {world} ranks: each tau whole or "
                                   f"split into C block-row shards (no data-path collective)"
                                   if use_dist else "single GPU"),
                   "plan": plan_desc,
                   "per_tau": table},
        "roofline": roofline,
        "clocks": clocks,
        # this library's kernels launched inside the timed region (all K steps)
        "gpu_launches": launches,
        "gpu_launches_per_step": launches // max(args.steps, 1),
    }

    if rank == 0 and world == 1 and not args.profile and n <= 16384:
        # --- context: dense cuBLAS GEMM on the same matrices
        at = torch.from_numpy(a_host).cuda()
        bt = at if b_host is a_host else torch.from_numpy(b_host).cuda()
        for _ in range(2):
            torch.matmul(at, bt)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        torch.matmul(at, bt)
        e1.record()
        torch.cuda.synchronize()
        dg = e0.elapsed_time(e1)
        line["config"]["context_dense_cublas_gemm"] = {
            "ms": dg, "tflops": 2.0 * n ** 3 / (dg * 1e-3) / 1e12}
        del at, bt
    elif rank == 0 and world == 1 and not args.profile:
        # 2 n^3 at the measured cuBLAS DGEMM 8192^3 rate (a 65536^3 product takes ~16 s)
        with open(os.path.join(ROOT, "profiles", "fp64_peaks.json")) as fh:
            rate = json.load(fh)["cublas_dgemm_8192_tflops"]
        line["config"]["context_dense_cublas_gemm"] = {
            "ms": 2.0 * n ** 3 / (rate * 1e12) * 1e3, "tflops": rate,
            "note": "estimated from the measured cuBLAS DGEMM 8192^3 rate"}

    if rank == 0 and world == 1 and not args.profile and not args.no_extra:
        same = fp64_peak_same_run()
        if same is not None:
            roofline["peak_same_run"] = same
            if f64_tensor:
                roofline["frac_same_run"] = achieved / same["dmma_tflops"]
        if cfg_name == "c2":
            # the rest of the metric's n range, device-timed like `value`
            # (parity for each: tests/test_gpu_parity.py, tests/test_gpu_fullsize.py)
            # (an extra that fails -- e.g. no room for c5's 34 GB operands on a
            # shared box -- is reported in its entry; the c2 line still prints)
            per = []
            for name, dt in (("c3_l2", "f64"), ("c5", "f64"), ("c5", "f32")):
                try:
                    per.append(measure_config(sp, name, dt, flush))
                except Exception as exc:  # noqa: BLE001
                    per.append({"workload": name, "dtype": dt,
                                "error": f"{type(exc).__name__}: {exc}"[:300]})
                    torch.cuda.empty_cache()
            line["config"]["per_config"] = per

    if not args.no_e2e and not args.profile:
        if dev_cfg:
            line["e2e"] = {"unavailable": "inputs generated on the GPU: host staging of a "
                                          f"{n}x{n} operand is {n * n * 8 / 1e9:.0f} GB"}
        elif use_dist:
            with NumaLocal(local):
                line["e2e"] = e2e_leg_dist(args, sp, spd, a_host, leaf, taus, pieces, b_host)
        else:
            with NumaLocal(local):
                # the K-step region is tens of milliseconds of host wall clock:
                # measured E2E_REGIONS times (each with its own warm-up), the
                # median region is reported and every region is listed
                regions = sorted((e2e_leg(args, sp, a_host, leaf, taus, shard, use_dist, b_host)
                                  for _ in range(E2E_REGIONS)), key=lambda r: r["ms_per_step"])
                line["e2e"] = regions[len(regions) // 2]
                line["e2e"]["regions_ms_per_step"] = [r["ms_per_step"] for r in regions]
                line["e2e"]["timing"] += (f"; median of {E2E_REGIONS} timed regions of "
                                          f"{args.steps} steps each (all listed)")
                if not use_dist:
                    # beside it: every product read back dense, as a reference
                    # caller does with to_dense(C) (quadtree.py:264-266)
                    try:
                        line["e2e"]["to_dense"] = e2e_leg(args, sp, a_host, leaf, taus, shard,
                                                          use_dist, b_host, readback="dense")
                    except Exception as exc:  # noqa: BLE001
                        line["e2e"]["to_dense"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    if rank == 0 and world == 1 and not args.no_cpu and not args.profile and not dev_cfg:
        cv, sec, cores = cpu_reference(a_host, leaf, taus, 1, 1, b_host)
        line["cpu_baseline"] = {"value": cv, "unit": "TFLOP/s", "cores": cores, "kind": "port",
                                "sample": f"one full {cfg_name} tau sweep ({sec:.2f} s) after "
                                          "one warm-up sweep",
                                "ms_per_step": sec * 1e3}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if use_dist:
        torch.distributed.destroy_process_group()


class NumaLocal:
    """Run the e2e leg on the CPUs nearest the GPU (NVML's ideal affinity), so
    the pinned staging buffers it allocates land in that NUMA node: a buffer
    on the far socket crosses the inter-socket link and cut host<->device
    bandwidth by ~40 % in some runs.  The previous affinity is restored."""

    def __init__(self, device):
        self.device = device
        self.saved = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.saved = os.sched_getaffinity(0)
            import torch
            # NVML numbers all GPUs, CUDA only the visible ones: match by UUID
            uuid = "GPU-" + str(torch.cuda.get_device_properties(self.device).uuid)
            h = pynvml.nvmlDeviceGetHandleByUUID(uuid.encode())
            pynvml.nvmlDeviceSetCpuAffinity(h)
        except Exception:  # no NVML / no affinity support: leave as is
            self.saved = None
        return self

    def __exit__(self, *exc):
        if self.saved is not None:
            try:
                os.sched_setaffinity(0, self.saved)
            except Exception:
                pass


def e2e_leg(args, sp, a_host, leaf, taus, shard, use_dist, b_host=None, readback="blocks"):
    """The same metric through the public API with host buffers.

    Every step: pinned host A (and B) -> from_dense (H2D + K1 pyramid), one
    spamm per tau, and each product back to pinned host memory -- as its
    nonzero leaf blocks and norm pyramid (readback="blocks"), or as the dense
    n x n matrix through to_dense (readback="dense", what a caller of the
    reference's API reads).  With row shards each rank multiplies its C
    block rows and reads back only those (bands partition C); wall time is
    the max over ranks."""
    import torch

    n = a_host.shape[0]
    tdt = torch.float32 if a_host.dtype == np.float32 else torch.float64
    esz = a_host.dtype.itemsize
    # two pinned input buffers per operand, alternating between steps (the
    # next step's input is copied while this step multiplies)
    pin_a = [torch.empty((n, n), dtype=tdt, pin_memory=True).numpy() for _ in range(2)]
    for p in pin_a:
        p[...] = a_host
    same = b_host is None or b_host is a_host
    if not same:
        pin_b = [torch.empty((n, n), dtype=tdt, pin_memory=True).numpy() for _ in range(2)]
        for p in pin_b:
            p[...] = b_host

    def inputs(it):
        """from_dense of step it's operands, returning before the copy is done:
        host->device copy + pyramid on the library's copy-in stream."""
        at = sp.from_dense(pin_a[it % 2], leaf_size=leaf, dtype=pin_a[0].dtype, wait=False)
        bt = at if same else sp.from_dense(pin_b[it % 2], leaf_size=leaf, dtype=pin_b[0].dtype,
                                           wait=False)
        return at, bt
    # the product comes back as its nonzero leaf blocks (the tree's content;
    # empty blocks are implicit zeros), in one transfer per multiply; with row
    # shards each rank holds (and reads back) only its own block rows
    nbk = -(-n // leaf)
    G = (1 << (max(nbk - 1, 0)).bit_length()) ** 2
    # one pinned buffer per tau: a product's copy overlaps the next multiply
    # (and the next step's host->device copy of A: PCIe is full duplex); a
    # buffer is reused only after its previous transfer has been waited for
    if readback == "dense":
        pin_blk = [torch.empty((n, n), dtype=tdt, pin_memory=True).numpy() for _ in taus]
    else:
        pin_blk = [torch.empty((G, leaf, leaf), dtype=tdt, pin_memory=True).numpy() for _ in taus]
    pending = [None] * len(taus)
    t0 = None
    e_f = 0.0
    d2h = 0
    total = args.warmup + args.steps
    nxt = None
    for it in range(total):
        if it == args.warmup:
            for p in pending:
                if p is not None:
                    p.wait()
            torch.cuda.synchronize()
            if use_dist:
                torch.distributed.barrier()
            t0 = time.perf_counter()
            d2h = 0
        at, bt = nxt if nxt is not None else inputs(it)
        # prefetch: the next step's inputs go host->device while this step's
        # multiplies run -- never across the start or the end of the timed
        # region, so every timed step's copy is inside it
        nxt = inputs(it + 1) if it + 1 < total and it + 1 != args.warmup else None
        f = 0.0
        for q, tau in enumerate(taus):
            if shard is None:
                c, st = sp.spamm(at, bt, sp.SpammConfig(tau=tau))
            else:
                c, st, _ = sp.spamm_detailed(at, bt, sp.SpammConfig(tau=tau), rows=shard)
            if readback == "dense":
                sp.to_dense(c, out=pin_blk[q])
                d2h += pin_blk[q].nbytes
            else:
                if pending[q] is not None:
                    pending[q].wait()
                pending[q] = c.nonzero_blocks(out=pin_blk[q], wait=False)
                d2h += (pending[q].blocks.nbytes + pending[q].ids.nbytes + c._pyramid()[2].nbytes
                        + c._pyramid()[3].nbytes)
            f += leaf_flops(leaf, st.leaf_matmuls)
            del c
        del at, bt
        if it >= args.warmup:
            e_f += f
        if os.environ.get("SPAMM_E2E_DEBUG"):
            print(f"[e2e] step {it} t={(time.perf_counter() - (t0 or 0)) * 1e3:.3f} ms",
                  file=sys.stderr, flush=True)
    for p in pending:
        if p is not None:
            p.wait()
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    d2h = d2h // max(args.steps, 1)
    if use_dist:
        t = torch.tensor([el, e_f, float(d2h)], dtype=torch.float64, device="cuda")
        mx = t[:1].clone()
        torch.distributed.all_reduce(mx, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(t[1:])
        el, e_f, d2h = float(mx.item()), float(t[1].item()), int(t[2].item())
    return {"value": e_f / el / 1e12, "unit": "TFLOP/s",
            "h2d_bytes_per_step": n * n * esz * (1 if same else 2) * (dist_world() if use_dist else 1),
            "d2h_bytes_per_step": d2h,
            "ms_per_step": el / args.steps * 1e3,
            "result": ("each product read back dense through to_dense(C, out=pinned) "
                       "(materialised on the device, one n x n copy)" if readback == "dense" else
                       "each product read back as its nonzero leaf blocks + norm pyramid "
                       "(QuadTreeMatrix.nonzero_blocks, copy-out stream overlapping the next "
                       "call; all copies waited for inside the timed region)"),
            "pipelining": "from_dense(wait=False): step s+1's host->device copy of A runs on the "
                          "copy-in stream during step s's multiplies (PCIe full duplex with the "
                          "read-backs); no copy crosses the timed region's boundaries",
            "timing": "host wall clock around synchronous public-API calls (max over ranks)"}


def e2e_leg_dist(args, sp, spd, a_host, leaf, taus, pieces, b_host=None):
    """e2e at N > 1 ranks: the operands cross PCIe once in total -- each rank
    copies its band of padded rows from pinned host memory, the bands are
    all-gathered over NVLink (NCCL) into every rank's tree storage (the
    pyramid is then built locally) -- and each rank runs its pieces of the
    sweep and reads back only their products (a piece's product holds only
    its rows), the copies overlapping the next piece.  Wall time: max over
    ranks."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    n = a_host.shape[0]
    N = spd.padded_blocks(n, leaf) * leaf
    tdt = torch.float32 if a_host.dtype == np.float32 else torch.float64
    same = b_host is None or b_host is a_host
    R0, R1 = rank * N // world, (rank + 1) * N // world  # padded rows of this rank
    assert N % world == 0, "equal bands for the all-gather"
    h = R1 - R0
    hosts = [a_host] if same else [a_host, b_host]
    pins = []
    for x in hosts:  # this rank's band, zero-padded to N columns, in pinned memory
        p = torch.zeros((h, N), dtype=tdt, pin_memory=True)
        r1 = min(R1, n)
        if r1 > R0:
            p[:r1 - R0, :n] = torch.from_numpy(np.ascontiguousarray(x[R0:r1]))
        pins.append(p)
    bands = [torch.empty((h, N), dtype=tdt, device="cuda") for _ in pins]
    fulls = [torch.empty((N, N), dtype=tdt, device="cuda") for _ in pins]
    nbk = N // leaf
    pin_blk = [torch.empty((nbk * nbk, leaf, leaf), dtype=tdt, pin_memory=True).numpy()
               for _ in pieces]
    pending = [None] * len(pieces)
    h2d = sum(p.numel() * p.element_size() for p in pins)

    def operands():
        trees = []
        for p, band, full in zip(pins, bands, fulls):
            band.copy_(p, non_blocking=True)                  # PCIe: 1/world of the rows
            dist.all_gather_into_tensor(full, band)           # NVLink
            trees.append(spd.tree_from_padded(full, n, leaf))  # pyramid on every rank
        return trees[0], trees[-1]

    t0 = None
    e_f = 0.0
    d2h = 0
    for it in range(args.warmup + args.steps):
        if it == args.warmup:
            for q in pending:
                if q is not None:
                    q.wait()
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            d2h = 0
        at, bt = operands()
        f = 0.0
        for j, (q, rows) in enumerate(pieces):
            c, st, _ = sp.spamm_detailed(at, bt, sp.SpammConfig(tau=taus[q]), rows=rows)
            if pending[j] is not None:
                pending[j].wait()
            pending[j] = c.nonzero_blocks(out=pin_blk[j], wait=False)
            d2h += (pending[j].blocks.nbytes + pending[j].ids.nbytes + c._pyramid()[2].nbytes
                    + c._pyramid()[3].nbytes)
            f += leaf_flops(leaf, st.leaf_matmuls)
            del c
        del at, bt
        if it >= args.warmup:
            e_f += f
    for q in pending:
        if q is not None:
            q.wait()
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    d2h = d2h // max(args.steps, 1)
    t = torch.tensor([el, e_f, float(d2h), float(h2d)], dtype=torch.float64, device="cuda")
    mx = t[:1].clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    dist.all_reduce(t[1:])
    el, e_f, d2h, h2d = float(mx.item()), float(t[1].item()), int(t[2].item()), int(t[3].item())
    return {"value": e_f / el / 1e12, "unit": "TFLOP/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": el / args.steps * 1e3,
            "result": "each rank's products read back as their nonzero leaf blocks + norm "
                      "pyramid (copy-out stream overlapping the next piece)",
            "operands": "each rank copies 1/N of the padded rows host->device; NCCL all-gather "
                        "over NVLink assembles the operand on every rank",
            "timing": "host wall clock around synchronous public-API calls (max over ranks)"}


def dist_world():
    import torch.distributed as dist
    return dist.get_world_size()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args, args.config)
    else:
        run_b200(args, args.config)


if __name__ == "__main__":
    main()
