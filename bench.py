#!/usr/bin/env python
"""Benchmark of the BBMM mBCG hot path on B200 (one JSON line on rank 0).

A "step" = one full one-call exact-GP MLL + gradient (bbmm_mll_and_grad):
pivoted Cholesky (k) -> probes -> mBCG (p iterations of Khat*[y, z_1..z_t])
-> SLQ log-det -> derivative pass, on BASELINE.json's metric workload
(C4: RBF, n = 1,000,000, d = 3, t = 16, k = 100, p = 20, on-the-fly K).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

Multi-GPU: launched by torchrun (one process per GPU); rows of K are
partitioned across ranks (strong scaling: the same n = 1M problem).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

BASELINE = json.load(open(os.path.join(ROOT, "BASELINE.json")))
METRIC = BASELINE["metric"]


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


# what the K^D arithmetic is, per operator (matmul_path of bbmm_stats_t)
DTYPE = {
    0: "fp32 kernel values x fp64 D, fp64 accumulation (FP64ACC, CUDA cores); fp64 CG",
    1: "stored fp32 K x fp64 D, fp64 accumulation (FP64ACC, CUDA cores); fp64 CG",
    2: "23-bit fixed-point k~ (3 u8 slices; fp32 MUFU ex2 of an fp16-split tensor-core exponent) x "
       "31-bit fixed-point D (4 u8 slices; Matern 39-bit, 5 slices), exact int32 accumulation of "
       "the slice products on tcgen05 (q0 p0, < 2^-38 of the scale, dropped); fp64 CG",
    3: "stored 30-bit fixed-point K (4 u8 slices, fp64-built) x 55-bit fixed-point D (7 u8 slices), "
       "exact int32 accumulation on tcgen05; fp64 CG",
}
DTYPE31M = ("31-bit fixed-point k~ (4 u8 slices: the fp32 Matern-5/2 value exactly, from fp32 direct "
            "distances and MUFU sqrt + ex2) x 55-bit fixed-point D (7 u8 slices), exact int32 "
            "accumulation of the slice products on tcgen05 (those below 2^-52 of the scale dropped); "
            "fp64 CG")
DTYPE31 = ("31-bit fixed-point k~ (4 u8 slices: the fp32 MUFU ex2 value exactly, of an fp16-split "
           "tensor-core exponent) x 31-bit fixed-point D (4 u8 slices), exact int32 accumulation of "
           "the slice products on tcgen05 (those below 2^-38 of the scale dropped); fp64 CG")


def work_per_matmul(cfg):
    """Algorithmic work of one Khat*D: n^2 kernel
    evaluations (one ex2 each for RBF; ex2 + sqrt for Matern) and 2 n^2 c
    useful contraction flops."""
    c = cfg.t + 1
    pairs = float(cfg.n) * float(cfg.n)
    return pairs, 2.0 * pairs * c


def tensor_frac(cfg, world, mm_ms, pk, detail=False, kgrid=23):
    """Tensor-pipe work of one K1-TC launch, per 128 x 128 tile: the distance
    (RBF: fp16 hi/lo, K = 32 packed at DA = 8, else 3 round16(DA); Matern: none) and the int8
    slice MMAs (K = 128; q2, q1 at N = ND BLK, q0 trimmed to round16(3 BLK), the 31-bit grid's
    residual slice at round16(2 BLK)), as dense-bf16-equivalent flops (f16 x1, int8 x0.5) over
    the launch time vs the measured bf16 peak."""
    r16 = lambda x: -(-x // 16) * 16
    c1 = cfg.t + 2
    da = -(-(cfg.d + 2) // 8) * 8
    if cfg.kind == synth.RBF:
        blk = -(-c1 // 4) * 4
        nb = 4 * blk
        kdist = 32 if da == 8 else 3 * r16(da)
        nsum = 2 * nb + min(nb, r16(3 * blk)) + (r16(2 * blk) if kgrid == 31 else 0)
    else:               # Matern: BLK = round16; five D slices x 3 k~ slices, or 7 x 4 (31-bit grid)
        blk = r16(c1)
        kdist = 0
        nsum = 15 * blk if kgrid != 31 else (7 + 6 + 5 + 4) * blk
    rows = -(-(-(-cfg.n // world)) // 128) * 128
    cols = -(-cfg.n // 128) * 128
    f16 = 2.0 * rows * cols * kdist
    i8 = 2.0 * rows * cols * nsum
    eq = f16 + 0.5 * i8
    ach = eq / (mm_ms * 1e-3) / 1e12
    peak = pk.get("bf16_tflops", 1590.0)
    return (ach / peak, ach, peak) if detail else ach / peak


# ------------------------------------------------------------------ clocks
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index=0, period=0.1):
        self.index, self.period = index, period
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for b, name in self.REASONS.items():
                    if mask & b:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}


# ----------------------------------------------------------- cpu baseline
def oracle_sample(cfg, pr, rows_target, seed=0):
    """Time the fp64 oracle's Khat*D on a bounded row sample of the workload
    (its dominant cost) and convert to the metric's unit."""
    import oracle
    c = cfg.t + 1
    rows = np.sort(np.random.default_rng(seed).choice(cfg.n, size=min(rows_target, cfg.n),
                                                      replace=False))
    D = synth.random_block(cfg.n, c, seed=4).astype(np.float64)
    t0 = time.perf_counter()
    oracle.kernel_matmul(cfg.kind, pr.X, pr.log_ls, pr.log_s, pr.log_noise, D, rows=rows)
    dt = time.perf_counter() - t0
    flops = 2.0 * len(rows) * cfg.n * c
    return dict(seconds=dt, rows=len(rows), gflops=flops / dt / 1e9, cores=oracle.num_threads())


def cpu_baseline(cfg, pr, rows_target=None):
    if rows_target is None:
        rows_target = int(os.environ.get("BBMM_ORACLE_ROWS", "0")) or None
    if rows_target is None:
        # calibrate: ~10-30 s of CPU work
        cal = oracle_sample(cfg, pr, 64)
        rows_target = int(max(64, min(cfg.n, 64 * 15.0 / max(cal["seconds"], 1e-3))))
    s = oracle_sample(cfg, pr, rows_target)
    c = cfg.t + 1
    per_matmul = s["seconds"] * cfg.n / s["rows"]
    return {"value": s["gflops"], "unit": "GFLOP/s", "cores": s["cores"], "kind": "oracle",
            "sample": (f"oracle fp64 Khat*D ({cfg.name}: n={cfg.n}, c={c}) on {s['rows']} sampled "
                       f"rows ({s['seconds']:.1f} s); extrapolated {per_matmul:.0f} s per full "
                       f"matmul, ~{per_matmul * (cfg.p + 2):.0f} s per MLL+grad")}


# ------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kmode", default=None, choices=[None, "onthefly", "stored"])
    ap.add_argument("--precision", default="int8exact", choices=["int8exact", "int8exact31", "int8exact23", "fp64acc", "fp32acc"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = synth.CONFIGS[args.config]

    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)

    import torch
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        # NCCL's own communicator lines (transport, NVLS / P2P channels) on stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    import paper_1809_11165_b200 as bb

    pr = synth.make_problem(cfg, seed=0)
    kmode = {"onthefly": bb.ONTHEFLY, "stored": bb.STORED}.get(
        args.kmode, bb.STORED if cfg.stored else bb.ONTHEFLY)
    ctx = bb.Context(local_rank)
    ctx.set_matmul_precision({"int8exact": bb.INT8EXACT, "int8exact31": bb.INT8EXACT31,
                              "int8exact23": bb.INT8EXACT23, "fp64acc": bb.FP64ACC,
                              "fp32acc": bb.FP32ACC}[args.precision])
    if world > 1:
        ctx.set_comm()
    X = torch.from_numpy(pr.X).cuda()
    y = torch.from_numpy(pr.y).cuda()
    h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)

    def step():
        return bb.mll_and_grad(ctx, X, y, h, cfg.t, cfg.k, cfg.p, tol=0.0, seed=1, kmode=kmode)

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    # inputs: X (n x d fp32) is 12 MB at C4, L2 is 126 MB, but every step
    # streams the full workspace (L: 800 MB, vectors ~0.7 GB) -> no L2 reuse
    # across steps; a 256 MB L2 flush is still done between steps.
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    times, stats = [], []
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            out = step()
            e1.record(stream)
            barrier()
            times.append(e0.elapsed_time(e1))
            stats.append(out["stats"])
    ms = float(np.mean(times))
    if dist:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # e2e: host buffers (pinned), H2D of X, y and D2H of (mll, grad) inside
    e2e = None
    if not args.no_e2e:
        Xh = torch.from_numpy(pr.X).pin_memory()
        yh = torch.from_numpy(pr.y).pin_memory()
        Xd = torch.empty_like(X)
        yd = torch.empty_like(y)
        etimes = []
        for _ in range(max(1, args.steps)):
            barrier()
            t0 = time.perf_counter()
            Xd.copy_(Xh, non_blocking=True)
            yd.copy_(yh, non_blocking=True)
            o = bb.mll_and_grad(ctx, Xd, yd, h, cfg.t, cfg.k, cfg.p, tol=0.0, seed=1, kmode=kmode)
            _ = (o["mll"], o["grad"].copy())      # scalars already on the host
            torch.cuda.synchronize()
            etimes.append((time.perf_counter() - t0) * 1e3)
        ems = float(np.mean(etimes))
        if dist:
            t = torch.tensor([ems], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        nq = int(np.atleast_1d(pr.log_ls).size) + 2
        e2e = {"value": None, "unit": "GFLOP/s", "ms_per_step": ems,
               "h2d_bytes_per_step": int(pr.X.nbytes + pr.y.nbytes),
               "d2h_bytes_per_step": int(8 * (1 + nq))}

    pairs, flops = work_per_matmul(cfg)
    iters = stats[-1]["iters"]
    value = iters * flops / (ms * 1e-3) / 1e9          # whole-step effective GFLOP/s
    if e2e:
        e2e["value"] = iters * flops / (e2e["ms_per_step"] * 1e-3) / 1e9
    # dominant kernel: Khat*D (K1), timed live with CUDA events on the launch stream
    mm_ms = float(np.mean([s["ms_matmul"] / max(s["matmul_launches"], 1) for s in stats]))
    pk, src = peaks()
    clocks = clk.summary()
    f_mhz = pk.get("sm_max_mhz", 1965.0)
    loc_pairs = pairs / world
    if cfg.kind == synth.RBF:
        mufu_per_pair = 1.0
    else:
        mufu_per_pair = 2.0
    peak_exp = 16.0 * 148 * f_mhz * 1e6 / 1e9          # Gops/s of the MUFU pipe
    achieved = loc_pairs * mufu_per_pair / (mm_ms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"traffic_{cfg.name}.json")
    path = stats[-1]["matmul_path"]
    if os.path.exists(tp):
        tj = json.load(open(tp))
        if tj.get("kernel_path") == path:     # measured for the kernel timed here
            traffic = tj.get("dram_bytes_per_launch")
    kname = {0: "k1_onthefly (CUDA-core Khat*D)", 1: "k2_stored (fp32 K, CUDA-core Khat*D)",
             2: "k1tc2_rbf (tcgen05 exact Khat*D)",
             3: "k2tc_stored (int8-slice K on tcgen05, exact Khat*D)"}[path]
    if path in (1, 3):
        # stored K: HBM-bound, algorithmic bytes = the stored representation per launch
        nloc = -(-cfg.n // world)
        if path == 3:
            byts = 4.0 * (-(-nloc // 128) * 128) * (-(-cfg.n // 384) * 384)
        else:
            byts = 4.0 * nloc * (-(-cfg.n // 4) * 4)
        gbs = byts / (mm_ms * 1e-3) / 1e9
        roofline = {"bound": "hbm", "kernel": kname, "achieved": gbs, "peak": pk["hbm_gbs"],
                    "unit": "GB/s", "frac": gbs / pk["hbm_gbs"], "traffic": traffic,
                    "peak_source": f"hbm_gbs of MEASURED_PEAKS.json ({src})",
                    "kernel_ms": mm_ms,
                    "kernel_gflops": loc_pairs * 2 * (cfg.t + 1) / (mm_ms * 1e-3) / 1e9}
    else:
        roofline = {"bound": "alu", "kernel": kname, "achieved": achieved,
                    "peak": peak_exp, "unit": "Gop/s (MUFU ex2/sqrt)", "frac": achieved / peak_exp,
                    "traffic": traffic,
                    "peak_source": f"derived: 16 MUFU ops/clk/SM x 148 SMs x {f_mhz:.0f} MHz "
                                   f"(sm_max_mhz of MEASURED_PEAKS.json, {src})",
                    "kernel_ms": mm_ms,
                    "kernel_gflops": loc_pairs * 2 * (cfg.t + 1) / (mm_ms * 1e-3) / 1e9}
        if path == 2:
            # secondary: the implementation's own tensor-pipe work (fp16 distance + int8 slice
            # products, as dense-bf16-equivalent flops) -- not the method's work
            tf, tach, tpk = tensor_frac(cfg, world, mm_ms, pk, detail=True,
                                        kgrid=stats[-1].get("kgrid_bits", 23))
            roofline["tensor_impl"] = {"achieved_tflops_bf16eq": tach, "peak": tpk, "frac": tf}
    launches = int(np.sum([s["gpu_launches"] for s in stats]))
    line = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "s_per_mll_grad": ms / 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": (DTYPE[path] if not (path == 2 and stats[-1].get("kgrid_bits") == 31)
                  else DTYPE31M if cfg.kind != synth.RBF else DTYPE31),
        "data": "synthetic (seeded; SURVEY.md §8d recipe)",
        "config": {"workload": f"{cfg.name}: exact GP MLL+grad, "
                               f"{'RBF' if cfg.kind == 0 else 'Matern-5/2'}"
                               f"{' ARD' if cfg.ard else ''}, n={cfg.n}, d={cfg.d}, t={cfg.t}, "
                               f"k={cfg.k}, p={cfg.p}, "
                               f"{'stored' if kmode == bb.STORED else 'on-the-fly'} K",
                   "parallelism": f"row-partition x{world}",
                   "matmul_precision": args.precision,
                   "kgrid_bits": stats[-1].get("kgrid_bits"),
                   "l2": "256 MB L2 flush between timed steps"},
        "roofline": roofline, "e2e": e2e, "gpu_launches": launches // max(len(stats), 1) * args.steps,
        "clocks": clocks,
        "detail": {k: stats[-1][k] for k in ("ms_pivchol", "ms_mbcg", "ms_matmul", "ms_slq",
                                               "ms_deriv", "ms_comm", "iters", "k_used", "logdet",
                                               "relres_y", "relres_max", "unconverged",
                                               "matmul_path")},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, pr)
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args, cfg, rank, world):
    """Reference arm = the fp64 oracle as it stands, on the host cores, each
    step a bounded row sample of the same workload (rank 0 only)."""
    if rank != 0:
        return
    import oracle
    oracle.build()
    pr = synth.make_problem(cfg, seed=0)
    rows = int(os.environ.get("BBMM_ORACLE_ROWS", "0")) or None
    if rows is None:
        cal = oracle_sample(cfg, pr, 32)
        rows = int(max(32, min(cfg.n, 32 * 8.0 / max(cal["seconds"], 1e-3))))
    for _ in range(args.warmup):
        oracle_sample(cfg, pr, max(1, rows // 8))
    res = [oracle_sample(cfg, pr, rows, seed=s) for s in range(args.steps)]
    g = float(np.mean([r["gflops"] for r in res]))
    sec = float(np.mean([r["seconds"] for r in res]))
    line = {"impl": "reference", "metric": METRIC, "value": g, "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
            "config": {"workload": f"{cfg.name} (oracle row sample)"},
            "cpu_baseline": {"value": g, "unit": "GFLOP/s", "cores": res[0]["cores"],
                             "kind": "oracle",
                             "sample": f"{rows} rows of Khat*D at {cfg.name} per step"},
            "e2e": {"value": g, "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
