"""Measure row f1 (bbmm_predict) at the C4 shape on one B200 and print one JSON line.

Workloads (inputs resident on the device, CUDA events around each call, 1 warm-up):
  * var16  : mean + variance of 16 test points = one batched mBCG call on
             [y | k_{X x*_1..16}] (p = 20 Khat*D products) + the cross-kernel columns;
  * mean1k : mean only of 1000 test points = one solve of y + 1000 cross-kernel columns.
The oracle's predict is timed beside it on a scaled-down problem (n_small rows, same
d, t, k, p) and extrapolated by the n^2 cost of its Khat*D passes.
usage: python scripts/bench_predict.py [n] [n_small]"""
import json, math, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_1809_11165_b200 as bb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
n_small = int(sys.argv[2]) if len(sys.argv) > 2 else 4000
cfg = synth.scaled(synth.CONFIGS["C4"], n)
pr = synth.make_problem(cfg, seed=0)
ctx = bb.Context(0)
X, y = torch.from_numpy(pr.X).cuda(), torch.from_numpy(pr.y).cuda()
h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)


def timed(ns, variance):
    Xs = torch.from_numpy(synth.test_points(cfg, ns, seed=9)).cuda()
    bb.predict(ctx, X, y, Xs, h, cfg.k, max_iter=cfg.p, variance=variance)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(torch.cuda.current_stream())
    m, v = bb.predict(ctx, X, y, Xs, h, cfg.k, max_iter=cfg.p, variance=variance)
    e1.record(torch.cuda.current_stream())
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


ms_var16 = timed(16, True)
ms_mean1k = timed(1000, False)
# oracle beside it (scaled problem, extrapolated by the n^2 matmul cost)
import oracle as orc_mod
cs = synth.scaled(synth.CONFIGS["C4"], n_small)
ps = synth.make_problem(cs, seed=0)
Xs_small = synth.test_points(cs, 16, seed=9)
t0 = time.perf_counter()
orc_mod.predict(cs.kind, ps.X, ps.y, Xs_small, ps.log_ls, ps.log_s, ps.log_noise, cs.k, cs.p)
t_orc = time.perf_counter() - t0
out = {"metric": "predict (row f1): ms per call at C4", "n": n, "d": cfg.d, "k": cfg.k, "p": cfg.p,
       "var16_ms": ms_var16, "mean1000_ms": ms_mean1k,
       "var16_pairs_per_s": (cfg.p + 1) * n * n / (ms_var16 * 1e-3),
       "oracle": {"n": n_small, "var16_s": t_orc, "cores": orc_mod.num_threads(),
                  "extrapolated_var16_s_at_n": t_orc * (n / n_small) ** 2}}
print(json.dumps(out))
