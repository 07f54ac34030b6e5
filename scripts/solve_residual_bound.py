#!/usr/bin/env python
"""North-star solve accuracy at n = 1M without an n = 1M oracle run (GPU; evidence script).

For the y column, u = the GPU's K̂⁻¹y after p mBCG iterations, and u* = K̂⁻¹y exactly:
    ||u - u*|| <= ||K̂⁻¹|| ||y - K̂u|| <= ||y - K̂u|| / sigma^2          (lambda_min(K̂) >= sigma^2)
The residual is evaluated with the fp64 oracle's K̂ (oracle.kernel_matmul, reading R1) on m
sampled rows; ||r||^2 is estimated as (n/m) sum_sampled r_i^2.  In regime A the oracle's own
iterate is within relres ~1e-11 of u*, so the bound also bounds the distance to the oracle's
solve.  At n = 131 072 the true distance to the cached oracle solve is known
(tests/golden/large), which calibrates how tight the bound is.

    python scripts/solve_residual_bound.py [n ...]      -> one JSON line per (n, precision)
"""
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_1809_11165_b200 as bb  # noqa: E402
import synth  # noqa: E402

M_ROWS = int(os.environ.get("RESBOUND_ROWS", "512"))


def run(ctx, n, prec, label):
    cfg = synth.scaled(synth.CONFIGS["C4"], n)
    pr = synth.make_problem(cfg, seed=0)
    h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
    ctx.set_matmul_precision(prec)
    try:
        g = bb.mll_and_grad(ctx, torch.from_numpy(pr.X).cuda(), torch.from_numpy(pr.y).cuda(), h, cfg.t,
                            cfg.k, cfg.p, seed=7, return_solves=True)
    finally:
        ctx.set_matmul_precision(bb.INT8EXACT)
    u = g["U"][:, 0].cpu().numpy().astype(np.float64)
    rows = np.sort(np.random.default_rng(11).choice(n, M_ROWS, replace=False))
    Ku = oracle.kernel_matmul(cfg.kind, pr.X, pr.log_ls, pr.log_s, pr.log_noise, u[:, None].copy(),
                              rows=rows)[:, 0]
    r = pr.y.astype(np.float64)[rows] - Ku
    rnorm = math.sqrt(n / M_ROWS * float((r ** 2).sum()))
    sigma2 = math.exp(2 * pr.log_noise)
    rec = dict(n=n, precision=label, sampled_rows=M_ROWS, relres_true_est=rnorm / float(np.linalg.norm(pr.y)),
               solve_bound=rnorm / (sigma2 * float(np.linalg.norm(u))), ms_total=g["stats"]["ms_total"])
    cache = os.path.join(ROOT, "tests", "golden", "large", f"C4_n{n}.npz")
    if os.path.exists(cache):
        z = np.load(cache)
        uo = z["U"][:, 0].astype(np.float64)
        rec["solve_vs_oracle"] = float(np.linalg.norm(u - uo) / z["Unorm"][0])
    return rec


def main():
    ns = [int(a) for a in sys.argv[1:]] or [131072, 1000000]
    ctx = bb.Context(0)
    for n in ns:
        for prec, label in [(bb.INT8EXACT23, "int8exact23"), (bb.INT8EXACT31, "int8exact31"),
                            (bb.FP64ACC, "fp64acc")]:
            if prec == bb.FP64ACC and n > 300000:
                continue                  # ~34 s per K̂·D at n = 1M on CUDA cores
            print(json.dumps(run(ctx, n, prec, label)), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
