#!/usr/bin/env python
"""Rounding-sensitivity floor of the fp64 oracle's mBCG solves (regime B evidence).

Calls ONLY oracle/ and synth/.  For one config-shaped case it forms the oracle's own right-hand
side B = [y | z_1..z_t] (pivoted Cholesky, probes z = L eps1 + sigma eps2 with the parity tests'
seed 7; Eq. 3, reading R13) and runs the oracle's mBCG (Alg. S2)
twice: on B, and on B with every entry moved by one unit in the last place (B (1 + 2^-52 r),
r = +-1 at random).  Both runs are the same fp64 program; they differ by one rounding of the
input.  The column-wise relative difference of the two solves is how far ANY fp64 implementation
of the method -- one that merely sums in another order -- can land from the oracle on this
problem.  Where mBCG has converged by p (regime A) it is ~1e-13; where it has not (regime B) the
unconverged Krylov iterate amplifies it by many orders of magnitude.

Writes tests/golden/large/<name>_n<n>_floor.json.
    python scripts/oracle_rounding_floor.py C2:45730
"""
from __future__ import annotations

import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "large")


def colrel(a, b):
    return np.linalg.norm(a - b, axis=0) / np.linalg.norm(b, axis=0)


def floor(name: str, n: int, seed_probes: int = 7) -> dict:
    cfg = synth.scaled(synth.CONFIGS[name], n)
    pr = synth.make_problem(cfg, seed=0)
    t0 = time.time()
    L, piv, ku, _ = oracle.pivchol_kernel(cfg.kind, pr.X, pr.log_ls, pr.log_s, cfg.k)
    eps = oracle.rademacher(seed_probes, n, cfg.k, cfg.t)
    Z = oracle.probes(eps, L[:, :ku], math.exp(pr.log_noise))
    B = np.concatenate([pr.y.astype(np.float64)[:, None], Z], axis=1)
    r = np.random.default_rng(11).choice([-1.0, 1.0], size=B.shape)
    B1 = B * (1.0 + 2.0**-52 * r)
    args = (cfg.kind, pr.X, pr.log_ls, pr.log_s, pr.log_noise)
    o0 = oracle.mbcg_kernel(*args, B, cfg.p, L=L[:, :ku])
    o1 = oracle.mbcg_kernel(*args, B1, cfg.p, L=L[:, :ku])
    d = colrel(o1["U"], o0["U"])
    res = dict(name=name, n=n, p=cfg.p, k=cfg.k, t=cfg.t, seed_probes=seed_probes,
               perturbation="B * (1 + 2^-52 r), r = +-1 (numpy seed 11)",
               relres_y=float(o0["relres"][0]), solve_floor_max=float(d.max()),
               solve_floor_y=float(d[0]), solve_floor_cols=[float(v) for v in d],
               seconds=round(time.time() - t0, 1), threads=oracle.num_threads(),
               script="scripts/oracle_rounding_floor.py")
    cache = os.path.join(OUT, f"{name}_n{n}.npz")
    if os.path.exists(cache):   # consistency with the cached one-call oracle (same arithmetic)
        res["vs_cached_mll_and_grad"] = float(colrel(o0["U"], np.load(cache)["U"]).max())
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, f"{name}_n{n}_floor.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res), flush=True)
    return res


if __name__ == "__main__":
    for arg in sys.argv[1:]:
        nm, nn = arg.split(":")
        floor(nm, int(nn))
