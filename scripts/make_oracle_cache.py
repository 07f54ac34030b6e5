#!/usr/bin/env python
"""Write the fp64 oracle's MLL + gradient at large n to tests/golden/large/ (test fixtures).

Calls ONLY oracle/ and synth/ (never the CUDA path): the stored values are the oracle's, on the
seeded synth inputs the GPU parity test rebuilds, keyed by a SHA-256 of X and y so a change of
the input recipe is detected instead of silently compared against stale values.

One case = one bbmm_mll_and_grad-equivalent call (pivoted Cholesky -> probes -> mBCG -> SLQ ->
derivative pass, §4 and Eq. 2) at the config's t, k, p with
probe seed 7 (the parity tests' seed), plus one extra oracle K̂·u₀ for the y column's relative
residual ||y - K̂u₀|| / ||y|| at p (regime A vs B), stated rather than assumed.

U is stored as fp32 (relative rounding 6e-8, far below the 1e-4 solve bar).

    python scripts/make_oracle_cache.py C4:131072 C3:80000 C2:45730
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "large")
SEED_X, SEED_PROBES = 0, 7


def input_hash(pr) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(pr.X).tobytes())
    h.update(np.ascontiguousarray(pr.y).tobytes())
    h.update(np.asarray(pr.log_ls, np.float64).tobytes())
    h.update(np.asarray([pr.log_s, pr.log_noise], np.float64).tobytes())
    return h.hexdigest()


def case_path(name: str, n: int) -> str:
    return os.path.join(OUT, f"{name}_n{n}.npz")


def make(name: str, n: int) -> str:
    cfg = synth.scaled(synth.CONFIGS[name], n)
    pr = synth.make_problem(cfg, seed=SEED_X)
    t0 = time.time()
    o = oracle.mll_and_grad(cfg.kind, pr.X, pr.y, pr.log_ls, pr.log_s, pr.log_noise, cfg.t,
                            cfg.k, cfg.p, seed=SEED_PROBES)
    t_mll = time.time() - t0
    Ku0 = oracle.kernel_matmul(cfg.kind, pr.X, pr.log_ls, pr.log_s, pr.log_noise,
                               o["U"][:, :1].copy())
    y64 = pr.y.astype(np.float64)
    relres_y = float(np.linalg.norm(y64 - Ku0[:, 0]) / np.linalg.norm(y64))
    meta = dict(name=name, n=n, d=cfg.d, t=cfg.t, k=cfg.k, p=cfg.p, kind=cfg.kind,
                seed_x=SEED_X, seed_probes=SEED_PROBES, input_sha256=input_hash(pr),
                oracle_s=round(t_mll, 1), oracle_threads=oracle.num_threads(),
                relres_y=relres_y, regime="A" if relres_y < 1e-3 else "B",
                script="scripts/make_oracle_cache.py")
    os.makedirs(OUT, exist_ok=True)
    path = case_path(name, n)
    np.savez_compressed(
        path, meta=json.dumps(meta), mll=o["mll"], grad=o["grad"], U=o["U"].astype(np.float32),
        Unorm=np.linalg.norm(o["U"], axis=0), pivots=o["pivots"], alpha=o["alpha"],
        beta=o["beta"], iters_col=o["iters"],
        **{k: o[k] for k in oracle.STAT_KEYS})
    print(json.dumps(meta), flush=True)
    return path


if __name__ == "__main__":
    for arg in sys.argv[1:]:
        nm, nn = arg.split(":")
        make(nm, int(nn))
