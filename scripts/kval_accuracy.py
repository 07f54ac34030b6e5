#!/usr/bin/env python
"""Per-entry accuracy of the kernel values each matmul operator uses (diagnostic, GPU).

With D = [e_j1 .. e_jm] (unit columns) one kernel-matmul returns V = s K[:, j] + sigma^2 e_j
exactly up to the operator's kernel-value rounding (a single nonzero per column: the contraction
adds nothing), so the columns expose the kernel values the operator computed.  They are compared
with the fp64 kernel (reading R1, numpy on the host) over all n rows.

    python scripts/kval_accuracy.py [C4] [m]
Prints one JSON line per operator: RMS / max of (k_gpu - k) relative to s, and of the relative
error where k > 1e-3 s.
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
if os.environ.get("KVAL_LIB"):   # a scratch build (scripts/k1_experiments) instead of the tree's
    sys.path.insert(0, os.environ["KVAL_LIB"])
import paper_1809_11165_b200 as bb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 16
cfg = synth.CONFIGS[name]
pr = synth.make_problem(cfg, seed=0)
n = cfg.n
cols = np.random.default_rng(5).choice(n, m, replace=False)
D = np.zeros((n, m))
D[cols, np.arange(m)] = 1.0
ls = np.exp(pr.log_ls)
Xs = pr.X.astype(np.float64) / (ls if ls.size > 1 else ls[0])
s = float(np.exp(pr.log_s))
noise = float(np.exp(2 * pr.log_noise))
Kref = np.empty((n, m))
for c, j in enumerate(cols):
    r2 = ((Xs - Xs[j]) ** 2).sum(1)
    if cfg.kind == synth.RBF:
        Kref[:, c] = s * np.exp(-0.5 * r2)
    else:
        r = np.sqrt(5.0 * r2)
        Kref[:, c] = s * (1 + r + r * r / 3.0) * np.exp(-r)
ctx = bb.Context(0)
X = torch.from_numpy(pr.X).cuda()
Dd = torch.from_numpy(D).cuda()
h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
for label, prec, km in [("int8exact", bb.INT8EXACT, bb.ONTHEFLY), ("int8exact31", bb.INT8EXACT31, bb.ONTHEFLY),
                        ("fp64acc", bb.FP64ACC, bb.ONTHEFLY)]:
    ctx.set_matmul_precision(prec)
    V = bb.kernel_matmul(ctx, X, Dd, h, km).cpu().numpy()
    V[cols, np.arange(m)] -= noise
    err = V - Kref
    big = Kref > 1e-3 * s
    rel = np.abs(err[big]) / Kref[big]
    print(json.dumps(dict(config=name, operator=label, m=m, abs_rms=float(np.sqrt((err ** 2).mean()) / s),
                          abs_max=float(np.abs(err).max() / s), rel_rms=float(np.sqrt((rel ** 2).mean())),
                          rel_max=float(rel.max()), mean_err=float(err.mean() / s))))
