"""Measure row f4 (SoR / SGPR operator through mBCG) at the C4 shape on one B200; one JSON line.

bbmm_sor_mbcg on [y | 16 Rademacher columns], m inducing points, rank-k pivoted Cholesky of
K_SoR, p iterations (tol 0).  Timed with CUDA events, inputs resident.  The per-iteration
matmul is HBM-bound: algorithmic bytes per K_SoR D = 2 * 8 m n (Bs read for T = Bs D and for
V = Bs^T T) + 2 * 8 n c (D read, V written); the roofline fraction divides the bytes of p
matmuls by the per-iteration time of an UNPRECONDITIONED run (k = 0) measured as the difference
of 20 and 10 iterations (setup cancels; k = 0 keeps the run far from convergence, so the
per-iteration cost is representative) against MEASURED_PEAKS.json hbm_gbs.
usage: python scripts/bench_sor.py [n] [m] [k] [p]"""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_1809_11165_b200 as bb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 300
k = int(sys.argv[3]) if len(sys.argv) > 3 else 100
p = int(sys.argv[4]) if len(sys.argv) > 4 else 40
cfg = synth.scaled(synth.CONFIGS["C4"], n)
pr = synth.make_problem(cfg, seed=0)
Xu = synth.test_points(cfg, m, seed=13)
rng = np.random.default_rng(11)
B = np.concatenate([pr.y.astype(np.float64)[:, None], rng.choice([-1.0, 1.0], size=(n, cfg.t))], 1)
ctx = bb.Context(0)
X, Xud, Bd = (torch.from_numpy(a).cuda() for a in (pr.X, Xu, B))
h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)


def run(iters, kk=k):
    bb.sor_mbcg(ctx, X, Xud, h, Bd, k=kk, max_iter=iters)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    r = bb.sor_mbcg(ctx, X, Xud, h, Bd, k=kk, max_iter=iters)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), r


ms_p, r = run(p)
ms20, r0 = run(20, 0)
ms10, _ = run(10, 0)
c = B.shape[1]
print("raw ms: k=%d p=%d %.1f | k=0 p=20 %.1f | k=0 p=10 %.1f" % (k, p, ms_p, ms20, ms10), file=sys.stderr)
per_iter_ms = (ms20 - ms10) / 10
bytes_mm = 2 * 8 * m * n + 2 * 8 * n * c
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
print(json.dumps({"metric": "SoR mBCG (row f4) at C4 shape", "n": n, "m": m, "k": k, "p": p, "c": c,
                  "ms_total": ms_p, "ms_per_iteration": per_iter_ms,
                  "relres_y_final": float(r["relres"][0]),
                  "k0_relres_y_at_20": float(r0["relres"][0]),
                  "roofline": {"bound": "hbm", "unit": "GB/s",
                               "achieved_matmul_only_lower_bound": bytes_mm / (per_iter_ms * 1e-3) / 1e9,
                               "peak": peak, "note": "per-iteration time includes the CG vector "
                               "passes and Woodbury (k x n L reads), so this is a lower bound for "
                               "the matmul's bandwidth"}}))
