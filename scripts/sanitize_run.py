"""Small calls through every kernel family, for compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python scripts/sanitize_run.py

C0 (fused mBCG, CUDA-core operator), C4-shaped n = 3000 (K1-TC, per-step kernels + the captured
graph), C1 stored K (K2-TC), C2-shaped Matern on the fly (K1-TC MODE 2) and its tensor-core
derivative pass, C3-shaped n = 20 000 (K1-TC <33>, the RBF-ARD tensor-core derivative pass),
predictions and the SoR operator (both skinny-product kernels), the 31-bit-grid K1-TC (MODE 3) and
the 23-bit one over more than one uint32 drain window, and K1-TC column chunks.  Prints one line
per call."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_1809_11165_b200 as bb  # noqa: E402

ctx = bb.Context(0)


def run(name, n, kmode=None, env=None, **over):
    cfg = synth.dataclasses.replace(synth.scaled(synth.CONFIGS[name], n), **over)
    pr = synth.make_problem(cfg, seed=0)
    X = torch.from_numpy(pr.X).cuda()
    y = torch.from_numpy(pr.y).cuda()
    h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
    km = kmode if kmode is not None else (bb.STORED if cfg.stored else bb.ONTHEFLY)
    for k, v in (env or {}).items():
        os.environ[k] = v
    try:
        g = bb.mll_and_grad(ctx, X, y, h, cfg.t, cfg.k, cfg.p, seed=7, kmode=km)
    finally:
        for k in (env or {}):
            os.environ.pop(k)
    print(f"{name} n={n} path={g['stats']['matmul_path']} mll={g['mll']:.6f}", flush=True)
    return cfg, pr, X, y, h


run("C0", 256)
run("C4", 3000)                                             # fused K1-TC
run("C4", 3000, env={"BBMM_NO_FUSED_MBCG": "1"})            # per-step kernels, CUDA graph
run("C1", 3338)                                             # stored K2-TC
run("C2", 3000, kmode=bb.ONTHEFLY, env={"BBMM_DERIV_TC_MIN_N": "0"})   # Matern MODE 2 + deriv_tc
run("C3", 20000, p=4)                                       # K1-TC <33>, deriv_tc2
ctx.set_matmul_precision(bb.INT8EXACT31)
run("C4", 30000, p=2, t=16, k=10)                           # K1-TC MODE 3: > 1 drain window
ctx.set_matmul_precision(bb.INT8EXACT)
run("C4", 30000, p=2, t=16, k=10)                           # K1-TC MODE 0: > 1 drain window
run("C4", 1500, t=40, k=10)                                 # column chunks (2 x 33) + MODE-1 chunks
cfg, pr, X, y, h = run("C4", 2000, t=5, k=10)
Xs = torch.from_numpy(synth.test_points(cfg, 20)).cuda()
mean, var = bb.predict(ctx, X, y, Xs, h, k=10, max_iter=10)
print("predict", float(mean[0]), float(var[0]))
Xu = torch.from_numpy(pr.X[:100].copy()).cuda()
B = torch.from_numpy(synth.random_block(cfg.n, 4, seed=1).astype(np.float64)).cuda()
r = bb.sor_mbcg(ctx, X, Xu, h, B, k=5, max_iter=10)
print("sor", float(r["relres"][0]))
Xu2 = torch.from_numpy(pr.X[:200].copy()).cuda()              # m >= 128: the cp.async k_LtR3 path
r = bb.sor_mbcg(ctx, X, Xu2, h, B, k=5, max_iter=10)
print("sor m=200", float(r["relres"][0]))
torch.cuda.synchronize()
ctx.close()
print("sanitize run done")
