import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch, synth
import paper_1809_11165_b200 as bb
cfg = synth.scaled(synth.CONFIGS["C2"], 1200)
pr = synth.make_problem(cfg, seed=1)
B = synth.random_block(1200, 17, seed=5).astype(np.float64)
ctx = bb.Context(0)
h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
X = torch.from_numpy(pr.X).cuda(); Bd = torch.from_numpy(B).cuda()
res = {}
for prec in [bb.FP64ACC, bb.INT8EXACT]:
    for fused in [0, 1]:
        if fused: os.environ.pop("BBMM_NO_FUSED_MBCG", None)
        else: os.environ["BBMM_NO_FUSED_MBCG"] = "1"
        ctx.set_matmul_precision(prec)
        r = bb.mbcg(ctx, X, h, Bd, L=None, max_iter=20)
        res[(prec, fused)] = r
for prec in [bb.FP64ACC, bb.INT8EXACT]:
    a0, a1 = res[(prec,0)]["alpha"], res[(prec,1)]["alpha"]
    rel = np.abs(a0 - a1).max(1) / np.abs(a0).max(1)
    print("prec", prec, "alpha rel diff per iter", np.array2string(rel, precision=1))
    print("  relres", res[(prec,0)]["relres"].max(), res[(prec,1)]["relres"].max())
