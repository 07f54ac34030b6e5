import sys, numpy as np, torch
sys.path.insert(0, '.')
import synth, oracle
import paper_1809_11165_b200 as bb
cfg = synth.scaled(synth.CONFIGS["C4"], 1001)
pr = synth.make_problem(cfg, seed=0)
ctx = bb.Context(0)
X = torch.from_numpy(pr.X).cuda(); y = torch.from_numpy(pr.y).cuda()
h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
o = oracle.mll_and_grad(cfg.kind, pr.X, pr.y, pr.log_ls, pr.log_s, pr.log_noise, cfg.t, cfg.k, cfg.p, seed=7)
print("oracle", o["grad"])
for prec in (bb.FP64ACC, bb.INT8EXACT):
    ctx.set_matmul_precision(prec)
    g = bb.mll_and_grad(ctx, X, y, h, cfg.t, cfg.k, cfg.p, seed=7)
    print(prec, g["grad"], g["stats"]["matmul_path"])
