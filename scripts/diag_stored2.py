"""Diagnostic: solve error vs the fp64 oracle for the operators / precisions at a small n."""
import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, oracle
import paper_1809_11165_b200 as bb
oracle.build()
ctx = bb.Context(0)
for name, n, p in [("C2", 3000, 20), ("C2", 3000, 40), ("C4", 3000, 20), ("C1", 3338, 20), ("C2", 3000, 8)]:
    cfg = synth.dataclasses.replace(synth.scaled(synth.CONFIGS[name], n), p=p)
    pr = synth.make_problem(cfg, seed=0)
    X = torch.from_numpy(pr.X).cuda(); y = torch.from_numpy(pr.y).cuda()
    h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
    o = oracle.mll_and_grad(cfg.kind, pr.X, pr.y, pr.log_ls, pr.log_s, pr.log_noise, cfg.t, cfg.k, cfg.p, seed=7)
    for lab, km, pc in [("int8_stored", bb.STORED, bb.INT8EXACT), ("int8_otf", bb.ONTHEFLY, bb.INT8EXACT),
                        ("fp64acc_stored", bb.STORED, bb.FP64ACC), ("fp32acc_stored", bb.STORED, bb.FP32ACC)]:
        ctx.set_matmul_precision(pc)
        g = bb.mll_and_grad(ctx, X, y, h, cfg.t, cfg.k, cfg.p, seed=7, kmode=km, return_solves=True)
        U = g["U"].cpu().numpy()
        e = np.linalg.norm(U - o["U"], axis=0) / np.linalg.norm(o["U"], axis=0)
        print(f"{name} n={n} p={p} {lab:15s} path {g['stats']['matmul_path']} relres_y {g['stats']['relres_y']:.2e} "
              f"solve err max {e.max():.2e} y {e[0]:.2e} mll rel {abs(g['mll']-o['mll'])/abs(o['mll']):.1e}")
    ctx.set_matmul_precision(bb.INT8EXACT)
