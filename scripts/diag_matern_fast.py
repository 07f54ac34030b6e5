"""Gradient / solve error vs the oracle of the on-the-fly Matern tensor-core path (K1-TC MODE 2)
against FP64ACC and the stored path at the C2 shape (small n).  python scripts/diag_matern_fast.py"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, oracle
import paper_1809_11165_b200 as bb
oracle.build()
ctx = bb.Context(0)
for n in (2048, 2500, 3000):
    cfg = synth.scaled(synth.CONFIGS["C2"], n)
    pr = synth.make_problem(cfg, seed=0)
    X = torch.from_numpy(pr.X).cuda(); y = torch.from_numpy(pr.y).cuda()
    h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
    o = oracle.mll_and_grad(cfg.kind, pr.X, pr.y, pr.log_ls, pr.log_s, pr.log_noise, cfg.t, cfg.k, cfg.p, seed=7)
    for lab, km, pc in [("tc_otf", bb.ONTHEFLY, bb.INT8EXACT), ("fp64acc_otf", bb.ONTHEFLY, bb.FP64ACC),
                        ("int8_stored", bb.STORED, bb.INT8EXACT)]:
        ctx.set_matmul_precision(pc)
        g = bb.mll_and_grad(ctx, X, y, h, cfg.t, cfg.k, cfg.p, seed=7, kmode=km, return_solves=True)
        U = g["U"].cpu().numpy()
        es = (np.linalg.norm(U - o["U"], axis=0) / np.linalg.norm(o["U"], axis=0)).max()
        eg = np.linalg.norm(g["grad"] - o["grad"]) / np.linalg.norm(o["grad"])
        print(f"n={n} {lab:12s} path {g['stats']['matmul_path']} solve {es:.2e} grad {eg:.2e} mll {abs(g['mll']-o['mll'])/abs(o['mll']):.1e}")
    ctx.set_matmul_precision(bb.INT8EXACT)
