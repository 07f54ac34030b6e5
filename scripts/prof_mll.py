"""One MLL+grad at a BASELINE config (for ncu captures of its kernels):
python scripts/prof_mll.py [config] [n]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_1809_11165_b200 as bb
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg = synth.CONFIGS[name]
if len(sys.argv) > 2:
    cfg = synth.scaled(cfg, int(sys.argv[2]))
pr = synth.make_problem(cfg, seed=0)
ctx = bb.Context(0)
g = bb.mll_and_grad(ctx, torch.from_numpy(pr.X).cuda(), torch.from_numpy(pr.y).cuda(),
                    bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise), cfg.t, cfg.k, cfg.p,
                    kmode=bb.STORED if cfg.stored else bb.ONTHEFLY)
print("mll", g["mll"], g["stats"]["ms_deriv"])
