"""Diagnostic: stored int8 K (k2tc) vs fp32 paths at the C2 shape: matmul element errors and
MLL / relres differences.  python scripts/diag_stored.py [n]"""
import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_1809_11165_b200 as bb
n = int(sys.argv[1]) if len(sys.argv) > 1 else 45730
cfg = synth.scaled(synth.CONFIGS["C2"], n)
pr = synth.make_problem(cfg, seed=0)
ctx = bb.Context(0)
X = torch.from_numpy(pr.X).cuda(); y = torch.from_numpy(pr.y).cuda()
h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
D = torch.from_numpy(synth.random_block(n, 17, seed=4).astype(np.float64)).cuda()
Va = bb.kernel_matmul(ctx, X, D, h, bb.STORED)
ctx.set_matmul_precision(bb.FP64ACC)
Vb = bb.kernel_matmul(ctx, X, D, h, bb.ONTHEFLY)
Vc = bb.kernel_matmul(ctx, X, D, h, bb.STORED)
Vab = bb.kernel_matmul(ctx, X, D.abs(), h, bb.ONTHEFLY)
ctx.set_matmul_precision(bb.INT8EXACT)
e1 = ((Va - Vb).abs() / Vab).max().item(); e2 = ((Vc - Vb).abs() / Vab).max().item()
print(f"n={n} matmul max |int8 stored - fp64acc otf| / (K|D|) = {e1:.3e};  fp32 stored vs otf {e2:.3e}")
print("  rel norm int8:", ((Va - Vb).norm(dim=0) / Vb.norm(dim=0)).max().item(),
      " fp32:", ((Vc - Vb).norm(dim=0) / Vb.norm(dim=0)).max().item())
res = {}
for lab, km, pc in [("int8_stored", bb.STORED, bb.INT8EXACT), ("fp64acc_otf", bb.ONTHEFLY, bb.FP64ACC),
                    ("fp64acc_stored", bb.STORED, bb.FP64ACC)]:
    ctx.set_matmul_precision(pc)
    g = bb.mll_and_grad(ctx, X, y, h, cfg.t, cfg.k, cfg.p, seed=7, kmode=km, return_solves=True)
    res[lab] = g
    st = g["stats"]
    print(f"{lab}: path {st['matmul_path']} mll {g['mll']:.6f} logdet {st['logdet']:.6f} quad {st['quad_y']:.6f} relres_y {st['relres_y']:.3e} grad {g['grad']}")
ctx.set_matmul_precision(bb.INT8EXACT)
Ua = res["int8_stored"]["U"]; Ub = res["fp64acc_otf"]["U"]
print("solve rel diff per col:", ((Ua - Ub).norm(dim=0) / Ub.norm(dim=0)).cpu().numpy())
