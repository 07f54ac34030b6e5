"""Run the kernel-matmul a few times (for ncu):
python scripts/prof_matmul.py [n] [prec] [config] [stored]"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import synth
import paper_1809_11165_b200 as bb
n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
prec = int(sys.argv[2]) if len(sys.argv) > 2 else bb.INT8EXACT
name = sys.argv[3] if len(sys.argv) > 3 else "C4"
kmode = bb.STORED if len(sys.argv) > 4 and sys.argv[4] == "stored" else bb.ONTHEFLY
cfg = synth.scaled(synth.CONFIGS[name], n)
pr = synth.make_problem(cfg, seed=0)
c = cfg.t + 1
D = synth.random_block(n, c, seed=4).astype(np.float64)
ctx = bb.Context(0).set_matmul_precision(prec)
X = torch.from_numpy(pr.X).cuda(); Dd = torch.from_numpy(D).cuda()
h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
for _ in range(3):
    V = bb.kernel_matmul(ctx, X, Dd, h, kmode)
torch.cuda.synchronize()
print("done", float(V[0, 0]))
