"""Time the C4 full-size kernel-matmul (INT8EXACT) -- variants via env vars."""
import sys, os, time, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, os.environ.get('BBMM_VARIANT', '.'))
import synth
import paper_1809_11165_b200 as bb
cfg = synth.CONFIGS["C4"]
pr = synth.make_problem(cfg, seed=0)
D = synth.random_block(cfg.n, 17, seed=4).astype(np.float64)
ctx = bb.Context(0).set_matmul_precision(bb.INT8EXACT)
Xd = torch.from_numpy(pr.X).cuda(); Dd = torch.from_numpy(D).cuda()
h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
V = bb.kernel_matmul(ctx, Xd, Dd, h)
ts = []
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.time()
    V = bb.kernel_matmul(ctx, Xd, Dd, h)
    torch.cuda.synchronize(); ts.append(time.time() - t0)
print("NQ", os.environ.get("BBMM_TC2_NQ", "4"), "C4 matmul s", ["%.3f" % x for x in ts], float(V[0, 0]))
