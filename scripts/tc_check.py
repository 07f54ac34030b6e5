"""Quick check of the tcgen05 exact kernel-matmul against the oracle + timing."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import synth, oracle
import paper_1809_11165_b200 as bb

ctx = bb.Context(0)
def dev(a, dt=torch.float32): return torch.as_tensor(np.ascontiguousarray(a)).to('cuda', dt)
for name, n, c in [("C4", 200, 17), ("C4", 4099, 17), ("C0", 256, 11), ("C0", 1000, 8), ("C4", 70, 1), ("C4", 3001, 33), ("C4", 20000, 17), ("C1", 3338, 11), ("C4", 5000, 4)]:
    pr = synth.make_problem(synth.scaled(synth.CONFIGS[name], n), seed=3)
    D = synth.random_block(n, c, seed=4).astype(np.float64)
    h = bb.Hyper(pr.cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
    ref = oracle.kernel_matmul(pr.cfg.kind, pr.X, pr.log_ls, pr.log_s, pr.log_noise, D)
    absb = oracle.kernel_matmul(pr.cfg.kind, pr.X, pr.log_ls, pr.log_s, pr.log_noise, np.abs(D))
    for prec in (bb.FP64ACC, bb.INT8EXACT):
        ctx.set_matmul_precision(prec)
        V = bb.kernel_matmul(ctx, dev(pr.X), dev(D, torch.float64), h).cpu().numpy()
        err = np.abs(V - ref)
        print(name, n, c, "prec", prec, "max err/absbound %.3e" % (err / absb).max(),
              "colrel %.3e" % (np.linalg.norm(V - ref, axis=0) / np.linalg.norm(ref, axis=0)).max(), flush=True)
# timing at C4 full size
cfg = synth.CONFIGS["C4"]
pr = synth.make_problem(cfg, seed=0)
D = synth.random_block(cfg.n, 17, seed=4).astype(np.float64)
Xd, Dd = dev(pr.X), dev(D, torch.float64)
h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
for prec in (bb.INT8EXACT, bb.FP64ACC):
    ctx.set_matmul_precision(prec)
    V = bb.kernel_matmul(ctx, Xd, Dd, h)
    torch.cuda.synchronize(); t0 = time.time()
    V = bb.kernel_matmul(ctx, Xd, Dd, h)
    torch.cuda.synchronize(); dt = time.time() - t0
    print("C4 full matmul prec", prec, "%.3f s" % dt, flush=True)
    if prec == bb.INT8EXACT: Vt = V.cpu().numpy()
rows = np.array([0, 1, 12345, 999999])
ref = oracle.kernel_matmul(cfg.kind, pr.X, pr.log_ls, pr.log_s, pr.log_noise, D, rows=rows)
absb = oracle.kernel_matmul(cfg.kind, pr.X, pr.log_ls, pr.log_s, pr.log_noise, np.abs(D), rows=rows)
print("C4 full sampled rows err/absbound %.3e" % (np.abs(Vt[rows] - ref) / absb).max())
