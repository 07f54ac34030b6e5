"""Row f3: preconditioner-rank study (the paper's Fig. 3 analog).

For k in {0, 2, 5, 9, 20, 100}: rank-k pivoted Cholesky (bbmm_pivchol) and one mBCG call
(bbmm_mbcg, tol = 0) on [y | z_1..z_t] at the C4 shape; records ||r_j|| / ||b|| after every
iteration for the y column and the mean over the probe columns, plus the time per call.
At a small n (dense on the host) it also reports kappa(Khat) and kappa(Phat^{-1} Khat).
Prints one JSON document. usage: python scripts/precond_study.py [n] [max_iter] [n_small]"""
import json, math, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_1809_11165_b200 as bb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
p = int(sys.argv[2]) if len(sys.argv) > 2 else 40
n_small = int(sys.argv[3]) if len(sys.argv) > 3 else 2000
KS = [0, 2, 5, 9, 20, 100]
cfg = synth.scaled(synth.CONFIGS["C4"], n)
pr = synth.make_problem(cfg, seed=0)
ctx = bb.Context(0)
X = torch.from_numpy(pr.X).cuda()
h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
rng = np.random.default_rng(11)
B = np.concatenate([pr.y.astype(np.float64)[:, None],
                    rng.choice([-1.0, 1.0], size=(n, cfg.t))], axis=1)
Bd = torch.from_numpy(B).cuda()
out = {"config": f"C4 shape n={n}, d={cfg.d}, t={cfg.t}, p={p}, RBF, theta of synth C4",
       "note": "probe columns here are plain Rademacher (same B for every k)", "runs": []}
for k in KS:
    L = bb.pivchol(ctx, X, h, k)[0] if k > 0 else None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    r = bb.mbcg(ctx, X, h, Bd, L=L, max_iter=p)
    e1.record()
    torch.cuda.synchronize()
    rh = r["relres_hist"]
    out["runs"].append({"k": k, "ms": e0.elapsed_time(e1),
                        "relres_y": rh[:, 0].tolist(),
                        "relres_probe_mean": rh[:, 1:].mean(1).tolist()})
    print(f"k={k:3d}  relres_y@5={rh[4, 0]:.3e} @10={rh[9, 0]:.3e} @20={rh[19, 0]:.3e} "
          f"@{p}={rh[p - 1, 0]:.3e}", file=sys.stderr)
# small-n condition numbers (dense, host): kappa(Khat), kappa(Phat^-1 Khat) for each k
cs = synth.scaled(synth.CONFIGS["C4"], n_small)
ps = synth.make_problem(cs, seed=0)
Xs = ps.X.astype(np.float64)
ls = math.exp(ps.log_ls[0])
D2 = ((Xs[:, None, :] - Xs[None, :, :]) ** 2).sum(-1) / ls**2
s2 = math.exp(2 * ps.log_noise)
Kh = math.exp(ps.log_s) * np.exp(-0.5 * D2) + s2 * np.eye(n_small)
hs = bb.Hyper(cs.kind, ps.log_ls, ps.log_s, ps.log_noise)
kap = []
for k in KS:
    if k == 0:
        ev = np.linalg.eigvalsh(Kh)
    else:
        L = bb.pivchol(ctx, torch.from_numpy(ps.X).cuda(), hs, k)[0].cpu().numpy().T   # n x k
        P = L @ L.T + s2 * np.eye(n_small)
        w, Q = np.linalg.eigh(P)
        Pih = (Q / np.sqrt(w)) @ Q.T
        ev = np.linalg.eigvalsh(Pih @ Kh @ Pih)
    kap.append({"k": k, "kappa": float(ev[-1] / ev[0])})
out["condition_small_n"] = {"n": n_small, "values": kap}
print(json.dumps(out))
