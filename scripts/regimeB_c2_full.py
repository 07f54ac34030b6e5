"""Regime-B evidence at the full C2 size (Matern-5/2 ARD, n = 45 730, k = 20, p = 20: the fp64
oracle's relres is ~0.2 at p, i.e. mBCG far from converged).  Runs the oracle once on the host
cores (~minutes) and the GPU operators, printing solve / MLL differences to the oracle.
One JSON line.  python scripts/regimeB_c2_full.py"""
import json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, oracle
import paper_1809_11165_b200 as bb
oracle.build()
cfg = synth.CONFIGS["C2"]
pr = synth.make_problem(cfg, seed=0)
t0 = time.time()
o = oracle.mll_and_grad(cfg.kind, pr.X, pr.y, pr.log_ls, pr.log_s, pr.log_noise, cfg.t, cfg.k, cfg.p, seed=7)
t_or = time.time() - t0
ctx = bb.Context(0)
X = torch.from_numpy(pr.X).cuda(); y = torch.from_numpy(pr.y).cuda()
h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
out = {"config": "C2 full (regime B)", "oracle_s": t_or, "oracle_threads": oracle.num_threads(),
       "oracle_mll": o["mll"], **{k: float(o[k]) for k in oracle.STAT_KEYS}}
for lab, km, pc in [("stored_int8", bb.STORED, bb.INT8EXACT), ("stored_fp32_fp64acc", bb.STORED, bb.FP64ACC),
                    ("onthefly_fp64acc", bb.ONTHEFLY, bb.FP64ACC), ("stored_fp32acc", bb.STORED, bb.FP32ACC)]:
    ctx.set_matmul_precision(pc)
    g = bb.mll_and_grad(ctx, X, y, h, cfg.t, cfg.k, cfg.p, seed=7, kmode=km, return_solves=True)
    U = g["U"].cpu().numpy()
    e = np.linalg.norm(U - o["U"], axis=0) / np.linalg.norm(o["U"], axis=0)
    out[lab] = {"path": g["stats"]["matmul_path"], "relres_y": g["stats"]["relres_y"],
                "solve_err_max": float(e.max()), "solve_err_y": float(e[0]),
                "mll_rel": abs(g["mll"] - o["mll"]) / abs(o["mll"]),
                "grad_rel": float(np.linalg.norm(g["grad"] - o["grad"]) / np.linalg.norm(o["grad"]))}
ctx.set_matmul_precision(bb.INT8EXACT)
print(json.dumps(out))
