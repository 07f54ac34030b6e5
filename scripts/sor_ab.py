"""A/B of the SoR mBCG per-iteration time (row f4) across builds, one subprocess per LIBROOT
(like k1_ab.py): n = 1M, m = 300, k = 0, (p = 20) - (p = 10) iterations, CUDA events.
    python scripts/sor_ab.py LIBROOT ..."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import json, sys, numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {lib!r})
import synth, paper_1809_11165_b200 as bb
cfg = synth.scaled(synth.CONFIGS["C4"], 1000000); pr = synth.make_problem(cfg, seed=0)
Xu = synth.test_points(cfg, 300, seed=13)
B = np.concatenate([pr.y.astype(np.float64)[:, None], np.random.default_rng(11).choice([-1.0, 1.0], size=(cfg.n, 16))], 1)
ctx = bb.Context(0); X, Xud, Bd = (torch.from_numpy(a).cuda() for a in (pr.X, Xu, B))
h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
def run(p):
    bb.sor_mbcg(ctx, X, Xud, h, Bd, k=0, max_iter=p)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(); r = bb.sor_mbcg(ctx, X, Xud, h, Bd, k=0, max_iter=p); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1), r
t20, r = run(20); t10, _ = run(10)
print(json.dumps(dict(ms_per_iter=(t20 - t10) / 10, relres0=float(r["relres"][0]))))
"""
for lib in sys.argv[1:]:
    lib = os.path.abspath(lib)
    out = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT, lib=lib)], capture_output=True, text=True)
    if out.returncode:
        print(json.dumps(dict(lib=lib, error=out.stderr[-500:]))); continue
    r = json.loads(out.stdout.strip().splitlines()[-1])
    print(json.dumps(dict(lib=os.path.relpath(lib, ROOT), **r)), flush=True)
