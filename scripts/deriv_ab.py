"""A/B of the derivative pass at a BASELINE shape: ms_deriv of bbmm_mll_and_grad for each build
(one subprocess per LIBROOT, like k1_ab.py).   python scripts/deriv_ab.py [--config C4] LIBROOT ..."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import json, sys, numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {lib!r})
import synth, paper_1809_11165_b200 as bb
cfg = synth.CONFIGS[{cfg!r}]; pr = synth.make_problem(cfg, seed=0)
ctx = bb.Context(0); X = torch.from_numpy(pr.X).cuda(); y = torch.from_numpy(pr.y).cuda()
h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
r = []
for _ in range(3):
    g = bb.mll_and_grad(ctx, X, y, h, cfg.t, cfg.k, cfg.p, seed=7)
    r.append((g["stats"]["ms_deriv"], g["stats"]["ms_total"], g["mll"], list(g["grad"])))
print(json.dumps(r))
"""
args = sys.argv[1:]
cfg = "C4"
if args and args[0] == "--config":
    cfg, args = args[1], args[2:]
for lib in args:
    lib = os.path.abspath(lib)
    out = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT, lib=lib, cfg=cfg)], capture_output=True, text=True)
    if out.returncode:
        print(json.dumps(dict(lib=lib, error=out.stderr[-600:]))); continue
    r = json.loads(out.stdout.strip().splitlines()[-1])
    print(json.dumps(dict(lib=os.path.relpath(lib, ROOT), ms_deriv=[round(x[0], 2) for x in r],
                          ms_total=[round(x[1], 1) for x in r], mll=r[-1][2], grad=r[-1][3])), flush=True)
