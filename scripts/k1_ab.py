#!/usr/bin/env python
"""A/B timing of K1-TC builds at a BASELINE shape (one subprocess per build).

    python scripts/k1_ab.py [--config C4] [--n N] [--reps 5] [--precision 2] LIBROOT ...

LIBROOT = a directory holding paper_1809_11165_b200/ (the repo itself: ".", a variant:
scratch/var_NAME).  Each build runs the kernel-matmul V = Khat D (INT8EXACT) once to warm up, then
`reps` times timed with CUDA events on the library stream; prints the median ms per launch, the
Gpairs/s and the largest deviation of its V from the first build's on 4096 sampled rows.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, os, sys, numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {lib!r})
import synth, paper_1809_11165_b200 as bb
assert os.path.abspath(bb.__file__).startswith(os.path.abspath({lib!r})), bb.__file__
cfg = synth.scaled(synth.CONFIGS[{cfg!r}], {n})
pr = synth.make_problem(cfg, seed=0)
D = synth.random_block(cfg.n, cfg.t + 1, seed=4).astype(np.float64)
ctx = bb.Context(0)
X = torch.from_numpy(pr.X).cuda(); Dd = torch.from_numpy(D).cuda()
h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
ctx.set_matmul_precision({prec})
V = bb.kernel_matmul(ctx, X, Dd, h)
ms = []
for _ in range({reps}):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); V = bb.kernel_matmul(ctx, X, Dd, h); e1.record(); torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
rows = np.random.default_rng(0).integers(0, cfg.n, 4096)
np.save({out!r}, V.cpu().numpy()[rows])
print(json.dumps(dict(ms=sorted(ms)[len(ms) // 2], all=ms, n=cfg.n)))
"""


def main():
    args = sys.argv[1:]
    cfg, n, reps, prec = "C4", None, 5, 2
    while args and args[0].startswith("--"):
        k, v = args[0], args[1]
        args = args[2:]
        if k == "--config":
            cfg = v
        elif k == "--n":
            n = int(v)
        elif k == "--reps":
            reps = int(v)
        elif k == "--precision":      # 2 = INT8EXACT, 3 = INT8EXACT31, 0 = FP64ACC
            prec = int(v)
    sys.path.insert(0, ROOT)
    import numpy as np
    import synth
    n = n or synth.CONFIGS[cfg].n
    ref = None
    for i, lib in enumerate(args):
        lib = os.path.abspath(lib)
        out = f"/tmp/k1ab_{i}.npy"
        code = CHILD.format(root=ROOT, lib=lib, cfg=cfg, n=n, reps=reps, out=out, prec=prec)
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
        if r.returncode != 0:
            print(json.dumps(dict(lib=lib, error=r.stderr[-800:])))
            continue
        res = json.loads(r.stdout.strip().splitlines()[-1])
        V = np.load(out)
        if ref is None:
            ref = V
        dev = float(np.abs(V - ref).max() / max(np.abs(ref).max(), 1e-300))
        pairs = float(n) * n
        print(json.dumps(dict(lib=os.path.relpath(lib, ROOT), config=cfg, n=n, ms=round(res["ms"], 3),
                              all=[round(x, 3) for x in res["all"]],
                              gpairs_s=round(pairs / (res["ms"] * 1e-3) / 1e9, 1),
                              max_rel_dev_vs_first=dev)), flush=True)


if __name__ == "__main__":
    main()
