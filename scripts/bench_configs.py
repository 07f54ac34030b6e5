"""One full bbmm_mll_and_grad per BASELINE config (C0..C4) at its full size on one B200.

Per config: the default operator of the config (C1/C2 stored K, else on the fly) under the default
precision (INT8EXACT: tcgen05 paths where they apply), one warm-up call, then the median of
`reps` timed calls (the library's CUDA events; inputs resident).  Reports ms per MLL+grad, the
K-hat*D time per launch, the matmul path, and relres of the y column at p (regime A/B indicator,
SURVEY.md §8c).  One JSON line per config.  python scripts/bench_configs.py [C0 C1 ...] [--reps R]"""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_1809_11165_b200 as bb  # noqa: E402

PATHS = {0: "CUDA-core on the fly (FP64ACC)", 1: "stored fp32 K (CUDA cores)",
         2: "tcgen05 on the fly (k1tc2)", 3: "tcgen05 stored int8 K (k2tc)"}


def main(argv):
    reps = 3
    if "--reps" in argv:
        i = argv.index("--reps")
        reps = int(argv[i + 1])
        argv = argv[:i] + argv[i + 2:]
    names = argv or ["C0", "C1", "C2", "C3", "C4"]
    ctx = bb.Context(0)
    for name in names:
        cfg = synth.CONFIGS[name]
        pr = synth.make_problem(cfg, seed=0)
        X, y = torch.from_numpy(pr.X).cuda(), torch.from_numpy(pr.y).cuda()
        h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
        km = bb.STORED if cfg.stored else bb.ONTHEFLY
        runs = [bb.mll_and_grad(ctx, X, y, h, cfg.t, cfg.k, cfg.p, seed=7, kmode=km)
                for _ in range(reps + 1)][1:]
        st = [r["stats"] for r in runs]
        ms = statistics.median(s["ms_total"] for s in st)
        mm = statistics.median(s["ms_matmul"] / max(s["matmul_launches"], 1) for s in st)
        s0 = st[-1]
        print(json.dumps({
            "config": name, "n": cfg.n, "d": cfg.d, "t": cfg.t, "k": cfg.k, "p": cfg.p,
            "kind": "matern52" if cfg.kind == bb.MATERN52 else "rbf",
            "kmode": "stored" if km == bb.STORED else "onthefly",
            "matmul_path": s0["matmul_path"], "path": PATHS.get(s0["matmul_path"]),
            "ms_mll_grad": ms, "ms_per_matmul": mm, "matmul_launches": s0["matmul_launches"],
            "ms_pivchol": s0["ms_pivchol"], "ms_mbcg": s0["ms_mbcg"], "ms_deriv": s0["ms_deriv"],
            "gpu_launches": s0["gpu_launches"], "relres_y_at_p": s0["relres_y"],
            "k_used": s0["k_used"], "mll": runs[-1]["mll"], "reps": reps}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main(sys.argv[1:])
