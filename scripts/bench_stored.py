"""Measure the stored-K kernel-matmul (row a6, stored variant) at the C2 / C1 shapes on one B200.

For each (config, operator) one full bbmm_mll_and_grad (pivoted Cholesky, p = 20 mBCG iterations,
SLQ, derivative pass) is run after a warm-up call; the library's own CUDA events give the K-hat*D
time per launch (ms_matmul / matmul_launches).  Operators:
  stored_int8  -- BBMM_STORED, INT8EXACT: K as four u8 slices (30-bit fixed point), tcgen05 (k2tc)
  stored_fp32  -- BBMM_STORED, FP64ACC:   K as fp32 (4 B per entry), CUDA-core DFMA (k2_stored)
  onthefly     -- BBMM_ONTHEFLY, default precision (tcgen05 where the kernel supports the shape)
  onthefly_fp64acc -- BBMM_ONTHEFLY, FP64ACC (CUDA-core DFMA)
Roofline of the stored variants: HBM, algorithmic bytes per launch = bytes of the stored
representation (4 x n_loc_pad x n_pad for the int8 slices, 4 x n_loc x n for fp32) / per-launch time vs MEASURED_PEAKS.json hbm_gbs.
One JSON line per (config, operator).  usage: python scripts/bench_stored.py [C2|C1 ...]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_1809_11165_b200 as bb  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]


def pad(x, m):
    return (x + m - 1) // m * m


def main(names):
    ctx = bb.Context(0)
    for name in names:
        cfg = synth.CONFIGS[name]
        pr = synth.make_problem(cfg, seed=0)
        X, y = torch.from_numpy(pr.X).cuda(), torch.from_numpy(pr.y).cuda()
        h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
        n = cfg.n
        for label, kmode, prec in [("stored_int8", bb.STORED, bb.INT8EXACT),
                                   ("stored_fp32", bb.STORED, bb.FP64ACC),
                                   ("onthefly", bb.ONTHEFLY, bb.INT8EXACT),
                                   ("onthefly_fp64acc", bb.ONTHEFLY, bb.FP64ACC)]:
            ctx.set_matmul_precision(prec)
            try:
                runs = []
                for _ in range(3):
                    runs.append(bb.mll_and_grad(ctx, X, y, h, cfg.t, cfg.k, cfg.p, seed=7,
                                                kmode=kmode))
            finally:
                ctx.set_matmul_precision(bb.INT8EXACT)
            st = runs[-1]["stats"]
            per = st["ms_matmul"] / max(st["matmul_launches"], 1)
            line = {"config": name, "operator": label, "n": n, "d": cfg.d, "c": cfg.t + 1,
                    "kind": "matern52" if cfg.kind == bb.MATERN52 else "rbf",
                    "matmul_path": st["matmul_path"], "ms_per_matmul": per,
                    "ms_mll_grad": st["ms_total"], "ms_matmul_total": st["ms_matmul"],
                    "ms_pivchol": st["ms_pivchol"], "ms_deriv": st["ms_deriv"],
                    "mll": runs[-1]["mll"]}
            if kmode == bb.STORED:
                bpe = 4
                tc = st["matmul_path"] == 3
                rows = pad(n, 128) if tc else n
                cols = pad(n, 384) if tc else pad(n, 4)
                byts = bpe * rows * cols
                gbs = byts / (per * 1e-3) / 1e9
                line["roofline"] = {"bound": "hbm", "achieved": gbs, "peak": PEAK, "unit": "GB/s",
                                    "frac": gbs / PEAK, "bytes_per_launch": byts,
                                    "bytes_per_entry": bpe}
            print(json.dumps(line), flush=True)
    ctx.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["C2", "C1"])
