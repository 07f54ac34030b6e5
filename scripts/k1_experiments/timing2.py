"""Build a K1-TC variant that records clock64() phase stamps (one CTA, tiles T0..T0+255), and
(with --run, on a GPU) run it at C4 and summarise.

    python scripts/k1_experiments/timing2.py build
    python scripts/k1_experiments/timing2.py run      # on the GPU box: prints the summary

Compute warp w (lane 0), per tile: c0 loop top, c1 s_full passed, c2 TMEM load done, c3 first half
quantised, c4 deferred publish done, c5 tile end.  MMA warp: i0 top, i1 x-stage ready, i2 a_full
passed, i3 D-slices ready, i4 int8 MMAs issued, i5 distance MMA issued.
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
VAR = os.path.join(ROOT, "scratch", "var_timing")
T0, NT, CTA = 1000, 256, 200


def build():
    from paper_1809_11165_b200 import _build as B
    src = open(os.path.join(B.CSRC, "k1tc2.cu")).read()

    def rep(a, b):
        nonlocal src
        assert a in src, a
        src = src.replace(a, b, 1)

    rep("namespace bbmm {\nnamespace tc2 {\n",
        f"__device__ long long g_ts[18][{NT}][6];\nnamespace bbmm {{\nnamespace tc2 {{\n")
    # compute warps (non-pipelined loop)
    rep("""        } else
        for (int t = 0; t < ntl; t++) {
            const int b = t % K::NBUF;
""", f"""        }} else
        for (int t = 0; t < ntl; t++) {{
            const bool rec_ = blockIdx.x == {CTA} && lane == 0 && t >= {T0} && t < {T0 + NT};
            long long *ts_ = g_ts[warp][rec_ ? t - {T0} : 0];
            if (rec_) ts_[0] = clock64();
            const int b = t % K::NBUF;
""")
    rep("""            ptx::tc_fence_after();
            uint32_t sv[JW];""", """            ptx::tc_fence_after();
            if (rec_) ts_[1] = clock64();
            uint32_t sv[JW];""")
    rep("""            if constexpr (MODE != 2) ptx::tmem_ld_wait();
            uint32_t w0[JW / 4], w1[JW / 4], w2[JW / 4];""",
        """            if constexpr (MODE != 2) ptx::tmem_ld_wait();
            if (rec_) ts_[2] = (long long)clock64() + (sv[0] == 0x7fffffffu);
            uint32_t w0[JW / 4], w1[JW / 4], w2[JW / 4];""")
    rep("""            if (DEFER && t > 0) publish(t - 1);""",
        """            if (rec_) ts_[3] = (long long)clock64() + (w0[3] == 0x12345u);
            if (DEFER && t > 0) publish(t - 1);
            if (rec_) ts_[4] = clock64();""")
    rep("""            if (!DEFER) publish(t);
        }""", """            if (!DEFER) publish(t);
            if (rec_) ts_[5] = (long long)clock64() + (w2[7] == 0x12345u);
        }""")
    # MMA issuer
    rep("""            const bool first = (t % TPW) == 0;
            // operands of the next distance MMA""", f"""            const bool first = (t % TPW) == 0;
            const bool irec_ = blockIdx.x == {CTA} && t >= {T0} && t < {T0 + NT};
            long long *its_ = g_ts[17][irec_ ? t - {T0} : 0];
            if (irec_ && leader) its_[0] = clock64();
            // operands of the next distance MMA""")
    rep("""            if (first && win > 0) wait_b(&acc_empty""", """            if (irec_ && leader) its_[1] = clock64();
            if (first && win > 0) wait_b(&acc_empty""")
    rep("""            wait_b(&full_q[qi], (uint32_t)((t / K::QS) & 1));""",
        """            if (irec_ && leader) its_[2] = clock64();
            wait_b(&full_q[qi], (uint32_t)((t / K::QS) & 1));
            if (irec_ && leader) its_[3] = clock64();""")
    rep("""            __syncwarp();
            if (t + K::NBUF < ntl) issue_dist(t + K::NBUF);""", """            __syncwarp();
            if (irec_ && leader) its_[4] = clock64();
            if (t + K::NBUF < ntl) issue_dist(t + K::NBUF);
            if (irec_ && leader) its_[5] = clock64();""")
    rep("int k1tc2_matmul(bbmm_ctx_s *ctx,", f"""extern "C" int bbmm_debug_ts(long long *out) {{
    return (int)cudaMemcpyFromSymbol(out, g_ts, sizeof(long long) * 18 * {NT} * 6);
}}
int k1tc2_matmul(bbmm_ctx_s *ctx,""")
    inc, libdir = B.nccl_paths()
    objs = [os.path.join(B.BUILD, f) for f in os.listdir(B.BUILD) if f.endswith(".o") and f != "k1tc2.cu.o"]
    d = os.path.join(VAR, "paper_1809_11165_b200")
    os.makedirs(os.path.join(d, "lib"), exist_ok=True)
    shutil.copy(os.path.join(ROOT, "paper_1809_11165_b200", "__init__.py"), d)
    f = os.path.join(VAR, "k1tc2.cu")
    open(f, "w").write(src)
    subprocess.check_call([B.NVCC, "-std=c++17", "-O3", *B.ARCH, "-Xcompiler", "-fPIC", "-I", inc, "-I",
                           B.CSRC, "-I", os.path.join(ROOT, "include"), "--expt-relaxed-constexpr",
                           "-c", f, "-o", f + ".o"])
    subprocess.check_call([B.NVCC, "-shared", *B.ARCH, "-o", os.path.join(d, "lib", "libbbmm.so"), f + ".o",
                           *objs, "-L", libdir, "-l:libnccl.so.2", "-Xlinker", f"-rpath={libdir}"])
    os.remove(f + ".o")
    print("ok")


def run():
    import ctypes
    import numpy as np
    import torch
    sys.path.insert(0, VAR)
    import synth
    import paper_1809_11165_b200 as bb
    assert bb.__file__.startswith(VAR)
    cfg = synth.CONFIGS["C4"]
    pr = synth.make_problem(cfg, seed=0)
    D = synth.random_block(cfg.n, 17, seed=4).astype(np.float64)
    ctx = bb.Context(0)
    X = torch.from_numpy(pr.X).cuda()
    Dd = torch.from_numpy(D).cuda()
    h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
    bb.kernel_matmul(ctx, X, Dd, h)
    torch.cuda.synchronize()
    ts = np.zeros((18, NT, 6), np.int64)
    bb._lib.bbmm_debug_ts(ts.ctypes.data_as(ctypes.c_void_p))
    np.save(os.path.join(ROOT, "gpurun_out", "k1_ts.npy"), ts)
    summarize(ts)


def summarize(ts):
    import numpy as np
    cw = ts[:16]
    dt = np.diff(cw[:, :, 0], axis=1)            # tile period per warp
    print("tile period (cycles): median %.0f mean %.0f" % (np.median(dt), dt.mean()))
    ph = ["wait s_full", "ld", "quant 1st half", "publish(t-1)", "rest (st, quant 2nd)"]
    for k in range(5):
        d = cw[:, :, k + 1] - cw[:, :, k]
        print("  %-22s median %6.0f mean %6.0f p90 %6.0f" % (ph[k], np.median(d), d.mean(), np.percentile(d, 90)))
    # lockstep: spread of the tile start among the 4 warps of each sub-partition (w % 4)
    for sub in range(4):
        st = cw[sub::4, :, 0]
        print("  SMSP %d start spread across its 4 warps: median %.0f cycles" % (sub, np.median(st.max(0) - st.min(0))))
    mw = ts[17]
    ph2 = ["wait x", "acc_empty/a_full", "full_q", "int8 issue", "dist issue"]
    dtm = np.diff(mw[:, 0])
    print("MMA loop period median %.0f" % np.median(dtm))
    for k in range(5):
        d = mw[:, k + 1] - mw[:, k]
        print("  MMA %-18s median %6.0f mean %6.0f" % (ph2[k], np.median(d), d.mean()))


if __name__ == "__main__":
    {"build": build, "run": run}[sys.argv[1]]()
