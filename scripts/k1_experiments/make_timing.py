"""Scratch: build a libbbmm variant whose K1-TC kernel records clock64() phase timestamps."""
import os, shutil, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_1809_11165_b200 import _build as B
src = open(os.path.join(B.CSRC, "k1tc2.cu")).read()
subs = [
 ("""namespace bbmm {
namespace tc2 {
""", """__device__ long long g_tstamp[64][512][8];
namespace bbmm {
namespace tc2 {
"""),
 ("""        for (int t = 0; t < ntl; t++) {
            const int b = t % K::NBUF;
            ptx::mbar_wait_a(a_sfull + 8 * b, (uint32_t)((t / K::NBUF) & 1));""", """        const bool rec = blockIdx.x == 100 && blockIdx.y == 0 && lane == 0;
        for (int t = 0; t < ntl; t++) {
            const int b = t % K::NBUF;
            long long c0 = clock64();
            ptx::mbar_wait_a(a_sfull + 8 * b, (uint32_t)((t / K::NBUF) & 1));
            long long c1 = clock64();"""),
 ("""            ptx::tmem_ld_wait();
            uint32_t w0[JW / 4], w1[JW / 4], w2[JW / 4];""", """            ptx::tmem_ld_wait();
            long long c2 = clock64();
            uint32_t w0[JW / 4], w1[JW / 4], w2[JW / 4];"""),
 ("""            if (t > 0) publish(t - 1);
#pragma unroll
            for (int u = JW / 8""", """            long long c3 = clock64();
            if (t > 0) publish(t - 1);
            long long c4 = clock64();
#pragma unroll
            for (int u = JW / 8"""),
 ("""                ptx::tmem_st8(col + 16, *reinterpret_cast<const uint32_t(*)[8]>(w2));""", """                ptx::tmem_st8(col + 16, *reinterpret_cast<const uint32_t(*)[8]>(w2));
                long long c5 = clock64();
                if (rec && t < 512) { long long *p = g_tstamp[warp][t]; p[0]=c0; p[1]=c1; p[2]=c2; p[3]=c3; p[4]=c4; p[5]=c5; }"""),
 ("""        auto wait_stage = [&](int t) {""", """        const bool irec = blockIdx.x == 100 && blockIdx.y == 0 && lane == 0;
        auto wait_stage = [&](int t) {"""),
 ("""            if (t + K::NBUF < ntl) wait_stage(t + K::NBUF);
            if (first && win > 0) ptx::mbar_wait(&acc_empty, (uint32_t)((win - 1) & 1));
            ptx::mbar_wait(&a_full[b], (uint32_t)((t / K::NBUF) & 1));""", """            long long i0 = clock64();
            if (t + K::NBUF < ntl) wait_stage(t + K::NBUF);
            long long i1 = clock64();
            if (first && win > 0) ptx::mbar_wait(&acc_empty, (uint32_t)((win - 1) & 1));
            long long i2 = clock64();
            ptx::mbar_wait(&a_full[b], (uint32_t)((t / K::NBUF) & 1));
            long long i3 = clock64();"""),
 ("""            __syncwarp();
            if (t + K::NBUF < ntl) issue_dist(t + K::NBUF);
        }""", """            __syncwarp();
            long long i4 = clock64();
            if (t + K::NBUF < ntl) issue_dist(t + K::NBUF);
            long long i5 = clock64();
            if (irec && t < 512) { long long *p = g_tstamp[63][t]; p[0]=i0; p[1]=i1; p[2]=i2; p[3]=i3; p[4]=i4; p[5]=i5; }
        }"""),
 ("""                ptx::mbar_wait(&free_b[st], ph ^ 1);""", """                long long q0 = clock64();
                ptx::mbar_wait(&free_b[st], ph ^ 1);
                if (blockIdx.x == 100 && blockIdx.y == 0 && t < 512) { g_tstamp[62][t][0] = q0; g_tstamp[62][t][1] = clock64(); }"""),
]
for a, b in subs:
    assert a in src, a[:60]
    src = src.replace(a, b)
src = src.replace("""int k1tc2_matmul(bbmm_ctx_s *ctx,""", """extern "C" int bbmm_debug_tstamps(long long *out) {
    return (int)cudaMemcpyFromSymbol(out, g_tstamp, sizeof(long long) * 64 * 512 * 8);
}
int k1tc2_matmul(bbmm_ctx_s *ctx,""")
inc, libdir = B.nccl_paths()
objs = [os.path.join(B.BUILD, f) for f in os.listdir(B.BUILD) if f.endswith(".o") and f != "k1tc2.cu.o"]
d = os.path.join(ROOT, "scratch", "timing", "paper_1809_11165_b200")
os.makedirs(os.path.join(d, "lib"), exist_ok=True)
shutil.copy(os.path.join(ROOT, "paper_1809_11165_b200", "__init__.py"), d)
f = os.path.join(ROOT, "scratch", "timing", "k1tc2.cu")
open(f, "w").write(src)
cmd = [B.NVCC, "-std=c++17", "-O3", *B.ARCH, "-Xcompiler", "-fPIC", "-I", inc, "-I", B.CSRC,
       "-I", os.path.join(ROOT, "include"), "-c", f, "-o", f + ".o"]
subprocess.check_call(cmd)
subprocess.check_call([B.NVCC, "-shared", *B.ARCH, "-o", os.path.join(d, "lib", "libbbmm.so"), f + ".o", *objs,
                       "-L", libdir, "-l:libnccl.so.2", "-Xlinker", f"-rpath={libdir}"])
print("ok")
