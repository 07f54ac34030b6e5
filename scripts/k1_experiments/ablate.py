"""Build K1-TC ablation variants (throw-away, results wrong by construction) for timing only.

    python scripts/k1_experiments/ablate.py NAME SUB[,SUB...] [-DFOO=1 ...]

SUBs: nomufu (kv = S instead of ex2), noi8 (no int8 MMAs), nodist (no distance MMAs: the S
buffer keeps stale values), nosttm (no A-slice stores; words kept live), noquant (no
FADD/PRMT: words = raw bits of k~).  Output: scratch/var_NAME (time with scripts/k1_ab.py).
"""
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_1809_11165_b200 import _build as B  # noqa: E402

name, subs = sys.argv[1], sys.argv[2].split(",")
defs = sys.argv[3:]
src = open(os.path.join(B.CSRC, "k1tc2.cu")).read()


def rep(a, b, count=1):
    global src
    assert a in src, a
    src = src.replace(a, b, count)


for sub in subs:
    if sub == "nomufu":
        rep("                    kv = ex2_approx(sj);", "                    kv = -sj * 1e-3f;")
    elif sub == "noi8":
        for a in ("ptx::mma_i8_ts(tmem + 0, aq", "ptx::mma_i8_ts(tmem + K::BLK, aq",
                  "ptx::mma_i8_ts(tmem + 2 * K::BLK, aq"):
            rep(a, "if (0) " + a)
    elif sub == "nodist":
        rep("ptx::mma_tf32_ss(tmem + K::BUF_OFF + b * BK, ad, bd, IDS, ks > 0 ? 1u : 0u);",
            "if (0) ptx::mma_tf32_ss(tmem + K::BUF_OFF + b * BK, ad, bd, IDS, ks > 0 ? 1u : 0u);")
    elif sub == "nosttm":
        # stores of the A slices dropped; the words folded into a value stored only if impossible
        src = re.sub(r"(\n\s*)(ptx::tmem_st4\(col \+ (?:0|8|16|4|12|20),)", r"\1if (0) \2", src)
        rep("            if (!DEFER) publish(t);",
            "            { uint32_t lv = 0;\n#pragma unroll\n              for (int u_ = 0; u_ < JW / 4; u_++) lv ^= w0[u_] + 3u * w1[u_] + 7u * w2[u_];\n"
            "              if (lv == 0x9e3779b9u) Vpart[threadIdx.x] = (double)lv; }\n            if (!DEFER) publish(t);")
    elif sub == "noquant":
        rep("            const uint32_t t01 = __byte_perm(q[0], q[1], 0x6240);\n"
            "            const uint32_t t23 = __byte_perm(q[2], q[3], 0x6240);\n"
            "            const uint32_t u01 = __byte_perm(q[0], q[1], 0x7351);\n"
            "            const uint32_t u23 = __byte_perm(q[2], q[3], 0x7351);\n"
            "            a0 = __byte_perm(t01, t23, 0x5410);\n"
            "            a2 = __byte_perm(t01, t23, 0x7632);\n"
            "            a1 = __byte_perm(u01, u23, 0x5410);",
            "            a0 = q[0]; a1 = q[1]; a2 = q[2] ^ q[3];")
    else:
        raise SystemExit("unknown ablation " + sub)

inc, libdir = B.nccl_paths()
objs = [os.path.join(B.BUILD, f) for f in os.listdir(B.BUILD) if f.endswith(".o") and f != "k1tc2.cu.o"]
d = os.path.join(ROOT, "scratch", "var_" + name, "paper_1809_11165_b200")
os.makedirs(os.path.join(d, "lib"), exist_ok=True)
shutil.copy(os.path.join(ROOT, "paper_1809_11165_b200", "__init__.py"), d)
f = os.path.join(ROOT, "scratch", "var_" + name, "k1tc2.cu")
open(f, "w").write(src)
o = f + ".o"
subprocess.check_call([B.NVCC, "-std=c++17", "-O3", *B.ARCH, "-Xcompiler", "-fPIC", *defs, "-I", inc,
                       "-I", B.CSRC, "-I", os.path.join(ROOT, "include"), "--expt-relaxed-constexpr",
                       "-c", f, "-o", o])
subprocess.check_call([B.NVCC, "-shared", *B.ARCH, "-o", os.path.join(d, "lib", "libbbmm.so"), o, *objs,
                       "-L", libdir, "-l:libnccl.so.2", "-Xlinker", f"-rpath={libdir}"])
print("ok", name)
