"""Build a libbbmm variant whose k1tc2.cu is compiled with extra -D flags (timing experiments).

    python scripts/k1_experiments/make_variant.py NAME -DBBMM_TC2_NPS=6 ...

Writes scratch/var_NAME/paper_1809_11165_b200/lib/libbbmm.so (the other objects from the main
build); time it with scripts/k1_ab.py.  Source ablations: ablate.py."""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_1809_11165_b200 import _build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
inc, libdir = B.nccl_paths()
SRCS = os.environ.get("VARIANT_SRC", "k1tc2.cu").split(",")   # sources compiled with the -D flags
objs = [os.path.join(B.BUILD, f) for f in os.listdir(B.BUILD) if f.endswith(".o") and f[:-2] not in SRCS]
d = os.path.join(ROOT, "scratch", "var_" + name, "paper_1809_11165_b200")
os.makedirs(os.path.join(d, "lib"), exist_ok=True)
shutil.copy(os.path.join(ROOT, "paper_1809_11165_b200", "__init__.py"), d)
vobjs = []
for src in SRCS:
    o = os.path.join(ROOT, "scratch", "var_" + name, src + ".o")
    subprocess.check_call([B.NVCC, "-std=c++17", "-O3", *B.ARCH, "-Xcompiler", "-fPIC", *defs, "-I", inc,
                           "-I", B.CSRC, "-I", os.path.join(ROOT, "include"), "--expt-relaxed-constexpr",
                           "-c", os.path.join(B.CSRC, src), "-o", o])
    vobjs.append(o)
subprocess.check_call([B.NVCC, "-shared", *B.ARCH, "-o", os.path.join(d, "lib", "libbbmm.so"), *vobjs, *objs,
                       "-L", libdir, "-l:libnccl.so.2", "-Xlinker", f"-rpath={libdir}"])
for o in vobjs:
    os.remove(o)
print("ok", name)
