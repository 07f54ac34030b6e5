#!/usr/bin/env python
"""Instruction histograms (tcgen05 / TMA / MUFU evidence) of the hot kernels' SASS.

    python scripts/sass_histogram.py > profiles/r02_sass_histograms.md

Runs cuobjdump -sass on the in-tree objects (paper_1809_11165_b200/build/*.o) and counts, per
kernel instantiation that the bench / tests run, the Blackwell-specific instructions:
UTCIMMA / UTCHMMA (tcgen05.mma kind::i8 / kind::tf32), UTCBAR (tcgen05.commit), LDTM / STTM
(tcgen05.ld / st), UBLKCP (cp.async.bulk, the TMA engine), SYNCS (mbarrier), MUFU.EX2 / MUFU.SQRT,
PRMT, FFMA2 / FADD2 / FMUL2 (paired FP32)."""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "paper_1809_11165_b200", "build")
KERNELS = [  # (object, mangled-name regex, label)
    ("k1tc2.cu.o", r"k1tc2_rbfILi17ELi8ELi3ELi8E", "k1tc2_rbf<17, 8, 3> (C4 K^D at n = 1M: 31-bit grid)"),
    ("k1tc2.cu.o", r"k1tc2_rbfILi17ELi8ELi0ELi8E", "k1tc2_rbf<17, 8, 0> (C4 K^D, 23-bit grid)"),
    ("k1tc2.cu.o", r"k1tc2_rbfILi17ELi8ELi1ELi8E", "k1tc2_rbf<17, 8, 1> (C4 derivative)"),
    ("k1tc2.cu.o", r"k1tc2_rbfILi33ELi32ELi0ELi32E", "k1tc2_rbf<33, 32, 0> (C3 K^D)"),
    ("k1tc2.cu.o", r"k1tc2_rbfILi17ELi16ELi2ELi9E", "k1tc2_rbf<17, 16, 2, 9> (C2 Matern on the fly)"),
    ("k2tc.cu.o", r"k2tc_storedILi17E", "k2tc_stored<17> (C2 stored K)"),
    ("deriv_tc2.cu.o", r"k_deriv_tc2ILi26ELi32ELi40E", "k_deriv_tc2<26, 32, 40> (C3 derivative)"),
    ("deriv_tc.cu.o", r"k_deriv_tcILi1ELi9ELi24E", "k_deriv_tc<1, 9, 24> (C2 Matern derivative)"),
]
OPS = ["UTCIMMA", "UTCHMMA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "SYNCS", "MUFU.EX2", "MUFU.SQRT",
       "PRMT", "FFMA2", "FADD2", "FMUL2", "FFMA", "DFMA"]


def main():
    print("# SASS instruction histograms of the hot kernels (round 2)\n")
    print("`cuobjdump -sass` of the in-tree objects built by `__graft_entry__.build()` "
          "(nvcc 12.9, `-gencode arch=compute_100a,code=sm_100a`); static instruction counts.\n")
    print("| kernel | " + " | ".join(OPS) + " | total |")
    print("|---|" + "---:|" * (len(OPS) + 1))
    cache = {}
    for obj, pat, label in KERNELS:
        path = os.path.join(BUILD, obj)
        if path not in cache:
            cache[path] = subprocess.run(["cuobjdump", "-sass", path], capture_output=True,
                                         text=True).stdout
        text = cache[path]
        funcs = re.split(r"\n\s*Function : ", text)
        body = next((f for f in funcs if re.match(r"\S*" + pat, f)), None)
        if body is None:
            print(f"| {label} | (not found) |")
            continue
        cnt = collections.Counter()
        total = 0
        for line in body.splitlines():
            m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
            if not m:
                continue
            op = m.group(2)
            total += 1
            for o in OPS:
                if op == o or op.startswith(o + "."):
                    cnt[o] += 1
        print(f"| {label} | " + " | ".join(str(cnt[o]) for o in OPS) + f" | {total} |")


if __name__ == "__main__":
    main()
