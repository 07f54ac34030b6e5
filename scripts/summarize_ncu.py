"""Summarise one `ncu --set full` report (first kernel) into markdown."""
import csv, io, subprocess, sys

rep, dst, title = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
m = {h: (u, v) for h, u, v in zip(hdr, units, vals)}


def g(name):
    u, v = m.get(name, ("", "n/a"))
    return f"{v} {u}".strip()


keys = [
    ("Kernel", "Kernel Name"), ("Grid", "Grid Size"), ("Block", "Block Size"),
    ("Duration", "gpu__time_duration.sum"), ("SM clock", "smsp__cycles_elapsed.avg.per_second"),
    ("Registers/thread", "launch__registers_per_thread"),
    ("Shared mem/block (dyn)", "launch__shared_mem_per_block_dynamic"),
    ("Warps active (pct of peak)", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("Issue slots busy", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
    ("XU pipe (MUFU ex2) inst", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
    ("Tensor pipe cycles active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
    ("ALU pipe inst", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
    ("FMA pipe inst", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
    ("TMEM pipe inst", "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active"),
    ("L1/TEX throughput", "l1tex__throughput.avg.pct_of_peak_sustained_active"),
    ("L2 throughput", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("DRAM bytes read", "dram__bytes_read.sum"), ("DRAM bytes write", "dram__bytes_write.sum"),
    ("DRAM throughput", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
]
out = [f"# {title}", "", f"Source: `{rep}` (ncu --set full --clock-control none --import-source on).", "",
       "| metric | value |", "|---|---|"]
for label, k in keys:
    out.append(f"| {label} | {g(k)} |")
st = [(h, float(v)) for h, v in zip(hdr, vals)
      if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")
      and v not in ("", "n/a")]
tot = sum(v for _, v in st) or 1.0
out += ["", "Warp-state samples (top):", "", "| stall reason | share |", "|---|---:|"]
for h, v in sorted(st, key=lambda x: -x[1])[:10]:
    out.append(f"| {h.replace('smsp__pcsamp_warps_issue_stalled_', '')} | {100 * v / tot:.1f}% |")
open(dst, "w").write("\n".join(out) + "\n")
print("\n".join(out))
