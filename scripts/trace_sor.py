"""CUPTI trace of one bbmm_sor_mbcg call at the C4 shape: per-kernel totals (row f4 profiling)."""
import collections, json, os, re, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_1809_11165_b200 as bb
from torch.profiler import profile, ProfilerActivity
n, m, k, p = 1_000_000, 300, int(os.environ.get("SOR_K", "100")), int(os.environ.get("SOR_P", "20"))
cfg = synth.scaled(synth.CONFIGS["C4"], n)
pr = synth.make_problem(cfg, seed=0)
Xu = synth.test_points(cfg, m, seed=13)
B = np.random.default_rng(1).standard_normal((n, 17))
ctx = bb.Context(0)
X, Xud, Bd = (torch.from_numpy(a).cuda() for a in (pr.X, Xu, B))
h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
bb.sor_mbcg(ctx, X, Xud, h, Bd, k=k, max_iter=p)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    bb.sor_mbcg(ctx, X, Xud, h, Bd, k=k, max_iter=p)
    torch.cuda.synchronize()
out = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "trace_sor.json")
prof.export_chrome_trace(out)
ev = [e for e in json.load(open(out))["traceEvents"] if e.get("cat") == "kernel"]
by = collections.defaultdict(lambda: [0, 0.0])
for e in ev:
    nm = e["name"]
    mm = re.search(r"(k_\w+)", nm)
    key = mm.group(1) if mm else nm[:50]
    by[key][0] += 1
    by[key][1] += e["dur"] / 1e3
for key, (c, v) in sorted(by.items(), key=lambda x: -x[1][1])[:15]:
    print("%9.2f ms %5d  %7.3f ms/launch  %s" % (v, c, v / c, key))
