"""Trace one C4 MLL+grad step with torch.profiler (CUPTI): kernel time vs gaps.
usage: python scripts/trace_step.py [config] [n]"""
import sys, json, os, numpy as np, torch
sys.path.insert(0, '.')
import synth
import paper_1809_11165_b200 as bb
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
cfg = synth.CONFIGS[name]
if len(sys.argv) > 2:
    cfg = synth.scaled(cfg, int(sys.argv[2]))
pr = synth.make_problem(cfg, seed=0)
ctx = bb.Context(0)
X = torch.from_numpy(pr.X).cuda(); y = torch.from_numpy(pr.y).cuda()
h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
kw = dict(t=cfg.t, k=cfg.k, max_iter=cfg.p, tol=0.0, seed=1,
          kmode=bb.STORED if cfg.stored else bb.ONTHEFLY)
r = bb.mll_and_grad(ctx, X, y, h, **kw)          # warm-up
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    r = bb.mll_and_grad(ctx, X, y, h, **kw)
    torch.cuda.synchronize()
out = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "trace_%s.json" % name)
prof.export_chrome_trace(out)
ev = [e for e in json.load(open(out))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
t0, t1 = ev[0]["ts"], ev[-1]["ts"] + ev[-1]["dur"]
busy = sum(e["dur"] for e in ev)
gaps = [(ev[i + 1]["ts"] - (ev[i]["ts"] + ev[i]["dur"]), ev[i]["name"][:60], ev[i + 1]["name"][:60]) for i in range(len(ev) - 1)]
gaps.sort(key=lambda g: -g[0])
print("kernels %d  span %.1f ms  busy %.1f ms  idle %.1f ms" % (len(ev), (t1 - t0) / 1e3, busy / 1e3, (t1 - t0 - busy) / 1e3))
for g in gaps[:12]:
    print("  gap %.2f ms after %s -> %s" % (g[0] / 1e3, g[1], g[2]))
by = {}
for e in ev:
    k = e["name"].split("(")[0][-60:]
    by[k] = by.get(k, 0) + e["dur"]
for k, v in sorted(by.items(), key=lambda x: -x[1])[:15]:
    print("  %8.2f ms  %s" % (v / 1e3, k))
