"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel."""
import collections, csv, re, sys

src, dst, title = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(src)))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
hdr = rows[hi]
idx = {h: i for i, h in enumerate(hdr)}
scale = {'ns': 1e-6, 'nsecond': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'ms': 1.0, 'msecond': 1.0}
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) < len(hdr) or r[idx['Metric Name']] != 'gpu__time_duration.sum':
        continue
    full = r[idx['Kernel Name']]
    base = full.replace('void ', '', 1)
    for pre in ('<unnamed>::', 'unnamed>::', '(anonymous namespace)::'):
        base = base.replace(pre, '')
    m = re.match(r'([\w:]+)', base)
    name = m.group(1) if m else full
    tmpl = re.search(r'<([^>]*)>', full)
    if tmpl and ('k1' in name or 'k2' in name or 'k7' in name or 'LtR' in name or 'expand' in name):
        name += '<' + tmpl.group(1) + '>'
    tot[name] += float(r[idx['Metric Value']].replace(',', '')) * scale[r[idx['Metric Unit']]]
    cnt[name] += 1
T = sum(tot.values())
out = [f"# {title}", "",
       "Per-launch device times from `ncu --metrics gpu__time_duration.sum --clock-control none`",
       "(cold-cache, serialised launches: compare SHARES of the step, not absolute times).", "",
       "| kernel | launches | total ms | share of step |", "|---|---:|---:|---:|"]
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    out.append(f"| `{k}` | {cnt[k]} | {v:.2f} | {100 * v / T:.2f}% |")
out.append(f"| **all** | {sum(cnt.values())} | {T:.2f} | 100% |")
open(dst, 'w').write("\n".join(out) + "\n")
print("\n".join(out))
