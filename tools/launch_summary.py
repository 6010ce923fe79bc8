"""Summarise an ncu launch-list CSV (gpu__time_duration.sum) per kernel: python tools/launch_summary.py FILE.csv [out.json]"""
import csv, sys, json, re, collections
rows = []
with open(sys.argv[1], newline="") as f:
    lines = [l for l in f if not l.startswith("==")]
rd = csv.DictReader(lines)
agg = collections.OrderedDict()
for r in rd:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("msy::", "").replace("void ", "")
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    us = v / 1e3 if unit in ("ns", "nsecond") else (v if unit in ("us", "usecond") else v * 1e3)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1; a[1] += us
tot = sum(a[1] for a in agg.values())
out = [{"kernel": k, "launches": a[0], "ms": a[1] / 1e3, "share": a[1] / tot, "avg_us": a[1] / a[0]}
       for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1])]
for o in out[:25]:
    print(f"{o['kernel'][:60]:60s} {o['launches']:7d} {o['ms']:9.2f} ms {100*o['share']:5.1f}% avg {o['avg_us']:8.1f} us")
print("total", tot / 1e3, "ms", sum(a[0] for a in agg.values()), "launches")
if len(sys.argv) > 2:
    json.dump({"total_kernel_ms": tot / 1e3, "launches": sum(a[0] for a in agg.values()), "kernels": out}, open(sys.argv[2], "w"), indent=1)
