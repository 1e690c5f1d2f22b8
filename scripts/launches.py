"""Summarize an ncu --metrics gpu__time_duration.sum --csv launch list (second half = warm rep)."""
import collections
import csv
import re
import sys

path = sys.argv[1]
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
rows = list(csv.reader(open(path)))
hdr = None
data = []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
ks = [d for d in data if d.get("Metric Name") == "gpu__time_duration.sum"]
part = ks[int(len(ks) * (1 - frac)):]
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for d in part:
    name = re.sub(r"\(.*", "", d["Kernel Name"])[:48]
    agg[name][0] += 1
    agg[name][1] += float(d["Metric Value"]) * scale[d["Metric Unit"]]
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':48s} {'launches':>8s} {'total ms':>9s} {'avg us':>8s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:48s} {v[0]:8d} {v[1] / 1e3:9.3f} {v[1] / v[0]:8.2f} {v[1] / tot:6.1%}")
print(f"{'total':48s} {sum(v[0] for v in agg.values()):8d} {tot / 1e3:9.3f}")
