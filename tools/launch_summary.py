"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per kernel launches, total/avg device time and share of all launches."""
import collections
import csv
import io
import json
import sys

path, cmd = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
text = open(path).read()
start = text.index('"ID"')
rows = list(csv.reader(io.StringIO(text[start:])))
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[1:]:
    if len(r) <= vi:
        continue
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
    t = float(r[vi].replace(",", "")) * scale
    tot[r[ki]] += t
    cnt[r[ki]] += 1
T = sum(tot.values())
out = {"command": cmd, "ncu": "--metrics gpu__time_duration.sum --clock-control none",
       "note": "cold-cache, serialised per-launch times: compare shares, not absolutes",
       "kernels": [{"kernel": k, "launches": cnt[k], "total_us": round(tot[k], 1),
                    "avg_us": round(tot[k] / cnt[k], 2), "share": round(tot[k] / T, 4)}
                   for k in sorted(tot, key=lambda k: -tot[k])]}
print(json.dumps(out, indent=1))
