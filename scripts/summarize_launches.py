"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) into
per-kernel counts / mean / share, keeping only libnj kernels (k_*) and the
step total.  Usage: python scripts/summarize_launches.py in.csv out.json [max_launches]
(max_launches: keep the first N libnj launches -- the bench's eager steps, not its e2e pass)"""
import csv
import json
import re
import sys
from collections import OrderedDict

rows = []
with open(sys.argv[1]) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    m = re.search(r"\b(k_[A-Za-z0-9_]+)", name)
    if not m:
        continue
    t = float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)   # -> us
    rows.append((m.group(1) + ("<" + name.split("<", 1)[1].split(">")[0] + ">" if "<" in name else ""), t,
                 r["Grid Size"], r["Block Size"]))
if len(sys.argv) > 3:
    rows = rows[:int(sys.argv[3])]
agg = OrderedDict()
for k, t, g, b in rows:
    a = agg.setdefault(k, {"launches": 0, "total_us": 0.0, "grid": g, "block": b})
    a["launches"] += 1
    a["total_us"] += t
tot = sum(a["total_us"] for a in agg.values())
for a in agg.values():
    a["mean_us"] = a["total_us"] / a["launches"]
    a["share"] = a["total_us"] / tot if tot else None
warm = "warm" in sys.argv[1]
out = {"source": sys.argv[1], "note": "ncu --metrics gpu__time_duration.sum --clock-control none" +
       ("; --cache-control none (no cache flush between kernels), serialised" if warm else "; cold-cache, serialised") +
       " per-launch times: compare SHARES with bench.py, not absolutes", "kernels": agg,
       "per_launch_us": [(k, round(t, 3)) for k, t, _, _ in rows]}
json.dump(out, open(sys.argv[2], "w"), indent=1)
for k, a in agg.items():
    print(f"{k:60s} n={a['launches']:4d} mean={a['mean_us']:9.2f}us share={a['share']:.3f}")
