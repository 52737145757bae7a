"""One line per bench JSON: config, value, ms/step, dominant kernel and its roofline fraction, e2e, clocks.
usage: python scripts/summarize_bench.py DIR"""
import glob
import json
import os
import sys

for f in sorted(glob.glob(os.path.join(sys.argv[1], "bench_*.json"))):
    try:
        d = json.loads(open(f).read().strip().split("\n")[-1])
    except Exception as e:   # noqa: BLE001
        print(os.path.basename(f), "unreadable", e)
        continue
    r = d.get("roofline") or {}
    e2e = d.get("e2e") or {}
    clk = d.get("clocks") or {}
    print(f"{os.path.basename(f)[6:-5]:18s} value={d.get('value', 0):12.1f} {d.get('unit', '')[:12]:12s} "
          f"ms/step={d.get('ms_per_step', 0) * 1e3:8.1f}us  kern={str(r.get('kernel', ''))[:28]:28s} "
          f"frac={r.get('frac', 0) or 0:.3f} kms={(r.get('kernel_ms_avg') or 0) * 1e3:7.1f}  "
          f"e2e={e2e.get('value', 0) or 0:10.1f}  clk={clk.get('sm_mhz')}")
