#!/bin/bash
# one line per bench JSON of an evidence directory
for f in $1/bench_*.json; do python - "$f" <<'PY'
import json,sys
f=sys.argv[1]
try:
    d=json.loads(open(f).read().strip().split('\n')[-1])
except Exception as e:
    print(f, 'ERR', e); sys.exit()
r=d.get('roofline') or {}
e=d.get('e2e') or {}
n=f.split('/')[-1][6:-5]
print(f"{n:18s} {d.get('value',0):11.1f} {d.get('unit','')[:12]:12s} {(d.get('ms_per_step') or 0)*1e3:8.1f}us kern {r.get('kernel_ms_avg',0)*1e3:7.1f}us frac {r.get('frac',0):.3f} burst {r.get('frac_burst',0):.3f} {r.get('bound','')[:6]:6s} e2e {e.get('value',0):9.1f} clk {d.get('clocks',{}).get('sm_mhz')} {d.get('clocks',{}).get('reasons')}")
PY
done
