#!/bin/bash
# A/B of bench.py configs under two env settings on one box, alternating runs
# usage: gpu_ab_env.sh TAG "ENV_A" "ENV_B" config...
O=gpurun_out/$1; A=$2; B=$3; shift 3; mkdir -p $O
for c in "$@"; do for r in 1 2 3; do
  for t in A B; do
    if [ $t = A ]; then E=$A; else E=$B; fi
    env $E timeout 300 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1 > $O/${c}_${t}_$r.json
    python -c "import json; d=json.loads(open('$O/${c}_${t}_$r.json').read()); print('$c $t($E) $r', round(d['ms_per_step']*1e3,1), round(d['roofline']['kernel_ms_avg']*1e3,1), d['clocks']['sm_mhz'])"
  done
done; done
