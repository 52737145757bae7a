#!/bin/bash
# quick check after a k_lmhead change: staged parity subset, bench lines of the tensor-bound rows, A/B
O=gpurun_out/${1:-r02e_check}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "staged or full_size or lmhead or production" > $O/t_parity.log 2>&1; tail -3 $O/t_parity.log
for c in ${CONFIGS:-c3_b64_g3 c3_b256_g2 c3_b256_g5}; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
  python -c "
import json; d=json.loads(open('$O/bench_$c.json').read().strip().split('\n')[-1]); r=d['roofline']
print('$c', round(d['value']), 'pos/s', round(d['ms_per_step']*1e3,1), 'us/step; kernel', round(r['kernel_ms_avg']*1e3,1), 'us frac', round(r['frac'],3), 'burst', round(r.get('frac_burst',0),3), d['clocks'])" 2>&1 | tail -1
done
timeout 600 python scripts/ab_lm.py ${AB_R:-512,1024,1536} 7 "" "NJ_LM_GK=1" > $O/ab.log 2>&1; cat $O/ab.log
