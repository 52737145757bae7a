#!/bin/bash
# k_lmhead bring-up: build, staged parity subset, quick bench lines
O=gpurun_out/${1:-lm}; mkdir -p $O
python -m paper_2512_22420_b200._build > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "staged_small or c1_golden" > $O/t_small.log 2>&1; tail -3 $O/t_small.log
if [ -z "$SMALL_ONLY" ]; then
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "staged_full_size or full_size_bench or staged_two" > $O/t_full.log 2>&1; tail -3 $O/t_full.log
for c in ${CONFIGS:-c3_b64_g3 c3_b256_g2 c3_b256_g5}; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
  python -c "
import json; d=json.loads(open('$O/bench_$c.json').read().strip().split('\n')[-1]); r=d['roofline']
print('$c', round(d['value']), 'pos/s', round(d['ms_per_step']*1e3,1), 'us/step; kernel', round(r['kernel_ms_avg']*1e3,1), 'us frac', round(r['frac'],3))" 2>&1 | tail -1
done
fi
