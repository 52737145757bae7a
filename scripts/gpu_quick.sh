#!/bin/bash
# quick perf + parity check: bench lines (no cpu baseline) for the given configs, then a test subset
O=gpurun_out/${1:-quick}; shift
mkdir -p $O
python -m paper_2512_22420_b200._build > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
for c in $CONFIGS; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
  python -c "
import json; d=json.loads(open('$O/bench_$c.json').read().strip().split('\n')[-1]); r=d['roofline']
print('$c', round(d['value']), 'pos/s', round(d['ms_per_step']*1e3,1), 'us/step; kernel', round(r['kernel_ms_avg']*1e3,1), 'us frac', round(r['frac'],3))" 2>&1 | tail -1
done
if [ -n "$TESTS" ]; then timeout 1500 python -m pytest tests -m gpu -q -x -k "$TESTS" > $O/tests.log 2>&1; tail -2 $O/tests.log; fi
