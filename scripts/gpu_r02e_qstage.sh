#!/bin/bash
O=gpurun_out/${1:-r02e_qstage}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "verify_host or cluster_sizes" > $O/parity.log 2>&1; tail -3 $O/parity.log
for c in c2 c3_b12_g3 c3_b16_g2; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline > $O/$c.json 2> $O/$c.err
  python -c "import json; d=json.loads(open('$O/$c.json').read().strip().split('\n')[-1]); e=d['e2e']; print('$c', round(d['ms_per_step']*1e3,1), 'e2e', round(e['value']), e['h2d_bytes_per_step'], e['q_rows'])"
done
