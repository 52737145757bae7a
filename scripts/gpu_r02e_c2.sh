#!/bin/bash
O=gpurun_out/${1:-r02e_c2}; mkdir -p $O
nvidia-smi -q | grep -i -E 'product name|serial|GPC|SM count' | head > $O/smi.txt
for v in 1 0; do
  NJ_SMALL_INFO=1 NJ_SMALL_CL16=$v timeout 300 python bench.py --config c2 --steps 100 --warmup 10 --no-cpu-baseline > $O/c2_cl16_$v.json 2> $O/c2_cl16_$v.err
  grep 'co-resident' $O/c2_cl16_$v.err | head -1
  python -c "import json; d=json.loads(open('$O/c2_cl16_$v.json').read().strip().split('\n')[-1]); print('cl16=$v', d['ms_per_step']*1e3, d['roofline']['kernel_ms_avg']*1e3)"
done
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "small" 2>&1 | tail -2
