#!/bin/bash
O=gpurun_out/${1:-r02e_flat}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small or staged_full_size or verify_host or graph" > $O/parity.log 2>&1; tail -2 $O/parity.log
for f in 1 0; do NJ_SMALL_FLAT=$f timeout 300 python scripts/small_timeline.py 8 3 3 > $O/timeline_flat$f.log 2>&1; tail -10 $O/timeline_flat$f.log; done
bash scripts/gpu_ab_env.sh ${1:-r02e_flat}/ab "NJ_SMALL_FLAT=0" "NJ_SMALL_FLAT=1" c2 c3_b12_g3 c3_b16_g2
