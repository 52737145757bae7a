#!/bin/bash
O=gpurun_out/${1:-r02e_flat3}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small or staged_full_size or verify_host or graph" > $O/parity.log 2>&1; tail -2 $O/parity.log
timeout 300 python scripts/small_timeline.py 8 3 3 > $O/timeline.log 2>&1; tail -10 $O/timeline.log
bash scripts/gpu_ab_env.sh ${1:-r02e_flat3}/ab "NJ_SMALL_FLAT=0" "NJ_SMALL_FLAT=1" c2 c3_b12_g3
bash scripts/gpu_ab_env.sh ${1:-r02e_flat3}/ab2 "NJ_SMALL_PF=0" "NJ_SMALL_PF=2" c2
