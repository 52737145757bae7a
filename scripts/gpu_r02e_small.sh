#!/bin/bash
O=gpurun_out/${1:-r02e_small}; mkdir -p $O
NJ_SMALL_INFO=1 timeout 300 python scripts/small_timeline.py 8 3 3 > $O/timeline_new.log 2>&1; grep -E 'co-resident|rep 4|   ' $O/timeline_new.log | tail -11
NJ_LM_PDL=0 NJ_SMALL_CL12=0 NJ_SMALL_REUSE=0 timeout 300 python scripts/small_timeline.py 8 3 3 > $O/timeline_old.log 2>&1; tail -10 $O/timeline_old.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "small or staged" 2>&1 | tail -2
bash scripts/gpu_ab_env.sh ${1:-r02e_small}/ab "NJ_LM_PDL=0 NJ_SMALL_CL12=0 NJ_SMALL_REUSE=0" "NJ_LM_PDL=1" c2 c3_b12_g3
