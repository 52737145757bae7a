#!/bin/bash
O=gpurun_out/${1:-r02e_fuseloc}; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_temperature.py -x -q -k "staged or full_size or graph or fallback or uncertified or temperature" > $O/parity.log 2>&1; tail -2 $O/parity.log
bash scripts/gpu_ab_env.sh ${1:-r02e_fuseloc}/ab "NJ_FUSE_LOCATE=0" "NJ_FUSE_LOCATE=1" c3_b64_g3 c3_b256_g5 c3_b256_g2
