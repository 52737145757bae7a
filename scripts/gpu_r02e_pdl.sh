#!/bin/bash
O=gpurun_out/${1:-r02e_pdl}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "staged or full_size_bench or graph" > $O/parity.log 2>&1; tail -2 $O/parity.log
bash scripts/gpu_ab_env.sh ${1:-r02e_pdl}/ab "NJ_PDL_CHAIN=0" "NJ_PDL_CHAIN=1" c3_b16_g2 c3_b64_g3 c3_b256_g5
