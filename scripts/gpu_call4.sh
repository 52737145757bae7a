#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/time_ks.py 1,2,4,8,16,56 > gpurun_out/time_ks.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_big -s 3 -c 1 -o gpurun_out/big_staged -f python scripts/prof_fused.py 64 3 staged > gpurun_out/ncu_big1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_big -s 2 -c 2 -o gpurun_out/big_b256g5 -f python scripts/prof_fused.py 256 5 twopass > gpurun_out/ncu_big2.log 2>&1
