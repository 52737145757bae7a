#!/bin/bash
# ncu --set full of the top kernels + C3 sweep.
mkdir -p gpurun_out
timeout 900 python bench.py --sweep --steps 20 --sweep-gamma 0,1,3,5,mixed:5 --sweep-B 1,8,16,32,48,64,128,256 > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused_verify -s 3 -c 1 -o gpurun_out/fused_c2 -f python scripts/prof_fused.py 8 3 fused > gpurun_out/ncu_fused.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_acc -s 2 -c 2 -o gpurun_out/gemmacc_b256g5 -f python scripts/prof_fused.py 256 5 twopass > gpurun_out/ncu_gemmacc.log 2>&1
