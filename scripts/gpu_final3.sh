#!/bin/bash
# Round-end evidence: bench lines, C3 sweep, C4 trace, launch list, ncu --set full of the top kernels.
mkdir -p gpurun_out
timeout 300 python bench.py > gpurun_out/final_bench_c2.json 2> gpurun_out/final_bench_c2.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
for c in c3_b64_g3 c3_b256_g2 c3_b256_g5 c3_b256_mixed c5; do
  timeout 400 python bench.py --config $c --steps 20 --cpu-budget 6 > gpurun_out/final_bench_$c.json 2> gpurun_out/final_bench_$c.err
done
timeout 900 python bench.py --sweep --steps 10 --sweep-gamma 0,1,2,3,5,mixed:5 --sweep-B 1,8,16,32,48,64,96,128,192,256 > gpurun_out/final_sweep.jsonl 2> gpurun_out/final_sweep.err
timeout 600 python bench.py --config c4 --trace-steps 600 --warmup 20 > gpurun_out/final_bench_c4.json 2> gpurun_out/final_bench_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/final_ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused_verify -s 3 -c 1 -o gpurun_out/final_fused_c2 -f python scripts/prof_fused.py 8 3 fused > gpurun_out/final_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_big -s 3 -c 1 -o gpurun_out/final_big_staged -f python scripts/prof_fused.py 64 3 staged > gpurun_out/final_ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_big|k_mass" -s 4 -c 3 -o gpurun_out/final_twopass_b256g5 -f python scripts/prof_fused.py 256 5 twopass > gpurun_out/final_ncu3.log 2>&1
