#!/bin/bash
mkdir -p gpurun_out
timeout 300 python bench.py > gpurun_out/final_bench_c2.json 2> gpurun_out/final_bench_c2.err
for c in c3_b64_g3 c3_b256_g2 c3_b256_g5 c3_b256_mixed c5; do
  timeout 400 python bench.py --config $c --steps 20 --cpu-budget 6 > gpurun_out/final_bench_$c.json 2> gpurun_out/final_bench_$c.err
done
timeout 900 python bench.py --sweep --steps 10 --sweep-gamma 0,1,2,3,5,mixed:5 --sweep-B 1,8,16,32,48,64,96,128,192,256 > gpurun_out/final_sweep.jsonl 2> gpurun_out/final_sweep.err
timeout 600 python bench.py --config c4 --trace-steps 600 --warmup 20 > gpurun_out/final_bench_c4.json 2> gpurun_out/final_bench_c4.err
