#!/bin/bash
# Round-end evidence (after the k_mass redesign, nj_propose, nj_verify_greedy): bench lines, C3 sweep, C4 trace,
# sampler launch list + ncu --set full of k_mass, GPU tests and smoke.
mkdir -p gpurun_out
python -m paper_2512_22420_b200._build > gpurun_out/f5_build.log 2>&1
timeout 300 python bench.py > gpurun_out/f5_bench_c2.json 2> gpurun_out/f5_bench_c2.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f5_bench_ref.json 2> gpurun_out/f5_bench_ref.err
for c in c3_b64_g3 c3_b256_g2 c3_b256_g5 c3_b256_mixed c5; do
  timeout 400 python bench.py --config $c --steps 20 --cpu-budget 6 > gpurun_out/f5_bench_$c.json 2> gpurun_out/f5_bench_$c.err
done
for c in propose greedy_c2 greedy_b256g5; do
  timeout 300 python bench.py --config $c --steps 30 > gpurun_out/f5_bench_$c.json 2> gpurun_out/f5_bench_$c.err
done
timeout 900 python bench.py --sweep --steps 10 --sweep-gamma 0,1,2,3,5,mixed:5 --sweep-B 1,8,16,32,48,64,96,128,192,256 > gpurun_out/f5_sweep.jsonl 2> gpurun_out/f5_sweep.err
timeout 600 python bench.py --config c4 --trace-steps 600 --warmup 20 > gpurun_out/f5_bench_c4.json 2> gpurun_out/f5_bench_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"^k_" --csv --log-file gpurun_out/f5_launches_b256g5.csv python scripts/prof_fused.py 256 5 twopass > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mass -s 1 -c 1 -o gpurun_out/f5_kmass_b256g5 -f python scripts/prof_fused.py 256 5 twopass > gpurun_out/f5_ncu_kmass.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/f5_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/f5_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f5_smoke.log 2>&1
