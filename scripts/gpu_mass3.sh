#!/bin/bash
mkdir -p gpurun_out
for nst in 2 3 4; do
  NJ_MASS_NST=$nst timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__occupancy_limit_shared_mem --clock-control none -k regex:"k_mass|k_locate|k_sample_lse" --csv --log-file gpurun_out/mass3_launches_b256g5_nst$nst.csv python scripts/prof_fused.py 256 5 twopass > /dev/null 2>&1
  NJ_MASS_NST=$nst timeout 300 python bench.py --config c3_b256_g5 --steps 20 --no-cpu-baseline > gpurun_out/mass3_bench_b256g5_nst$nst.json 2>/dev/null
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "twopass or staged or sampler or stage" > gpurun_out/mass3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/mass3_pytest.log
