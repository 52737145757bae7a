#!/bin/bash
mkdir -p gpurun_out
for nst in 2 3 4; do for pr in 0; do
  NJ_MASS_PROBE=$pr NJ_MASS_NST=$nst timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_mass" --csv --log-file gpurun_out/mass8_nst${nst}_p$pr.csv python scripts/prof_fused.py 256 5 twopass > /dev/null 2>&1
done; done
for nst in 2 3 4; do
  NJ_MASS_NST=$nst timeout 300 python bench.py --config c3_b256_g5 --steps 20 --no-cpu-baseline > gpurun_out/mass8_bench_b256g5_nst$nst.json 2>/dev/null
  NJ_MASS_NST=$nst timeout 300 python bench.py --config c3_b256_mixed --steps 20 --no-cpu-baseline > gpurun_out/mass8_bench_mixed_nst$nst.json 2>/dev/null
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_statistical.py -x -q  > gpurun_out/mass8_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/mass8_pytest.log
