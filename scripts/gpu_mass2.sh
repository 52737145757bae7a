#!/bin/bash
# k_mass cp.async ring: parity subset, NST sweep on bench points, sampler launch list.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q > gpurun_out/mass2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/mass2_pytest.log
for nst in 2 3 4; do
  for c in c3_b256_mixed c3_b256_g5 c3_b64_g3; do
    NJ_MASS_NST=$nst timeout 300 python bench.py --config $c --steps 20 --no-cpu-baseline > gpurun_out/mass2_bench_${c}_nst$nst.json 2>/dev/null
  done
  NJ_MASS_NST=$nst timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_mass|k_locate|k_sample_lse" --csv --log-file gpurun_out/mass2_launches_b256g5_nst$nst.csv python scripts/prof_fused.py 256 5 twopass > /dev/null 2>&1
done
