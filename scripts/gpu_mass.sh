#!/bin/bash
# k_mass ticket scheduler: GPU tests, bench points, launch list of the sampler kernels.
mkdir -p gpurun_out
python -m paper_2512_22420_b200._build > gpurun_out/mass_build.log 2>&1
for c in c3_b256_mixed c3_b256_g5 c3_b256_g2 c3_b64_g3; do
  timeout 300 python bench.py --config $c --steps 20 --no-cpu-baseline > gpurun_out/mass_bench_$c.json 2> gpurun_out/mass_bench_$c.err
done
for occ in 2 3; do
  NJ_MASS_OCC=$occ timeout 300 python bench.py --config c3_b256_mixed --steps 20 --no-cpu-baseline > gpurun_out/mass_bench_occ$occ.json 2>/dev/null
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_mass|k_locate|k_sample_lse" --csv --log-file gpurun_out/mass_launches_b256g5.csv python scripts/prof_fused.py 256 5 twopass > gpurun_out/mass_ncu1.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_mass|k_locate|k_sample_lse" --csv --log-file gpurun_out/mass_launches_b256g2.csv python scripts/prof_fused.py 256 2 twopass > gpurun_out/mass_ncu2.log 2>&1
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/mass_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/mass_pytest_gpu.log
