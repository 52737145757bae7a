#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_mass|k_locate|k_sample_lse|k_accept|k_lse_rows" --csv --log-file gpurun_out/loc_b256g5.csv python scripts/prof_fused.py 256 5 twopass > /dev/null 2>&1
for c in c3_b256_g5 c3_b256_mixed c3_b256_g2 c3_b64_g3; do
  timeout 300 python bench.py --config $c --steps 20 --no-cpu-baseline > gpurun_out/loc_bench_$c.json 2>/dev/null
done
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/loc_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/loc_pytest.log
