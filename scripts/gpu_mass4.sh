#!/bin/bash
mkdir -p gpurun_out
for nst in 2 4; do for pr in 0 1 2 3; do
  NJ_MASS_PROBE=$pr NJ_MASS_NST=$nst timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_mass" --csv --log-file gpurun_out/mass4_nst${nst}_p$pr.csv python scripts/prof_fused.py 256 5 twopass > /dev/null 2>&1
done; done
