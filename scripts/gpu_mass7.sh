#!/bin/bash
mkdir -p gpurun_out
for pr in 1 3 4 5 7; do
  NJ_MASS_PROBE=$pr NJ_MASS_NST=4 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_mass" --csv --log-file gpurun_out/mass7_nst4_p$pr.csv python scripts/prof_fused.py 256 5 twopass > /dev/null 2>&1
done
NJ_MASS_NST=4 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_mass" -s 1 -c 1 -o gpurun_out/mass7_full_nst4 -f python scripts/prof_fused.py 256 5 twopass > gpurun_out/mass7_ncu.log 2>&1
NJ_MASS_NST=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_mass" -s 1 -c 1 -o gpurun_out/mass7_full_nst2 -f python scripts/prof_fused.py 256 5 twopass >> gpurun_out/mass7_ncu.log 2>&1
