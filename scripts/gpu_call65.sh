for mb in 1 6 8; do
  cp gpurun_tmp/libnj_mb$mb.so paper_2512_22420_b200/libnj.so
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:k_mass -s 1 -c 3 --csv --log-file gpurun_out/km_mb$mb.csv python scripts/prof_fused.py 256 5 twopass > /dev/null 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:k_mass -s 1 -c 3 --csv --log-file gpurun_out/km64_mb$mb.csv python scripts/prof_fused.py 64 3 staged > /dev/null 2>&1
done
