timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:k_mass -s 1 -c 3 --csv --log-file gpurun_out/km_new.csv python scripts/prof_fused.py 256 5 twopass > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:k_mass -s 1 -c 3 --csv --log-file gpurun_out/km64_new.csv python scripts/prof_fused.py 64 3 staged > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
