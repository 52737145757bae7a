timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"^k_" -s 15 -c 40 --csv --log-file gpurun_out/launches_b64.csv python bench.py --config c3_b64_g3 --steps 5 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/ncu_b64.log 2>&1
timeout 300 python bench.py --config c3_b64_g3 --steps 30 --no-cpu-baseline > gpurun_out/bench_b64.json 2> gpurun_out/bench_b64.err
