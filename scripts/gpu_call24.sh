timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "host" > gpurun_out/pytest_host.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_host.log
timeout 300 python bench.py --steps 100 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 300 python bench.py --config c3_b256_g5 --steps 20 --no-cpu-baseline > gpurun_out/bench_c3_b256_g5.json 2> gpurun_out/bench_c3.err
