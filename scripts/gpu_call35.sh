timeout 300 python bench.py --steps 100 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 300 python bench.py --config c3_b64_g3 --steps 30 --no-cpu-baseline > gpurun_out/bench_b64.json 2> gpurun_out/bench_b64.err
timeout 300 python bench.py --config c3_b256_g5 --steps 20 --no-cpu-baseline > gpurun_out/bench_b256.json 2> gpurun_out/bench_b256.err
