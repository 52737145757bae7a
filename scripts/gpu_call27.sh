timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --sweep --steps 10 --sweep-gamma 1,2,3,5,mixed:5 --sweep-B 64,96,128,192 > gpurun_out/sweep2.jsonl 2> gpurun_out/sweep2.err
