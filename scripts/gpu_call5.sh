#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --sweep --steps 10 --sweep-gamma 0,1,3,5,mixed:5 --sweep-B 1,8,16,32,48,64,128,256 > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
