#!/bin/bash
mkdir -p gpurun_out
timeout 400 python scripts/time_cg.py > gpurun_out/time_cg.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
