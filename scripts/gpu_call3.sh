#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/gpu_big_check.py > gpurun_out/big_check.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
