#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/pytest_sharded.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sharded.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "uncertified or staged_full or twopass" > gpurun_out/pytest_unc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_unc.log
timeout 900 python bench.py --sweep --steps 10 --sweep-gamma 0,3,5,mixed:5 --sweep-B 8,32,64,128,256 > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
