timeout 600 python scripts/explore_fused.py > gpurun_out/explore_fused.log 2>&1
for s in 0 1; do NJ_SACC=$s timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or uncertified" > gpurun_out/pytest_sacc$s.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sacc$s.log; done
