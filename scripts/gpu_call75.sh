for v in 0 1 0 1; do
  cp gpurun_tmp/libnj_fma$v.so paper_2512_22420_b200/libnj.so
  echo "== fma_exp=$v" >> gpurun_out/timeline9.log
  timeout 300 python scripts/big_timeline3.py >> gpurun_out/timeline9.log 2>&1
done
cp gpurun_tmp/libnj_fma1.so paper_2512_22420_b200/libnj.so
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "staged or twopass or uncertified" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
