timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --sweep --steps 10 --sweep-gamma 0,1,2,3,5,mixed:5 --sweep-B 1,8,16,32,48,64,96,128,192,256 > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
timeout 600 python bench.py --config c4 --trace-steps 600 --warmup 20 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
