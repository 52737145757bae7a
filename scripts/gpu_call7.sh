#!/bin/bash
mkdir -p gpurun_out
timeout 300 python bench.py --steps 50 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for c in c5 c3_b64_g3 c3_b256_g5; do
timeout 400 python bench.py --config $c --steps 20 --cpu-budget 8 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
