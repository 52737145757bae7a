#!/bin/bash
# ncu --set full captures of k_gemm_big (staged N=256 and two-pass K-A at B=256 gamma=5), CG=1 and CG=2
set -u
O=gpurun_out/${1:-r02p}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
for cg in 1 2; do
  NJ_CG=$cg timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_big -s 3 -c 1 \
     -o $O/gemmbig_staged_cg$cg python bench.py --config c3_b64_g3 --steps 2 --warmup 3 --no-cpu-baseline --no-graph > $O/ncu_staged_cg$cg.log 2>&1
  NJ_CG=$cg timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_big -s 6 -c 1 \
     -o $O/gemmbig_ka_cg$cg python bench.py --config c3_b256_g5 --steps 2 --warmup 3 --no-cpu-baseline --no-graph > $O/ncu_ka_cg$cg.log 2>&1
done
for cg in 1 2; do
  NJ_CG=$cg timeout 300 python bench.py --config c3_b64_g3 --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_b64g3_cg$cg.json 2>/dev/null
  NJ_CG=$cg timeout 300 python bench.py --config c3_b256_g5 --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_b256g5_cg$cg.json 2>/dev/null
done
timeout 900 python scripts/measure_cprefill.py > $O/cprefill.log 2>&1; cp profiles/r02_cprefill_b200.* $O/
timeout 600 python bench.py --config c5 --steps 30 --warmup 5 > $O/bench_c5.json 2> $O/bench_c5.err
ls -la $O
