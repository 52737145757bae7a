#!/bin/bash
# Round-2 final evidence: bench lines for every row, C3 sweep, launch lists, ncu --set full of the
# dominant kernels.  Outputs under gpurun_out/$1.
set -u
O=gpurun_out/$1; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
run() { local name=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$name.json 2> $O/bench_$name.err; tail -c 250 $O/bench_$name.json; echo; }
run c4 --config c4 --warmup 50
run propose --config propose --steps 50 --warmup 5
run greedy_c2 --config greedy_c2 --steps 50 --warmup 5
run greedy_b256g5 --config greedy_b256g5 --steps 20 --warmup 3
run c2_T0.7 --config c2 --temperature 0.7 --steps 50 --warmup 5 --no-cpu-baseline
run c3_b256_g5_T1.5 --config c3_b256_g5 --temperature 1.5 --steps 30 --warmup 5 --no-cpu-baseline
run ref_c2 --impl reference --steps 3 --warmup 1
run ref_propose --impl reference --config propose --steps 3 --warmup 1
timeout 1500 python bench.py --sweep --steps 20 > $O/sweep_c3.jsonl 2> $O/sweep.err; wc -l $O/sweep_c3.jsonl
# launch lists (device time per launch, ncu serialised / cold-cache: compare shares)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 60 --csv --log-file $O/launches_c2.csv \
    python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 60 --csv --log-file $O/launches_b256g5.csv \
    python bench.py --config c3_b256_g5 --steps 5 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
# full captures of the dominant kernels
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused_verify -s 3 -c 1 -o $O/fused_c2 \
    python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_big -s 6 -c 1 -o $O/gemmbig_ka_b256g5 \
    python bench.py --config c3_b256_g5 --steps 2 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mass -s 3 -c 1 -o $O/kmass_b256g5 \
    python bench.py --config c3_b256_g5 --steps 2 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
ls $O
