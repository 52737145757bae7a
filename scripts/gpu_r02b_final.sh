#!/bin/bash
# Round-2 (second session) evidence: bench lines for every row, C3 sweep, launch lists and
# ncu --set full captures of the dominant kernels (k_lmhead, k_fused_verify, k_mass).
# usage: bash scripts/gpu_r02b_final.sh TAG [parts...]  (parts: bench sweep launches ncu acc; default all)
set -u
O=gpurun_out/$1; shift; mkdir -p $O
PARTS=${*:-bench sweep launches ncu acc}
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
run() { local name=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$name.json 2> $O/bench_$name.err; tail -c 200 $O/bench_$name.json; echo; }
for part in $PARTS; do case $part in
bench)
  run c2 --config c2 --steps 100 --warmup 10
  for c in c3_b64_g3 c3_b256_g2 c3_b256_g5 c3_b256_mixed c3_b16_g2; do run $c --config $c --steps 50 --warmup 5 --no-cpu-baseline; done
  run c5 --config c5 --steps 30 --warmup 5
  run c4 --config c4 --warmup 50
  run propose --config propose --steps 50 --warmup 5
  run greedy_c2 --config greedy_c2 --steps 50 --warmup 5
  run greedy_b256g5 --config greedy_b256g5 --steps 20 --warmup 3
  run c2_T0.7 --config c2 --temperature 0.7 --steps 50 --warmup 5 --no-cpu-baseline
  run c3_b256_g5_T1.5 --config c3_b256_g5 --temperature 1.5 --steps 30 --warmup 5 --no-cpu-baseline
  run ref_c2 --impl reference --steps 3 --warmup 1 ;;
sweep)
  timeout 1500 python bench.py --sweep --steps 20 > $O/sweep_c3.jsonl 2> $O/sweep.err; wc -l $O/sweep_c3.jsonl ;;
launches)
  for c in c2 c3_b64_g3 c3_b256_g5; do
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -c 60 --csv --log-file $O/launches_$c.csv \
      python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
    python scripts/summarize_launches.py $O/launches_$c.csv $O/launches_$c.json > /dev/null
  done ;;
ncu)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused_verify -s 3 -c 1 -o $O/fused_c2 \
    python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lmhead -s 3 -c 1 -o $O/lmhead_b64g3 \
    python bench.py --config c3_b64_g3 --steps 2 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lmhead -s 3 -c 1 -o $O/lmhead_b256g5 \
    python bench.py --config c3_b256_g5 --steps 2 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mass -s 3 -c 1 -o $O/kmass_b256g5 \
    python bench.py --config c3_b256_g5 --steps 2 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1 ;;
acc)
  timeout 900 python scripts/lm_accuracy.py > $O/lm_accuracy.log 2>&1; cp gpurun_out/lm_accuracy.json $O/ 2>/dev/null; tail -3 $O/lm_accuracy.log ;;
esac; done
ls $O
