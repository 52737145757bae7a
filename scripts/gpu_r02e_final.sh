#!/bin/bash
# Round-2 (third session) evidence at HEAD: GPU suite, bench lines for every row, C3 sweep,
# launch lists and ncu --set full captures of the dominant kernels.
# usage: bash scripts/gpu_r02e_final.sh TAG [parts...]  (parts: tests bench sweep launches launches_warm ncu; default all)
set -u
O=gpurun_out/$1; shift; mkdir -p $O
PARTS=${*:-tests bench sweep launches launches_warm ncu}
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
run() { local name=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$name.json 2> $O/bench_$name.err; tail -c 200 $O/bench_$name.json; echo; }
for part in $PARTS; do case $part in
tests)
  timeout 2400 python -m pytest tests -m gpu -q -rs > $O/gpu_tests.log 2>&1; tail -n 40 $O/gpu_tests.log | grep -E 'TOTAL|passed|failed|error' ;
  timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log ;;
bench)
  run c2 --config c2 --steps 100 --warmup 10
  for c in c3_b64_g3 c3_b256_g2 c3_b256_g5 c3_b256_mixed c3_b16_g2 c3_b12_g3; do run $c --config $c --steps 50 --warmup 5 --no-cpu-baseline; done
  run c1 --config c1 --steps 100 --warmup 10 --no-cpu-baseline
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
  # -c: the 8 eager steps only (3 warm-up + 5 timed; C2 3 launches per step, the others 6) -- later
  # launches belong to the e2e pass, where k_mass reads the q rows over the host link
  for c in c2 c3_b64_g3 c3_b256_g5; do
    n=48; [ $c = c2 ] && n=24
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -c $n --csv --log-file $O/launches_$c.csv \
      python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
    python scripts/summarize_launches.py $O/launches_$c.csv $O/launches_$c.json > /dev/null
  done ;;
launches_warm)
  # the same launch lists without ncu's cache flush between kernels (the recipe's list is cold-cache)
  for c in c2 c3_b64_g3 c3_b256_g5; do
    n=48; [ $c = c2 ] && n=24
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:k_ -c $n --csv \
      --log-file $O/launches_warm_$c.csv python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
    python scripts/summarize_launches.py $O/launches_warm_$c.csv $O/launches_warm_$c.json > /dev/null
  done ;;
ncu)
  for spec in "lmhead_c2 c2 k_lmhead" "ksmall_c2 c2 k_sample_small" "lmhead_b64g3 c3_b64_g3 k_lmhead" "lmhead_b256g5 c3_b256_g5 k_lmhead" "kmass_b256g5 c3_b256_g5 k_mass"; do
    set -- $spec
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$3 -s 3 -c 1 -o $O/$1 \
      python bench.py --config $2 --steps 2 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
    python scripts/ncu_summary.py $O/$1.ncu-rep $O/ncu_$1.json "$3 at $2, ncu --set full" > /dev/null 2>&1
    rm -f $O/$1.ncu-rep   # reports exceed gpurun's 64 MiB copy-back
  done ;;
esac; done
ls $O
