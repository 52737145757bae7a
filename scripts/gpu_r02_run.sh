#!/bin/bash
# Round-2 GPU session: tests, smoke, c_prefill measurement, bench lines.
# usage: bash scripts/gpu_r02_run.sh TAG [parts...]   (parts: tests smoke cprefill bench c4 c5 sweep ref)
set -u
TAG=$1; shift
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAILED; tail -20 $O/build.log; exit 1; }
for part in "$@"; do
  case $part in
    tests) timeout 1800 python -m pytest tests -m gpu -q --durations=15 > $O/gputest.log 2>&1; tail -3 $O/gputest.log ;;
    smoke) timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log ;;
    cprefill) timeout 900 python scripts/measure_cprefill.py > $O/cprefill.log 2>&1; tail -2 $O/cprefill.log; cp profiles/r02_cprefill_b200.* $O/ 2>/dev/null ;;
    bench) for c in c2 c3_b64_g3 c3_b256_g2 c3_b256_g5 c3_b256_mixed; do timeout 600 python bench.py --config $c --steps 50 --warmup 5 > $O/bench_$c.json 2> $O/bench_$c.err; tail -c 300 $O/bench_$c.json; echo; done ;;
    c4) timeout 900 python bench.py --config c4 --warmup 50 > $O/bench_c4.json 2> $O/bench_c4.err; tail -c 600 $O/bench_c4.json; echo ;;
    c5) timeout 600 python bench.py --config c5 --steps 30 --warmup 5 > $O/bench_c5.json 2> $O/bench_c5.err; tail -c 300 $O/bench_c5.json; echo ;;
    sweep) timeout 1200 python bench.py --sweep --steps 20 > $O/sweep_c3.jsonl 2> $O/sweep.err; wc -l $O/sweep_c3.jsonl ;;
    ref) timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_c2.json 2> $O/bench_ref.err; tail -c 300 $O/bench_ref_c2.json; echo ;;
  esac
done
