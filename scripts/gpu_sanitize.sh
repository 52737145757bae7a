#!/bin/bash
# compute-sanitizer over scripts/sanitize_cases.py; summaries -> gpurun_out/sanitize/
O=gpurun_out/sanitize; mkdir -p $O
python -m paper_2512_22420_b200._build > /dev/null 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --print-limit 20 python scripts/sanitize_cases.py --c2 > $O/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 $O/memcheck.log
timeout 1500 $CS --tool synccheck --print-limit 20 python scripts/sanitize_cases.py > $O/synccheck.log 2>&1; echo "synccheck rc=$?"; tail -3 $O/synccheck.log
timeout 2400 $CS --tool racecheck --racecheck-report analysis --print-limit 20 python scripts/sanitize_cases.py > $O/racecheck.log 2>&1; echo "racecheck rc=$?"; tail -3 $O/racecheck.log
timeout 1500 $CS --tool initcheck --print-limit 20 python scripts/sanitize_cases.py > $O/initcheck.log 2>&1; echo "initcheck rc=$?"; tail -3 $O/initcheck.log
