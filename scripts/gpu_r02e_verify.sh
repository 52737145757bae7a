#!/bin/bash
# parity of the changed sampler paths + compute-sanitizer memcheck / synccheck over the sanitize cases
O=gpurun_out/${1:-r02e_verify}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cluster_sizes or staged_full_size or staged_small" > $O/parity.log 2>&1; tail -2 $O/parity.log
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --print-limit 20 python scripts/sanitize_cases.py --c2 > $O/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 $O/memcheck.log
timeout 1500 $CS --tool synccheck --print-limit 20 python scripts/sanitize_cases.py > $O/synccheck.log 2>&1; echo "synccheck rc=$?"; tail -3 $O/synccheck.log
