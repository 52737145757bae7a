#!/bin/bash
# Discriminating sanitizer runs for the round-3 k_lmhead findings:
#  initcheck with direct stores (NJ_LM_TMA_OUT=0): are the reported reads the TMA-stored logits?
#  racecheck of k_gemm_big's CTA pair (NJ_LM=0 NJ_CG=2): the same cta_group::2 TMEM-alloc report?
O=gpurun_out/sanitize2; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
NJ_LM_TMA_OUT=0 timeout 900 $CS --tool initcheck --print-limit 5 python scripts/sanitize_cases.py > $O/initcheck_direct_stores.log 2>&1; tail -2 $O/initcheck_direct_stores.log
NJ_LM=0 NJ_CG=2 timeout 900 $CS --tool racecheck --racecheck-report analysis --print-limit 5 python scripts/sanitize_cases.py > $O/racecheck_gemmbig_cg2.log 2>&1; tail -2 $O/racecheck_gemmbig_cg2.log
NJ_LM_CG=1 timeout 900 $CS --tool racecheck --racecheck-report analysis --print-limit 5 python scripts/sanitize_cases.py > $O/racecheck_lm_cg1.log 2>&1; tail -2 $O/racecheck_lm_cg1.log
