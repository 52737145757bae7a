#!/bin/bash
O=gpurun_out/${1:-r02e_probe3}; mkdir -p $O
timeout 600 python scripts/time_lm.py 1536 "NJ_LM_GK=2" "NJ_LM_GK=2;NJ_LM_DBG=48" "NJ_LM_GK=2;NJ_LM_DBG=8" "NJ_LM_GK=2;NJ_LM_DBG=2" "NJ_LM_GK=2;NJ_LM_DBG=10" "NJ_LM_GK=2;NJ_LM_DBG=128" "NJ_LM_GK=2;NJ_LM_DBG=256" "NJ_LM_GK=2;NJ_LM_DBG=16" "NJ_LM_GK=2;NJ_LM_DBG=32" "NJ_LM_GK=2;NJ_LM_DBG=1" > $O/time_lm.log 2>&1
timeout 600 python scripts/time_lm.py 384,512,768,1024 "" "NJ_LM_GK=2" "NJ_LM_GK=2;NJ_LM_CG=2" "NJ_LM_CG=2" >> $O/time_lm.log 2>&1
cat $O/time_lm.log
