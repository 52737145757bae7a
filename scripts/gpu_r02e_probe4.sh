#!/bin/bash
O=gpurun_out/${1:-r02e_probe4}; mkdir -p $O
timeout 300 python scripts/lm_timeline.py 1536 "0,8,570,58" > $O/timeline_1536.log 2>&1
timeout 300 python scripts/time_lm.py 1536 "" "NJ_LM_DBG=384" "NJ_LM_DBG=8" "NJ_LM_DBG=2" "NJ_LM_KS=8" "NJ_LM_KS=56" "NJ_LM_DBG=58;NJ_LM_KS=56" "NJ_LM_DBG=570;NJ_LM_KS=8" "NJ_LM_OST=2" "NJ_LM_TMA_OUT=0" "NJ_LM_ARV1=1" > $O/time_lm.log 2>&1
cat $O/timeline_1536.log $O/time_lm.log
