#!/bin/bash
O=gpurun_out/${1:-r02e_probe2}; mkdir -p $O
timeout 600 python scripts/time_lm.py 1536 "NJ_LM_DBG=58" "NJ_LM_DBG=58;NJ_LM_MB=1" "NJ_LM_DBG=58;NJ_LM_MB=3" "NJ_LM_DBG=58;NJ_LM_MB=4" "NJ_LM_DBG=58;NJ_LM_S=8;NJ_LM_MB=4" "NJ_LM_DBG=58;NJ_LM_S=8;NJ_LM_MB=6" "NJ_LM_DBG=570" "NJ_LM_DBG=570;NJ_LM_KS=56" "NJ_LM_DBG=58;NJ_LM_KS=56" "NJ_LM_DBG=58;NJ_LM_GK=2" "NJ_LM_DBG=58;NJ_LM_GK=2;NJ_LM_MB=2" "" "NJ_LM_MB=1" "NJ_LM_MB=3" "NJ_LM_MB=4" "NJ_LM_GK=2;NJ_LM_MB=1" "NJ_LM_GK=2;NJ_LM_MB=2" "NJ_LM_DBG=570;NJ_LM_CG=1" "NJ_LM_DBG=58;NJ_LM_CG=1" > $O/time_lm.log 2>&1
cat $O/time_lm.log
