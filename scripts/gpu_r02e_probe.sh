#!/bin/bash
# k_lmhead decomposition at HEAD: timings with probe bits, MMA-warp timeline
O=gpurun_out/${1:-r02e_probe}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/smi.txt
timeout 300 python scripts/time_lm.py 256,384,512,1536 "" "NJ_LM_DBG=48" "NJ_LM_DBG=58" "NJ_LM_DBG=570" "NJ_LM_DBG=1" "NJ_LM_DBG=8" > $O/time_lm.log 2>&1
timeout 300 python scripts/lm_timeline.py 1536 "0,58,48" > $O/timeline_1536.log 2>&1
timeout 300 python scripts/lm_timeline.py 256 "0,58" > $O/timeline_256.log 2>&1
tail -n 40 $O/time_lm.log
