#!/bin/bash
# where the k_lmhead operand waits come from (R = 1536, 2-k-block stages): no H loads (16),
# no W loads (32), every unit loading unit 0's W rows (64: L2-resident W)
O=gpurun_out/${1:-r02e_probe5}; mkdir -p $O
timeout 600 python scripts/lm_timeline.py 1536 "0,16,32,64" > $O/timeline_1536.log 2>&1
timeout 600 python scripts/lm_timeline.py 768 "0,16,32,64" > $O/timeline_768.log 2>&1
grep -E 'dbg=|mean per stage|aempty' $O/timeline_*.log
