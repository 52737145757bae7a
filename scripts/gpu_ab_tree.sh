#!/bin/bash
# A/B of the bench between the current tree and an older build in _ab_old/ (same box, alternating)
O=gpurun_out/${1:-ab_tree}; shift; mkdir -p $O
CFGS=${*:-c2}
for c in $CFGS; do for r in 1 2 3; do
  for t in new old; do
    if [ $t = new ]; then D=.; else D=_ab_old; fi
    (cd $D && NJ_SMALL_CL16=${CL16:-1} timeout 300 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1) > $O/${c}_${t}_$r.json
    python -c "import json; d=json.loads(open('$O/${c}_${t}_$r.json').read()); print('$c $t $r', round(d['ms_per_step']*1e3,1), round(d['roofline']['kernel_ms_avg']*1e3,1))"
  done
done; done
