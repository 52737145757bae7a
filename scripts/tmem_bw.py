"""TMEM read bandwidth on B200 (scripts/probes k_tmem_bw): bytes per SM-cycle of
tcgen05.ld.32x32b.x16/.x32 with 1-4 loads in flight per wait, 4-16 warps, plus
the register adds of the restart drain.  Answers: how long does draining one
128-lane x 256-column fp32 accumulator (128 KB) take?"""
import json
import sys

import torch

sys.path.insert(0, ".")
from scripts.probes import _probe  # noqa: E402

sms = torch.cuda.get_device_properties(0).multi_processor_count
out = torch.zeros(2 * sms, dtype=torch.int64, device="cuda")
res = []
for nw in (4, 8, 16):
    for x in (16, 32):
        for inf in (1, 2, 4):
            cols, rounds = 512, 200
            for _ in range(2):
                _probe.tmem_bw(nw, x, inf, cols, rounds, out)
            torch.cuda.synchronize()
            cyc = out[0::2].double().median().item()
            byts = 128 * cols * 4 * rounds   # every lane x column read once per round
            r = {"warps": nw, "x": x, "inflight": inf, "B_per_cycle": byts / cyc,
                 "drain_128KB_cycles": 131072 / (byts / cyc)}
            res.append(r)
            print(json.dumps(r), flush=True)
json.dump(res, open("gpurun_out/tmem_bw.json", "w"), indent=1)
