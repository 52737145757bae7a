"""tcgen05.mma issue rate: cycles per 4-MMA group (one 64-deep k-block), single CTA
(M=128, N=n) and CTA pair (cta_group::2, M=256, each SM 128 x n), operands
resident in shared memory.  Modes: 0 commit at the end, 2 commit per group (the
ring's), 1 commit + wait per group, 4 / 5 the whole warp convergent with elect-predicated
issue (per MMA / four MMAs under one elect), commit per group; pair mode 3 rotates the
operands over 4 shared-memory stages (as a ring does).  Tensor floor per SM: 4 * 128 * n / 256 cycles."""
import sys

import torch

sys.path.insert(0, ".")
from scripts.probes import _probe  # noqa: E402

dev = torch.device("cuda:0")
out = torch.zeros(148, dtype=torch.int64, device=dev)
for cg, fn, ns, modes in ((1, _probe.mma_probe, (32, 64, 128, 192, 240, 256), (0, 2, 1, 4, 5, 6, 7)),
                          (2, _probe.mma_probe_cg2, (64, 128, 176, 192, 208, 224, 240, 256), (0, 2, 1, 3))):
    for mode in modes:
        for n in ns:
            out.zero_()
            for _ in range(2):
                fn(n, 4096, mode, out)
            torch.cuda.synchronize()
            c = out.float()
            c = c[c > 0]
            ideal = 4 * 128 * n / 256
            print(f"cg {cg} mode {mode} N={n}: cycles/group median {c.median():.0f} (min {c.min():.0f} max {c.max():.0f});"
                  f" tensor floor {ideal:.0f}", flush=True)
