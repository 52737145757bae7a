"""Host logic of bench.py (CPU): the strong-scaling split (every request of the
global batch on exactly one rank, rows balanced) and the per-step statistics."""
import numpy as np
import torch

import bench
from paper_2512_22420_b200 import dist as njdist
from synth.inputs import make_batch


def test_strong_scaling_split_reassembles_the_batch():
    b = make_batch(37, "mixed:5", V=64, d=16, seed=3)
    for ws in (1, 2, 3, 4, 8):
        parts = [bench.sub_batch(b, *njdist.split_requests(b.gamma, ws, r)) for r in range(ws)]
        assert sum(p.B for p in parts) == b.B
        assert np.array_equal(np.concatenate([p.gamma for p in parts]), b.gamma)
        assert torch.equal(torch.cat([p.hidden for p in parts]), b.hidden)
        assert torch.equal(torch.cat([p.uniforms for p in parts]), b.uniforms)
        assert torch.equal(torch.cat([p.draft_tokens for p in parts]), b.draft_tokens)
        G = [p.G for p in parts]
        assert torch.equal(torch.cat([p.draft_probs[:g] for p, g in zip(parts, G)]), b.draft_probs[:b.G])
        rows = [p.N for p in parts]
        assert max(rows) - min(rows) <= 2 * 6   # balanced to within two requests' rows


def test_step_stats():
    s = bench.step_stats([1.0, 2.0, 3.0, 4.0, 10.0])
    assert s["median"] == 3.0 and s["n"] == 5 and s["p10"] < s["median"] < s["p90"]
