"""Multi-process (torch.distributed, gloo, world_size 2-4) CPU tests of the
N > 1 paths' host logic and exchange protocol:

* request-sharded mode: the row-balanced request split covers every request
  exactly once and the max-over-ranks timing reduce;
* NCCL bootstrap plumbing: rank 0's bytes reach every rank (broadcast);
* vocab-sharded mode: the exchange protocol (oracle/sharded_ref.py, the
  arithmetic libnj's sharded kernels implement) run by real ranks that
  all_gather / all_reduce(MAX) over gloo reproduces the UNSHARDED fp64
  oracle's decisions (single-process loop for G = 1..8 as well).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from oracle import sharded_ref
from paper_2512_22420_b200 import dist as njdist
from synth.inputs import make_batch


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batch(seed=3, B=7, V=600, d=32):
    return make_batch(B, "mixed:4", V=V, d=d, seed=seed, q_vocab=V - 9)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        # request split + max-over-ranks
        gamma = np.array([0, 5, 1, 3, 2, 2, 4, 0, 1, 5, 3], np.int32)
        out["split"] = njdist.split_requests(gamma, world, rank)
        out["tmax"] = njdist.max_over_ranks(1.0 + rank)
        # bootstrap bytes
        out["uid"] = njdist.broadcast_bytes(b"nccl-id-%d" % 42 if rank == 0 else None)
        # sharded exchange protocol over gloo
        b = _batch()
        n = b.to_numpy()

        def gather(a):
            t = torch.from_numpy(np.ascontiguousarray(a))
            lst = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(lst, t)
            return [x.numpy() for x in lst]

        def allmax(a):
            t = torch.from_numpy(np.ascontiguousarray(a).astype(np.int64))
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return t.numpy().astype(np.int32)

        acc, tok = sharded_ref.rank_step(rank, world, n["hidden_bits"], n["W_bits"], n["draft_tokens"],
                                         n["draft_probs"], n["gamma"], n["uniforms"], gather, allmax)
        out["acc"], out["tok"] = acc, tok
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_multirank(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # request split: contiguous, disjoint, covering
    spans = [res[r]["split"] for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == 11
    assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
    assert all(res[r]["tmax"] == float(world) for r in range(world))
    assert all(res[r]["uid"] == b"nccl-id-42" for r in range(world))
    # every rank holds identical outputs == the unsharded oracle (ties excused)
    b = _batch()
    n = b.to_numpy()
    ref = oracle.verify(n["hidden_bits"], n["W_bits"], n["draft_tokens"], n["draft_probs"], n["gamma"],
                        n["uniforms"])
    ok = ~ref["tie"]
    for r in range(world):
        assert (res[r]["acc"] == res[0]["acc"]).all() and (res[r]["tok"] == res[0]["tok"]).all()
        assert (res[r]["acc"][ok] == ref["accept_len"][ok]).all()
        assert (res[r]["tok"][ok] == ref["next_token"][ok]).all()


@pytest.mark.parametrize("G", [1, 2, 4, 5, 8])
def test_sharded_protocol_threads(G):
    """Same protocol with G ranks as threads and an in-process collective."""
    import threading
    for seed in range(3):
        b = make_batch(9, "mixed:5", V=1100, d=24, seed=seed + 10 * G, q_vocab=1090)
        n = b.to_numpy()
        args = (n["hidden_bits"], n["W_bits"], n["draft_tokens"], n["draft_probs"], n["gamma"], n["uniforms"])
        bar = threading.Barrier(G)
        slots = [None] * G
        res = [None] * G

        def coll(rank, a, red):
            bar.wait()
            slots[rank] = a
            bar.wait()
            out = red(list(slots))
            bar.wait()
            return out

        def body(rank):
            gather = lambda a: coll(rank, a, lambda xs: xs)
            allmax = lambda a: coll(rank, a, lambda xs: np.max(np.stack(xs), axis=0))
            res[rank] = sharded_ref.rank_step(rank, G, *args, gather, allmax)

        th = [threading.Thread(target=body, args=(r,)) for r in range(G)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        ref = oracle.verify(*args)
        ok = ~ref["tie"]
        for acc, tok in res:
            assert (acc[ok] == ref["accept_len"][ok]).all()
            assert (tok[ok] == ref["next_token"][ok]).all()


def test_split_requests_balanced():
    g = np.array([5] * 10 + [0] * 30, np.int32)
    for world in (1, 2, 4, 8):
        spans = [njdist.split_requests(g, world, r) for r in range(world)]
        rows = [int((g[a:b] + 1).sum()) for a, b in spans]
        assert sum(rows) == int((g + 1).sum())
        assert max(rows) - min(rows) <= 6 + 1


@pytest.mark.parametrize("G", [2, 4])
def test_sharded_protocol_zero_residual_mass(G):
    """R6 across shards: q_0 = p_0 rounded UP to fp32 (so max(0, p - q) == 0
    everywhere) and u_0 = 1 (forced rejection): every rank switches to p_0 with
    masses e^{lse_r(0) - M}, and the drawn token equals the unsharded oracle's
    (which draws from p_0, R6)."""
    import threading
    import scipy.special
    for seed in range(3):
        b = make_batch(1, 1, V=700, d=24, seed=seed + 50)
        n = b.to_numpy()
        from oracle.verify_np import bf16_to_f64
        p0 = scipy.special.softmax(bf16_to_f64(n["hidden_bits"][:1]) @ bf16_to_f64(n["W_bits"]).T, axis=1)[0]
        q = np.nextafter(p0.astype(np.float32), np.float32(2.0)).reshape(1, -1)
        u = np.array([1.0, 0.1 + 0.25 * seed])
        args = (n["hidden_bits"], n["W_bits"], n["draft_tokens"], q, n["gamma"], u)
        ref = oracle.verify(*args)
        assert ref["flags"][0] & oracle.F_ZERO_MASS and ref["accept_len"][0] == 0
        bar = threading.Barrier(G)
        slots = [None] * G
        res = [None] * G

        def coll(rank, a, red):
            bar.wait()
            slots[rank] = a
            bar.wait()
            out = red(list(slots))
            bar.wait()
            return out

        def body(rank):
            gather = lambda a: coll(rank, a, lambda xs: xs)
            allmax = lambda a: coll(rank, a, lambda xs: np.max(np.stack(xs), axis=0))
            res[rank] = sharded_ref.rank_step(rank, G, *args, gather, allmax)

        th = [threading.Thread(target=body, args=(r,)) for r in range(G)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for acc, tok in res:
            assert acc[0] == 0 and tok[0] == ref["next_token"][0]
