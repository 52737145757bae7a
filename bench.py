#!/usr/bin/env python
"""bench.py — verified positions/s of batched speculative-decoding verification
(Nightjar's data-parallel hot path, arXiv 2512.22420) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl nj|reference]

A step = one nj_verify over one packed batch (LM-head GEMM + online softmax +
Leviathan rejection sampling, all in libnj's kernels), inputs resident in HBM.
Default workload = BASELINE.json configs[1] (C2): Qwen-7B shape d=3584,
V=152064, B=8, gamma=3.  N > 1 (torchrun): request-sharded weak scaling, every
rank verifies its own batch, no collective on the data path; time = max over
ranks.  Prints ONE JSON line on rank 0.

--impl reference runs the fp64 oracle (oracle/, the only reference this tier
has) on the host cores: each step is a bounded sample (one request of the
batch) of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "verified positions/s"
UNIT = "positions/s"
V_Q, D_Q = 152064, 3584

CONFIGS = {
    # name: (B, gamma, path)   gamma may be "mixed:5"
    "c2": (8, 3, "auto"),                 # BASELINE configs[1]
    "c1": (1, 3, "auto"),                 # toy shape at Qwen scale (B=1)
    "c3_b64_g3": (64, 3, "auto"),
    "c3_b256_g2": (256, 2, "auto"),
    "c3_b256_g5": (256, 5, "auto"),
    "c3_b256_mixed": (256, "mixed:5", "auto"),
    "c3_b16_g2": (16, 2, "auto"),
    "c3_b12_g3": (12, 3, "auto"),
    "c3_b8_g5": (8, 5, "auto"),
    "c5": (256, 2, "auto"),                # BASELINE configs[4] (vocab-sharded run: bench_c5)
}


_OUT = None   # the real stdout: result lines only (stray library output goes to stderr)


def emit(obj):
    print(json.dumps(obj), file=_OUT or sys.stdout, flush=True)


def _claim_stdout():
    """Route fd 1 to stderr for the rest of the run (NCCL prints its version
    banner to stdout) and keep the original stdout for the JSON lines."""
    global _OUT
    sys.stdout.flush()
    _OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


def tensor_roof(name, flops, kern_ms, tf_burst, tf_sust):
    """Roofline entry of a tensor-bound GEMM.  The kernel is timed inside the repeated
    step loop (K back-to-back steps, the SM clock under sw_power_cap: see `clocks`), so
    its peak is MEASURED_PEAKS' sustained bf16 figure (cuBLAS back to back for 4 s);
    the burst figure (a kernel timed alone) is kept beside it."""
    a = flops / (kern_ms / 1e3) / 1e12
    return {"kernel": name, "bound": "tensor", "achieved": a, "peak": tf_sust, "unit": "TFLOP/s",
            "frac": a / tf_sust, "peak_kind": "sustained (kernel timed inside the back-to-back step loop)",
            "peak_burst": tf_burst, "frac_burst": a / tf_burst, "algorithmic_flops_per_launch": flops}


class ClockSampler:
    """NVML SM clock + throttle reasons sampled during the timed region."""
    NAMES = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
             0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, index: int, period: float = 0.005):
        self.samples, self.reasons, self.stop = [], set(), threading.Event()
        self.period = period
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover
            self.nv = None
            self.max_mhz = None

    def _run(self):
        while not self.stop.is_set():
            self._sample()
            time.sleep(self.period)

    def _sample(self):
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for bit, name in self.NAMES.items():
                if r & bit:
                    self.reasons.add(name)
        except Exception:
            pass

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._sample()
            self.stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def spawn_ranks(n: int) -> int:
    """`python bench.py --gpus N` without a launcher: start N ranks with
    torch.distributed.run on this node (127.0.0.1, a free port); rank 0 prints
    the JSON line.  Returns the launcher's exit code."""
    import socket
    import subprocess
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def bench_reference(args, ws, rank):
    """Oracle arm: fp64 CPU oracle, one request of the configured batch per step."""
    if ws > 1 and rank != 0:
        return
    import numpy as np

    import oracle
    from synth.inputs import make_batch, make_weight

    metric, unit = METRIC, UNIT
    Vr, dr = V_Q, D_Q
    if args.config == "propose":                       # draft proposal row
        B, gamma, Vr, dr = 64, 0, 151936, 896
        metric, unit = "proposed tokens/s (draft LM head + softmax + inverse-CDF draw)", "proposed tokens/s"
    elif args.config.startswith("greedy"):             # greedy verification row
        B, gamma = (8, 3) if args.config == "greedy_c2" else (256, 5)
        metric = "verified positions/s (greedy target)"
    elif args.config == "c4":                          # the trace's largest batch shape
        B, gamma = 256, "mixed:5"
    else:
        B, gamma, _ = CONFIGS[args.config]
    W = make_weight(Vr, dr, args.seed + (9 if args.config == "propose" else 0))
    b = make_batch(B, gamma, V=Vr, d=dr, seed=args.seed, W=W)
    n = b.to_numpy()
    g = n["gamma"]
    ro = np.concatenate([[0], np.cumsum(g + 1)])
    do = np.concatenate([[0], np.cumsum(g)])

    def one(i):
        k = i % B
        sl = slice(ro[k], ro[k + 1])
        if args.config == "propose":
            oracle.propose(n["hidden_bits"][sl], n["W_bits"], n["uniforms"][sl])
        elif args.config.startswith("greedy"):
            oracle.verify_greedy(n["hidden_bits"][sl], n["W_bits"], n["draft_tokens"][do[k]:do[k + 1]], g[k:k + 1])
        else:
            oracle.verify(n["hidden_bits"][sl], n["W_bits"], n["draft_tokens"][do[k]:do[k + 1]],
                          n["draft_probs"][do[k]:do[k + 1]] if g[k] else n["draft_probs"][:1], g[k:k + 1],
                          n["uniforms"][sl])
        return int(g[k]) + 1

    for i in range(args.warmup):
        one(i)
    t0 = time.perf_counter()
    pos = sum(one(i) for i in range(args.steps))
    dt = time.perf_counter() - t0
    val = pos / dt
    line = {"impl": "reference", "metric": metric, "value": val, "unit": unit, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"qwen7b_{args.config}", "B": B, "gamma": gamma, "d": dr, "V": Vr,
                       "step": "one request of the batch (bounded sample)"},
            "cpu_baseline": {"value": val, "unit": unit, "cores": oracle.max_threads(), "kind": "oracle",
                             "sample": f"{args.steps} single-request steps of the {args.config} batch"},
            "e2e": {"value": val, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


def cpu_baseline(b, budget_s: float, max_requests: int | None = None):
    """Oracle on the bounded sample: the batch (or its first max_requests
    requests), repeated up to budget_s."""
    import numpy as np

    import oracle
    n = b.to_numpy()
    g = n["gamma"]
    k = len(g) if max_requests is None else min(len(g), max_requests)
    nr, nd = int((g[:k] + 1).sum()), int(g[:k].sum())
    args = (n["hidden_bits"][:nr], n["W_bits"], n["draft_tokens"][:nd],
            n["draft_probs"][:max(nd, 1)], g[:k], n["uniforms"][:nr])
    runs, t0 = 0, time.perf_counter()
    while True:
        oracle.verify(*args)
        runs += 1
        if time.perf_counter() - t0 > budget_s or runs >= 20:
            break
    dt = time.perf_counter() - t0
    # per-core figure: one thread on the first request only
    nr1, nd1 = int(g[0] + 1), int(g[0])
    t1 = time.perf_counter()
    oracle.verify(n["hidden_bits"][:nr1], n["W_bits"], n["draft_tokens"][:nd1], n["draft_probs"][:max(nd1, 1)],
                  g[:1], n["uniforms"][:nr1], nthreads=1)
    dt1 = time.perf_counter() - t1
    return {"value": nr * runs / dt, "unit": UNIT, "cores": oracle.max_threads(), "kind": "oracle",
            "cpu_model": cpu_model(), "per_core_value": nr1 / dt1,
            "sample": f"{runs} full run(s) of {k} request(s) of the {b.B}-request batch ({nr} positions), {dt:.1f} s; "
                      f"per core: 1 thread, 1 request ({nr1} positions), {dt1:.1f} s"}


def sub_batch(b, b0: int, b1: int):
    """Requests [b0, b1) of a packed batch as their own packed batch (contiguous
    copies): the row-balanced share of one rank in the strong-scaling mode."""
    import numpy as np

    from synth.inputs import Batch
    g = b.gamma
    ro = np.concatenate([[0], np.cumsum(g + 1)])
    do = np.concatenate([[0], np.cumsum(g)])
    G = int(do[b1] - do[b0])
    q = b.draft_probs[do[b0]:do[b1]].contiguous() if G else b.draft_probs[:1].contiguous()
    return Batch(b.hidden[ro[b0]:ro[b1]].contiguous(), b.W, b.draft_tokens[do[b0]:do[b1]].contiguous(), q,
                 np.ascontiguousarray(g[b0:b1]), b.uniforms[ro[b0]:ro[b1]].contiguous())


def step_stats(ms):
    """median / p10 / p90 / mean of per-step device times (ms)."""
    import numpy as np
    a = np.asarray(ms, np.float64)
    if a.size == 0:
        return None
    return {"median": float(np.median(a)), "p10": float(np.percentile(a, 10)), "p90": float(np.percentile(a, 90)),
            "mean": float(a.mean()), "n": int(a.size)}


def timed_steps(run_step, steps: int, stream, local: int):
    """Time `steps` calls of run_step(i) on `stream` with CUDA events: one event
    before the first and one after every step (so per-step device times come
    from consecutive events), NVML clocks sampled meanwhile.  Returns
    (total_ms, per_step_ms, clock summary)."""
    import torch
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    with ClockSampler(local) as clk:
        ev[0].record(stream)
        for i in range(steps):
            run_step(i)
            ev[i + 1].record(stream)
        torch.cuda.synchronize()
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    return ev[0].elapsed_time(ev[-1]), per, clk.summary()


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def bench_nj(args, ws, rank, local):
    import numpy as np
    import torch

    from paper_2512_22420_b200 import NJ_OPT_PATH, NJ_OPT_PROFILE, NJ_PATH_FUSED, NJ_PATH_STAGED, Verifier
    from paper_2512_22420_b200 import dist as njdist
    from synth.inputs import make_batch, make_weight

    # more ranks than GPUs (a 1-GPU box exercising the N > 1 code path): ranks share
    # the devices round-robin and the host-side plumbing runs over gloo; the timing
    # is then contended and is flagged, never a scaling number
    ndev = torch.cuda.device_count()
    over = ws > ndev
    local = local % ndev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cdev = None if over else dev   # device of the plumbing collectives' tensors
    if ws > 1:
        import torch.distributed as dist
        if over:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    B, gamma, path = CONFIGS[args.config]
    path = PATH_NAMES.index(args.path or path)
    strong = args.scaling == "strong" and ws > 1
    W = make_weight(V_Q, D_Q, args.seed, dev)
    nb = 4   # rotating independent batches
    if strong:
        # one global batch per step, identical on every rank; each rank verifies its
        # row-balanced contiguous share (no data-path collective)
        full = [make_batch(B, gamma, V=V_Q, d=D_Q, seed=args.seed * 1000 + i, device=dev, W=W) for i in range(nb)]
        batches = []
        for bf in full:
            b0, b1 = njdist.split_requests(bf.gamma, ws, rank)
            batches.append(sub_batch(bf, b0, b1))
        N_global = full[0].N
        del full
    else:
        batches = [make_batch(B, gamma, V=V_Q, d=D_Q, seed=args.seed * 1000 + rank * 16 + i, device=dev, W=W)
                   for i in range(nb)]
        N_global = batches[0].N * ws
    Bl = batches[0].B
    gmax = max([int(b.gamma.max()) for b in batches if b.B] + [1])
    v = Verifier(D_Q, V_Q, max_batch=max(Bl, 1), gamma_max=max(gmax, 1), device=local)
    v.set_option(NJ_OPT_PATH, path)
    if args.temperature != 1.0:
        v.set_temperature(args.temperature)   # target softmax(l / T)
    p_used, launches = v.plan(batches[0].gamma) if Bl else (0, 0)
    acc = [torch.empty(max(Bl, 1), dtype=torch.int32, device=dev) for _ in range(nb)]
    nxt = [torch.empty(max(Bl, 1), dtype=torch.int32, device=dev) for _ in range(nb)]
    stream = torch.cuda.current_stream()

    def step(i):
        b = batches[i % nb]
        if b.B:
            v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc[i % nb], nxt[i % nb])

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    # eager pass: the dominant kernel bracketed by CUDA events on the launch stream
    v.set_option(NJ_OPT_PROFILE, 1)
    v.kernel_time(reset=True)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms_eager, per_eager, clk = timed_steps(step, args.steps, stream, local)
    kms, kn = v.kernel_time(reset=True)
    v.set_option(NJ_OPT_PROFILE, 0)
    ms, per, graph_ok = ms_eager, per_eager, False
    if not args.no_graph and Bl:
        # the same steps replayed from CUDA graphs (one per rotating batch; nj_verify does
        # no host synchronisation, so a call is capturable): no per-launch host overhead
        try:
            graphs = []
            cap = torch.cuda.Stream()
            cap.wait_stream(stream)
            with torch.cuda.stream(cap):
                for j in range(nb):
                    step(j)          # warm the capture stream
                cap.synchronize()
                for j in range(nb):
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=cap):
                        step(j)
                    graphs.append(g)
            stream.wait_stream(cap)
            for i in range(args.warmup):
                graphs[i % nb].replay()
            torch.cuda.synchronize()
            if ws > 1:
                dist.barrier()
            torch.cuda.synchronize()
            ms, per, clk = timed_steps(lambda i: graphs[i % nb].replay(), args.steps, stream, local)
            graph_ok = True
        except Exception as e:   # graph capture unavailable: keep the eager timing
            print(f"[bench] CUDA graph timing skipped: {e}", file=sys.stderr)
    if ws > 1:
        dist.barrier()
    # accepted tokens in the timed steps (the last outputs of each rotating batch)
    per_batch = []
    for j in range(nb):
        a = acc[j][:Bl].cpu().numpy()
        per_batch.append((int((a + 1).sum()), int((a < batches[j].gamma).sum())))
    acc_tok = sum(per_batch[i % nb][0] for i in range(args.steps))
    rejected = sum(per_batch[i % nb][1] for i in range(args.steps))
    N, G = batches[0].N, batches[0].G
    t_max = njdist.max_over_ranks(ms, cdev)
    tok_all = acc_tok
    if ws > 1:
        t = torch.tensor([float(acc_tok)], dtype=torch.float64, device=cdev)
        dist.all_reduce(t)
        tok_all = float(t.item())
    value = N_global * args.steps / (t_max / 1e3)
    hbm, tf_burst, tf_sust, peak_src = load_peaks()
    # roofline of the dominant kernel (DESIGN.md §5 / §8): fused path -> HBM bytes;
    # staged -> the one GEMM pass over N rows; two-pass -> K-A over the G draft rows.
    # A GEMM over R rows is HBM-bound below the ridge (R < peak_flops / hbm_bw
    # ~ 248 rows: algorithmic bytes = W + H) and tensor-bound above (2 R V d flops).
    kern_ms = kms / max(kn, 1)
    R_avg = rejected / args.steps
    ridge = tf_burst * 1e12 / (hbm * 1e9)
    if p_used == NJ_PATH_FUSED:
        byts = 2 * V_Q * D_Q + 2 * N * D_Q + 4 * R_avg * V_Q + 8 * G + 4 * N
        achieved = byts / (kern_ms / 1e3) / 1e9
        roof = {"kernel": "k_fused_verify", "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "algorithmic_bytes_per_launch": byts}
    else:
        R = N if p_used == NJ_PATH_STAGED else G / max(kn // args.steps, 1)
        name = "k_lmhead<logits,stats,capture> (staged, all N rows)" if p_used == NJ_PATH_STAGED else \
            "k_gemm_big<stats,capture> (K-A, draft rows)"
        if R < ridge:
            byts = 2 * V_Q * D_Q + 2 * R * D_Q
            achieved = byts / (kern_ms / 1e3) / 1e9
            roof = {"kernel": name, "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                    "frac": achieved / hbm, "algorithmic_bytes_per_launch": byts, "rows": R}
        else:
            roof = tensor_roof(name, 2.0 * R * V_Q * D_Q, kern_ms, tf_burst, tf_sust)
            roof["rows"] = R
    roof["peak_source"] = peak_src
    roof["kernel_ms_avg"] = kern_ms
    # share of the step in the SAME (eager, event-bracketed) pass the kernel was timed in
    roof["kernel_share_of_step"] = kms / ms_eager if ms_eager > 0 else None
    traffic_file = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    roof["traffic"] = None
    if os.path.exists(traffic_file):
        roof["traffic"] = json.load(open(traffic_file)).get(args.config, {}).get(roof["kernel"].split()[0])
    # end-to-end through the host API (pinned host buffers, copies inside the timed region)
    e2e = None
    if Bl:
        b = batches[0]
        pin = lambda t: t.cpu().pin_memory()
        hh, th, qh, uh = pin(b.hidden), pin(b.draft_tokens), pin(b.draft_probs), pin(b.uniforms)
        ah = torch.empty(Bl, dtype=torch.int32).pin_memory()
        nh = torch.empty(Bl, dtype=torch.int32).pin_memory()
        k_e2e = max(5, min(args.steps, 50))
        for _ in range(3):
            v.verify_host(hh, W, th, qh, b.gamma, uh, ah, nh)
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(k_e2e):
            v.verify_host(hh, W, th, qh, b.gamma, uh, ah, nh)
        s1.record(stream)
        torch.cuda.synchronize()
        e_ms = njdist.max_over_ranks(s0.elapsed_time(s1), cdev)
        # bytes that cross the host link per step: the copied hidden / tokens / uniforms,
        # plus the draft-probability bytes the kernels read in place (zero copy):
        # q_i(x_i) of every draft and the sample row of every rejected request
        # (+ the likely sample rows nj_verify_host staged over the copy stream during the
        # GEMM, NJ_OPT_Q_STAGE_ROWS; a rejected request's row is read in place only when
        # it was not staged).  Every e2e step verifies the same batch, so the last call's
        # outputs and staged rows are every step's.
        staged = set(int(r) for r in v.host_staged_rows())
        gam = np.asarray(b.gamma)
        g0 = np.concatenate([[0], np.cumsum(gam)[:-1]])
        an = ah.numpy()
        rej_rows = [int(g0[i] + an[i]) for i in range(Bl) if an[i] < gam[i]]
        inplace_rows = sum(1 for r in rej_rows if r not in staged)
        h2d = (b.hidden.numel() * 2 + b.draft_tokens.numel() * 4 + b.N * 4 + b.G * 4
               + (len(staged) + inplace_rows) * V_Q * 4)
        e2e = {"value": N_global * k_e2e / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(2 * Bl * 4), "steps": k_e2e, "api": "nj_verify_host",
               "q_rows": (f"{len(staged)} likely sample rows staged to the device during the GEMM, "
                          f"{inplace_rows} rejected rows read in place from pinned host memory"
                          if staged else "read in place from pinned host memory (NJ_OPT_Q_ZERO_COPY)")}
    if ws > 1:
        dist.barrier()
    if rank != 0:
        dist.destroy_process_group()
        return
    cpu = None if args.no_cpu_baseline else cpu_baseline(_cpu_batch(batches[0]), args.cpu_budget)
    scaling = "strong" if strong else "weak"
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"qwen7b_{args.config}" + (f"_T{args.temperature:g}" if args.temperature != 1.0 else ""),
                       "temperature": args.temperature, "B": B, "gamma": gamma, "N_per_step": N_global,
                       "N_per_rank_rank0": N, "d": D_Q, "V": V_Q, "global_batch": B * (1 if strong else ws),
                       "path": PATH_NAMES[p_used],
                       "parallelism": (f"request-sharded x{ws}, " + ("one global batch split by rows"
                                                                     if strong else "own batch per rank")
                                       + " (no data-path collective)"),
                       "l2": "inputs larger than L2: W_lm (1.09 GB > 126 MB L2) streamed from HBM every step; "
                             "4 rotating batches",
                       "launch": "CUDA graph replay per step" if graph_ok else "eager launches",
                       "ms_per_step_eager": ms_eager / args.steps},
            "step_ms": step_stats(per), "step_ms_eager": step_stats(per_eager),
            "accepted_tokens_per_s": tok_all / (t_max / 1e3),
            "realised_tokens_per_request": acc_tok / (args.steps * max(Bl, 1)),
            "oversubscribed": (f"{ws} ranks on {ndev} GPU(s): ranks share devices, timing contended "
                               "(code-path check, not a scaling number)") if over else None,
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
            "gpu_launches": int(launches * args.steps)}
    emit(line)
    if ws > 1:
        dist.destroy_process_group()


# batch sizes a continuous-batching server captures CUDA graphs for (vLLM's
# default capture sizes up to 256): the C4 trace pads B_t up to one of them
GRAPH_BUCKETS = [1, 2, 4] + list(range(8, 257, 8))


def load_cprefill(args):
    """c_prefill(L_max, B) table for the bandit (Eq. 3): the B200 measurement of
    scripts/measure_cprefill.py when present (profiles/r02_cprefill_b200.csv),
    else PAPER Table 1 (RTX 4090, tests/golden/table1_cprefill.csv) x
    --cprefill-scale.  Returns (len_buckets, batch_buckets, cost_ms, source)."""
    import numpy as np
    meas = os.path.join(ROOT, "profiles", "r02_cprefill_b200.csv")
    if os.path.exists(meas) and not args.cprefill_table1:
        # the reward here is the VERIFICATION step's goodput, ~14x the full serving
        # step's (the LM head is ~7 % of a 7B target forward); Eq. 3's
        # switching term is scaled by the same factor so the two terms keep the
        # proportion they have with full-step rewards (Eq. 3 verbatim otherwise)
        path, scale = meas, args.cprefill_b200_scale
        src = f"B200-measured draft KV-reconstruction prefill (profiles/r02_cprefill_b200.csv) x {scale}"
    else:
        path, scale = os.path.join(ROOT, "tests", "golden", "table1_cprefill.csv"), args.cprefill_scale
        src = f"PAPER Table 1 (RTX 4090) x {scale}"
    rows = [l.strip().split(",") for l in open(path) if l[0].isdigit()]
    L = sorted({int(r[0]) for r in rows})
    Bb = sorted({int(r[1]) for r in rows})
    C = np.zeros((len(L), len(Bb)))
    for r in rows:
        C[L.index(int(r[0])), Bb.index(int(r[1]))] = float(r[2]) * scale
    return L, Bb, C, src


def bench_c4(args, ws, rank, local):
    """BASELINE configs[3]: Nightjar-driven trace.  B_t follows a synthetic QPS
    ramp 5 -> 300 -> 5 over --trace-steps steps (fig:trace1 shape),
    padded up to the server's CUDA-graph batch buckets; gamma_t =
    nj_select_gamma(B_t, L_max) (Algorithm 1 + Eq. 3 with the c_prefill table
    of load_cprefill); every step replays the CUDA graph of nj_verify for
    (B_t, gamma_t) on the first B_t requests of a pre-generated pool, is timed
    with CUDA events, and feeds the realised goodput sum(n_b + 1) / t_step back
    through nj_observe.  Reported: accepted tokens/s over
    the trace, and gamma histograms per B range split into exploration and
    exploitation bins (Algorithm 1's bin type), whose exploitation means show
    gamma* falling as load rises."""
    import numpy as np
    import torch

    from paper_2512_22420_b200 import Bandit, Verifier
    from synth.inputs import make_batch, make_weight, qps_ramp

    if ws > 1 and rank != 0:
        return
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    BMAX, GMAX = 256, 5
    W = make_weight(V_Q, D_Q, args.seed, dev)
    pools = {g: make_batch(BMAX, g, V=V_Q, d=D_Q, seed=args.seed * 100 + g, device=dev, W=W) for g in range(GMAX + 1)}
    v = Verifier(D_Q, V_Q, max_batch=BMAX, gamma_max=GMAX, device=local)
    L, Bb, C, csrc = load_cprefill(args)
    bandit = Bandit(GMAX, BMAX, args.seed, L, Bb, C)
    trace = qps_ramp(args.trace_steps, seed=args.seed)
    if args.c4_buckets == "graph":
        trace = np.array([min(x for x in GRAPH_BUCKETS if x >= int(B)) for B in trace], np.int32)
    acc = torch.empty(BMAX, dtype=torch.int32, device=dev)
    nxt = torch.empty(BMAX, dtype=torch.int32, device=dev)
    acc_h = torch.empty(BMAX, dtype=torch.int32).pin_memory()
    stream = torch.cuda.current_stream()
    cap = torch.cuda.Stream()
    graphs = {}

    def launch(B, g):
        b = pools[g]
        n_rows, n_dr = B * (g + 1), B * g
        gam = np.full(B, g, np.int32)
        v.verify(b.hidden[:n_rows], W, b.draft_tokens[:n_dr], b.draft_probs[:max(n_dr, 1)], gam,
                 b.uniforms[:n_rows], acc, nxt)

    def graph_for(B, g):
        key = (B, g)
        if key not in graphs and not args.no_graph:
            try:
                cap.wait_stream(stream)
                with torch.cuda.stream(cap):
                    launch(B, g)
                    cap.synchronize()
                    gr = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(gr, stream=cap):
                        launch(B, g)
                stream.wait_stream(cap)
                graphs[key] = gr
            except Exception as e:   # pragma: no cover
                print(f"[bench] c4 graph capture failed: {e}", file=sys.stderr)
                graphs[key] = None
        return graphs.get(key)

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lag, tok_tot, t_tot, pos_tot = 0, 0, 0.0, 0
    hist = {"explore": {}, "exploit": {}}
    sel_us, step_ms = [], []
    with ClockSampler(local) as clk:
        for t, B in enumerate(trace):
            B = int(B)
            t0 = time.perf_counter()
            g = bandit.select(B, lag if bandit.last_gamma == 0 else 0)
            sel_us.append((time.perf_counter() - t0) * 1e6)
            kind = "explore" if bandit.state(B)[4] == 1 else "exploit"
            gr = graph_for(B, g)
            e0.record(stream)
            if gr is not None:
                gr.replay()
            else:
                launch(B, g)
            e1.record(stream)
            acc_h[:B].copy_(acc[:B], non_blocking=True)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            toks = int((acc_h[:B] + 1).sum())
            bandit.observe(B, g, toks / (ms / 1e3))
            lag = lag + 1 if g == 0 else 0
            if t >= args.warmup:
                tok_tot += toks
                pos_tot += B * (g + 1)
                t_tot += ms / 1e3
                step_ms.append(ms)
                key = f"B{(B - 1) // 32 * 32 + 1}-{(B - 1) // 32 * 32 + 32}"
                hist[kind].setdefault(key, [0] * (GMAX + 1))[g] += 1
    keys = sorted(set(hist["explore"]) | set(hist["exploit"]), key=lambda k: int(k[1:].split("-")[0]))
    mean_exploit = {k: (float(np.dot(hist["exploit"][k], np.arange(GMAX + 1)) / sum(hist["exploit"][k]))
                        if k in hist["exploit"] and sum(hist["exploit"][k]) else None) for k in keys}
    # the bandit's learned greedy choice per graph bucket at the end of the trace (no switch cost)
    greedy = {}
    for Bq in GRAPH_BUCKETS:
        sc = [bandit.score(Bq, 1, gg) for gg in range(GMAX + 1)]
        if not all(np.isnan(sc)):
            greedy[str(Bq)] = int(np.nanargmin(sc))
    nsteps = len(step_ms)
    line = {"metric": "accepted tokens/s (bandit-driven trace)", "value": tok_tot / t_tot, "unit": "tokens/s",
            "n_gpus": 1, "steps": nsteps, "warmup": args.warmup,
            "ms_per_step": t_tot / nsteps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "qwen7b_c4_nightjar_trace", "qps": "5->300->5 linear ramp",
                       "trace_steps": int(len(trace)), "batch_buckets": args.c4_buckets,
                       "batch_max": BMAX, "gamma_max": GMAX, "cprefill": csrc,
                       "launch": "CUDA graph replay per (B, gamma)" if not args.no_graph else "eager launches"},
            "verified_positions_per_s": pos_tot / t_tot,
            "step_ms": step_stats(step_ms),
            "gamma_histogram_per_B": {"exploit": hist["exploit"], "explore": hist["explore"]},
            "mean_gamma_exploit_per_B": mean_exploit,
            "greedy_gamma_at_end_per_B": greedy,
            "select_gamma_us_median": statistics.median(sel_us),
            "graphs_captured": len(graphs), "clocks": clk.summary(),
            "bandit_snapshot_batches": len(bandit.snapshot()["batches"])}
    emit(line)


def bench_c5(args, ws, rank, local):
    """BASELINE configs[4]: vocab-sharded LM head (B=256, gamma=2) over the
    ranks of this job, libnj's own NCCL communicator for the three exchanges
    per step.  Strong scaling: the same batch on every rank,
    each rank streams V/G rows of W.  At N=1 the same code runs with a one-rank
    communicator."""
    import torch

    from paper_2512_22420_b200 import NJ_OPT_PROFILE, NJ_PATH_STAGED, NcclComm, Verifier, nccl_unique_id, shard_range
    from paper_2512_22420_b200 import dist as njdist
    from synth.inputs import make_batch, make_weight

    if ws > torch.cuda.device_count():
        # NCCL needs one device per rank: the vocab-sharded step cannot oversubscribe a GPU
        # (the request-sharded configs can); every rank stops, rank 0 reports
        if rank == 0:
            emit({"metric": METRIC, "config": {"workload": "qwen7b_c5_vocab_sharded"}, "n_gpus": ws,
                  "unavailable": f"c5 needs one GPU per rank (NCCL): {ws} ranks, "
                                 f"{torch.cuda.device_count()} GPU(s) visible"})
        return
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        comm = njdist.nccl_comm_for_world(local)
    else:
        comm = NcclComm(1, nccl_unique_id(), 0, local)
    B, g = 256, 2
    vb, ve = shard_range(V_Q, ws, rank)
    Wf = make_weight(V_Q, D_Q, args.seed, dev)
    b = make_batch(B, g, V=V_Q, d=D_Q, seed=args.seed, device=dev, W=Wf)
    # rotating copies of the rank's W shard so consecutive steps never find it in
    # L2 (126 MB): at G = 8 a shard is 136 MB, so one copy would be largely
    # L2-resident from the previous step
    L2_BYTES = 126 * 2 ** 20
    nW = 1 if (ve - vb) * D_Q * 2 > 2 * L2_BYTES else 3
    Ws = [Wf[vb:ve].contiguous() for _ in range(nW)]
    W = Ws[0]
    del Wf
    torch.cuda.empty_cache()
    v = Verifier(D_Q, V_Q, max_batch=B, gamma_max=g, device=local, v_begin=vb, v_end=ve, nccl_comm=comm.handle)
    _, launches = v.plan(b.gamma)
    acc = torch.empty(B, dtype=torch.int32, device=dev)
    nxt = torch.empty(B, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()

    def step(i=0):
        v.verify(b.hidden, Ws[i % nW], b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    v.set_option(NJ_OPT_PROFILE, 1)
    v.kernel_time(reset=True)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms_eager, per_eager, clk = timed_steps(step, args.steps, stream, local)
    ms, per = ms_eager, per_eager
    kms, kn = v.kernel_time(reset=True)
    v.set_option(NJ_OPT_PROFILE, 0)
    graph_ok = False
    if not args.no_graph:
        # one step (kernels + NCCL collectives on the stream) per W copy, replayed from CUDA graphs
        try:
            cap = torch.cuda.Stream()
            cap.wait_stream(stream)
            graphs = []
            with torch.cuda.stream(cap):
                step()
                cap.synchronize()
                for j in range(nW):
                    graph = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(graph, stream=cap):
                        step(j)
                    graphs.append(graph)
            stream.wait_stream(cap)
            for i in range(args.warmup):
                graphs[i % nW].replay()
            torch.cuda.synchronize()
            if ws > 1:
                dist.barrier()
            torch.cuda.synchronize()
            ms, per, clk = timed_steps(lambda i: graphs[i % nW].replay(), args.steps, stream, local)
            graph_ok = True
        except Exception as e:
            print(f"[bench] CUDA graph timing skipped: {e}", file=sys.stderr)
    t_max = njdist.max_over_ranks(ms, dev)
    toks = int((acc + 1).sum().item())
    hbm, tf_burst, tf_sust, peak_src = load_peaks()
    kern_ms = kms / max(kn, 1)
    staged = v.plan(b.gamma)[0] == NJ_PATH_STAGED   # the staged sharded step: k_lmhead over all N rows
    flops = 2.0 * (b.N if staged else b.G) * (ve - vb) * D_Q
    roof = tensor_roof("k_lmhead<logits,stats,capture> (all N rows, this rank's shard)" if staged else
                       "k_gemm_big<stats> (K-A, draft rows, this rank's shard)", flops, kern_ms, tf_burst, tf_sust)
    roof.update({"peak_source": peak_src, "kernel_ms_avg": kern_ms, "kernel_share_of_step": kms / ms_eager,
                 "traffic": None})
    # end to end through nj_verify_host (pinned host inputs, copies inside the timed region)
    pin = lambda t: t.cpu().pin_memory()
    hh, th, qh, uh = pin(b.hidden), pin(b.draft_tokens), pin(b.draft_probs), pin(b.uniforms)
    ah = torch.empty(B, dtype=torch.int32).pin_memory()
    nh = torch.empty(B, dtype=torch.int32).pin_memory()
    k_e2e = max(5, min(args.steps, 30))
    for _ in range(2):
        v.verify_host(hh, W, th, qh, b.gamma, uh, ah, nh)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for _ in range(k_e2e):
        v.verify_host(hh, W, th, qh, b.gamma, uh, ah, nh)
    s1.record(stream)
    torch.cuda.synchronize()
    e_ms = njdist.max_over_ranks(s0.elapsed_time(s1), dev)
    rej = int((acc.cpu().numpy() < b.gamma).sum())
    h2d = b.hidden.numel() * 2 + b.draft_tokens.numel() * 4 + b.N * 4 + b.G * 4 + rej * (ve - vb) * 4
    e2e = {"value": b.N * k_e2e / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": int(2 * B * 4), "steps": k_e2e, "api": "nj_verify_host",
           "q_rows": "read in place from pinned host memory (NJ_OPT_Q_ZERO_COPY); bytes per rank"}
    v.close()
    comm.close()
    if ws > 1:
        dist.barrier()
    if rank != 0:
        dist.destroy_process_group()
        return
    cpu = None if args.no_cpu_baseline else cpu_baseline(_cpu_batch(b), args.cpu_budget, max_requests=8)
    line = {"metric": METRIC, "value": b.N * args.steps / (t_max / 1e3), "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "qwen7b_c5_vocab_sharded", "B": B, "gamma": g, "N_per_step": b.N, "d": D_Q,
                       "V": V_Q, "V_per_rank_max": max(shard_range(V_Q, ws, r)[1] - shard_range(V_Q, ws, r)[0]
                                                      for r in range(ws)),
                       "parallelism": f"vocab-sharded x{ws} (4 NCCL collectives per step: allgather x3 + allreduce-MAX)",
                       "l2": (f"W shard {(ve - vb) * D_Q * 2 / 2 ** 20:.0f} MiB x {nW} rotating copies "
                              "(> L2 between reuses); streamed from HBM every step"),
                       "launch": "CUDA graph replay per step" if graph_ok else "eager launches",
                       "ms_per_step_eager": ms_eager / args.steps},
            "accepted_tokens_per_s": toks * args.steps / (t_max / 1e3),
            "step_ms": step_stats(per), "step_ms_eager": step_stats(per_eager),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
            "gpu_launches": int(launches * args.steps)}
    emit(line)
    if ws > 1:
        dist.destroy_process_group()


def bench_propose(args, ws, rank, local):
    """the draft-side proposal step (nj_propose) at a
    0.5B-style draft head (d = 896, V = 151936), B = 64 positions per step:
    draft LM head -> q rows -> inverse-CDF draws.  Metric: proposed tokens/s.
    Replicas only (each rank proposes for its own requests, no exchange)."""
    import numpy as np
    import torch

    import oracle
    from paper_2512_22420_b200 import NJ_OPT_PROFILE, Verifier
    from paper_2512_22420_b200 import dist as njdist
    from synth.inputs import make_batch, make_weight

    if ws > torch.cuda.device_count():
        # NCCL needs one device per rank: the vocab-sharded step cannot oversubscribe a GPU
        # (the request-sharded configs can); every rank stops, rank 0 reports
        if rank == 0:
            emit({"metric": METRIC, "config": {"workload": "qwen7b_c5_vocab_sharded"}, "n_gpus": ws,
                  "unavailable": f"c5 needs one GPU per rank (NCCL): {ws} ranks, "
                                 f"{torch.cuda.device_count()} GPU(s) visible"})
        return
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    DV, DD, B = 151936, 896, 64
    W = make_weight(DV, DD, args.seed + 9, dev)
    b = make_batch(B, 0, V=DV, d=DD, seed=args.seed + rank, device=dev, W=W)
    v = Verifier(DD, DV, max_batch=B, gamma_max=1, device=local)
    tok = torch.empty(B, dtype=torch.int32, device=dev)
    q = torch.empty(B, DV, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        v.propose(b.hidden, W, b.uniforms, tok, q)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    v.set_option(NJ_OPT_PROFILE, 1)
    v.kernel_time(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms_eager = e0.elapsed_time(e1)
    kms, kn = v.kernel_time(reset=True)
    v.set_option(NJ_OPT_PROFILE, 0)
    ms, graph_ok = ms_eager, False
    clk = None
    if not args.no_graph:
        try:
            cap = torch.cuda.Stream()
            cap.wait_stream(stream)
            with torch.cuda.stream(cap):
                step()
                cap.synchronize()
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph, stream=cap):
                    step()
            stream.wait_stream(cap)
            for _ in range(args.warmup):
                graph.replay()
            if ws > 1:
                dist.barrier()
            torch.cuda.synchronize()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with ClockSampler(local) as clk:
                g0.record(stream)
                for _ in range(args.steps):
                    graph.replay()
                g1.record(stream)
                torch.cuda.synchronize()
            ms, graph_ok = g0.elapsed_time(g1), True
        except Exception as e:
            print(f"[bench] CUDA graph timing skipped: {e}", file=sys.stderr)
    t_max = njdist.max_over_ranks(ms, dev) if ws > 1 else ms
    hbm, _, _, peak_src = load_peaks()
    kern_ms = kms / max(kn, 1)
    byts = 2 * DV * DD + 2 * B * DD + 4 * B * DV   # W once, hidden, fp32 logits written
    roof = {"kernel": "k_lmhead<logits,stats> (draft LM head)", "bound": "hbm",
            "achieved": byts / (kern_ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
            "frac": byts / (kern_ms / 1e3) / 1e9 / hbm, "algorithmic_bytes_per_launch": byts,
            "peak_source": peak_src, "kernel_ms_avg": kern_ms,
            "kernel_share_of_step": kms / ms_eager if ms_eager > 0 else None, "traffic": None}
    # end to end: pinned host hidden / uniforms in, tokens out (q stays on the device for nj_verify)
    hh, uh = b.hidden.cpu().pin_memory(), b.uniforms.cpu().pin_memory()
    th = torch.empty(B, dtype=torch.int32).pin_memory()
    hd, ud = torch.empty_like(b.hidden), torch.empty_like(b.uniforms)
    k_e2e = max(5, min(args.steps, 30))
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s0.record(stream)
    for _ in range(k_e2e):
        hd.copy_(hh, non_blocking=True)
        ud.copy_(uh, non_blocking=True)
        v.propose(hd, W, ud, tok, q)
        th.copy_(tok, non_blocking=True)
        stream.synchronize()
    s1.record(stream)
    torch.cuda.synchronize()
    e_ms = s0.elapsed_time(s1)
    e2e = {"value": B * k_e2e / (e_ms / 1e3), "unit": "proposed tokens/s", "h2d_bytes_per_step": int(B * DD * 2 + B * 4),
           "d2h_bytes_per_step": int(B * 4), "steps": k_e2e, "api": "nj_propose (torch pinned copies around it)"}
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        n = b.to_numpy()
        k = 2
        runs, t0 = 0, time.perf_counter()
        while True:
            oracle.propose(n["hidden_bits"][:k], n["W_bits"], n["uniforms"][:k])
            runs += 1
            if time.perf_counter() - t0 > min(args.cpu_budget, 10.0) or runs >= 20:
                break
        dt = time.perf_counter() - t0
        cpu = {"value": k * runs / dt, "unit": "proposed tokens/s", "cores": oracle.max_threads(), "kind": "oracle",
               "sample": f"{runs} run(s) of {k} of the {B} positions, {dt:.1f} s"}
    v.close()
    if ws > 1:
        dist.barrier()
        if rank != 0:
            dist.destroy_process_group()
            return
    line = {"metric": "proposed tokens/s (draft LM head + softmax + inverse-CDF draw)",
            "value": B * ws * args.steps / (t_max / 1e3), "unit": "proposed tokens/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "draft_propose_0.5b_head", "B": B, "d": DD, "V": DV,
                       "parallelism": f"replicas x{ws}", "l2": "inputs larger than L2 (W 272 MB streamed every step)",
                       "launch": "CUDA graph replay per step" if graph_ok else "eager launches",
                       "ms_per_step_eager": ms_eager / args.steps},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary() if clk else None,
            "gpu_launches": 4 * args.steps}
    emit(line)
    if ws > 1:
        dist.destroy_process_group()


def bench_greedy(args, ws, rank, local):
    """greedy verification (argmax target,
    nj_verify_greedy) at the Qwen shape, B = 8 (config greedy_c2) or B = 256,
    gamma = 5 (greedy_b256g5).  Metric: verified positions/s.  Replicas only."""
    import numpy as np
    import torch

    import oracle
    from paper_2512_22420_b200 import NJ_OPT_PROFILE, Verifier
    from paper_2512_22420_b200 import dist as njdist
    from synth.inputs import make_batch, make_weight

    if ws > torch.cuda.device_count():
        # NCCL needs one device per rank: the vocab-sharded step cannot oversubscribe a GPU
        # (the request-sharded configs can); every rank stops, rank 0 reports
        if rank == 0:
            emit({"metric": METRIC, "config": {"workload": "qwen7b_c5_vocab_sharded"}, "n_gpus": ws,
                  "unavailable": f"c5 needs one GPU per rank (NCCL): {ws} ranks, "
                                 f"{torch.cuda.device_count()} GPU(s) visible"})
        return
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    B, g = (8, 3) if args.config == "greedy_c2" else (256, 5)
    W = make_weight(V_Q, D_Q, args.seed, dev)
    b = make_batch(B, g, V=V_Q, d=D_Q, seed=args.seed + rank, device=dev, W=W)
    v = Verifier(D_Q, V_Q, max_batch=B, gamma_max=5, device=local)
    acc = torch.empty(B, dtype=torch.int32, device=dev)
    nxt = torch.empty(B, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    nblk = -(-b.N // 2048)   # k_lmhead blocks of <= kStagedMaxRows rows (argmax epilogue, no logits)

    def step():
        v.verify_greedy(b.hidden, W, b.draft_tokens, b.gamma, acc, nxt)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    v.set_option(NJ_OPT_PROFILE, 1)
    v.kernel_time(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms_eager = e0.elapsed_time(e1)
    kms, kn = v.kernel_time(reset=True)
    v.set_option(NJ_OPT_PROFILE, 0)
    ms, graph_ok, clk = ms_eager, False, None
    if not args.no_graph:
        try:
            cap = torch.cuda.Stream()
            cap.wait_stream(stream)
            with torch.cuda.stream(cap):
                step()
                cap.synchronize()
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph, stream=cap):
                    step()
            stream.wait_stream(cap)
            for _ in range(args.warmup):
                graph.replay()
            if ws > 1:
                dist.barrier()
            torch.cuda.synchronize()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with ClockSampler(local) as clk:
                g0.record(stream)
                for _ in range(args.steps):
                    graph.replay()
                g1.record(stream)
                torch.cuda.synchronize()
            ms, graph_ok = g0.elapsed_time(g1), True
        except Exception as e:
            print(f"[bench] CUDA graph timing skipped: {e}", file=sys.stderr)
    t_max = njdist.max_over_ranks(ms, dev) if ws > 1 else ms
    hbm, tf_burst, tf_sust, peak_src = load_peaks()
    kern_ms = kms / max(kn, 1)
    R = b.N / nblk
    ridge = tf_burst * 1e12 / (hbm * 1e9)
    if R < ridge:
        byts = 2 * V_Q * D_Q + 2 * R * D_Q
        roof = {"kernel": "k_lmhead<argmax> (all rows)", "bound": "hbm", "achieved": byts / (kern_ms / 1e3) / 1e9,
                "peak": hbm, "unit": "GB/s", "frac": byts / (kern_ms / 1e3) / 1e9 / hbm,
                "algorithmic_bytes_per_launch": byts}
    else:
        roof = tensor_roof("k_lmhead<argmax> (all rows)", 2.0 * R * V_Q * D_Q, kern_ms, tf_burst, tf_sust)
    roof.update({"peak_source": peak_src, "kernel_ms_avg": kern_ms,
                 "kernel_share_of_step": kms / ms_eager if ms_eager > 0 else None, "traffic": None, "rows": R})
    # end to end: pinned host hidden + draft tokens in, accept_len / next_token out
    hh, th = b.hidden.cpu().pin_memory(), b.draft_tokens.cpu().pin_memory()
    hd, td = torch.empty_like(b.hidden), torch.empty_like(b.draft_tokens)
    ah = torch.empty(B, dtype=torch.int32).pin_memory()
    nh = torch.empty(B, dtype=torch.int32).pin_memory()
    k_e2e = max(5, min(args.steps, 30))
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for _ in range(k_e2e):
        hd.copy_(hh, non_blocking=True)
        td.copy_(th, non_blocking=True)
        v.verify_greedy(hd, W, td, b.gamma, acc, nxt)
        ah.copy_(acc, non_blocking=True)
        nh.copy_(nxt, non_blocking=True)
        stream.synchronize()
    s1.record(stream)
    torch.cuda.synchronize()
    e_ms = s0.elapsed_time(s1)
    e2e = {"value": b.N * k_e2e / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(hh.numel() * 2 + th.numel() * 4),
           "d2h_bytes_per_step": int(2 * B * 4), "steps": k_e2e, "api": "nj_verify_greedy (torch pinned copies around it)"}
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        n = b.to_numpy()
        k = min(B, 4)
        nr, nd = int((n["gamma"][:k] + 1).sum()), int(n["gamma"][:k].sum())
        runs, t0 = 0, time.perf_counter()
        while True:
            oracle.verify_greedy(n["hidden_bits"][:nr], n["W_bits"], n["draft_tokens"][:nd], n["gamma"][:k])
            runs += 1
            if time.perf_counter() - t0 > min(args.cpu_budget, 10.0) or runs >= 20:
                break
        dt = time.perf_counter() - t0
        cpu = {"value": nr * runs / dt, "unit": UNIT, "cores": oracle.max_threads(), "kind": "oracle",
               "sample": f"{runs} run(s) of {k} of the {B} requests ({nr} positions), {dt:.1f} s"}
    v.close()
    if ws > 1:
        dist.barrier()
        if rank != 0:
            dist.destroy_process_group()
            return
    line = {"metric": "verified positions/s (greedy target)", "value": b.N * ws * args.steps / (t_max / 1e3),
            "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"qwen7b_greedy_B{B}_g{g}", "B": B, "gamma": g, "N_per_step": b.N, "d": D_Q,
                       "V": V_Q, "parallelism": f"replicas x{ws}", "gemm_blocks": nblk,
                       "l2": "inputs larger than L2 (W 1.09 GB streamed per block)",
                       "launch": "CUDA graph replay per step" if graph_ok else "eager launches",
                       "ms_per_step_eager": ms_eager / args.steps},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary() if clk else None,
            "gpu_launches": (2 * nblk + 1) * args.steps}
    emit(line)
    if ws > 1:
        dist.destroy_process_group()


PATH_NAMES = ["auto", "fused", "twopass", "staged"]


def bench_sweep(args, ws, rank, local):
    """BASELINE configs[2]: B x gamma sweep (C3); one JSON line per point."""
    import torch

    from paper_2512_22420_b200 import NJ_OPT_PATH, NJ_OPT_PROFILE, Verifier
    from synth.inputs import make_batch, make_weight

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    W = make_weight(V_Q, D_Q, args.seed, dev)
    hbm, tf_burst, tf_sust, _ = load_peaks()
    Bs = [int(x) for x in args.sweep_B.split(",")]
    Gs = [x if x.startswith("mixed") else int(x) for x in args.sweep_gamma.split(",")]
    for g in Gs:
        for B in Bs:
            b = make_batch(B, g, V=V_Q, d=D_Q, seed=args.seed + B, device=dev, W=W)
            v = Verifier(D_Q, V_Q, max_batch=B, gamma_max=5, device=local)
            if args.path:
                v.set_option(NJ_OPT_PATH, PATH_NAMES.index(args.path))
            try:
                path, launches = v.plan(b.gamma)
            except Exception as e:   # forced path not applicable at this point
                emit({"config": f"B{B}_g{g}", "skipped": str(e)})
                continue
            acc = torch.empty(B, dtype=torch.int32, device=dev)
            nxt = torch.empty(B, dtype=torch.int32, device=dev)
            for _ in range(3):
                v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            v.set_option(NJ_OPT_PROFILE, 1)
            v.kernel_time(True)
            e0.record()
            for _ in range(args.steps):
                v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.steps
            kms, kn = v.kernel_time(True)
            v.set_option(NJ_OPT_PROFILE, 0)
            # the same step replayed from a CUDA graph (the bench lines' launch mode)
            ms_graph = None
            if not args.no_graph:
                try:
                    cap = torch.cuda.Stream()
                    cap.wait_stream(torch.cuda.current_stream())
                    with torch.cuda.stream(cap):
                        v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
                        cap.synchronize()
                        gr = torch.cuda.CUDAGraph()
                        with torch.cuda.graph(gr, stream=cap):
                            v.verify(b.hidden, W, b.draft_tokens, b.draft_probs, b.gamma, b.uniforms, acc, nxt)
                    torch.cuda.current_stream().wait_stream(cap)
                    for _ in range(3):
                        gr.replay()
                    torch.cuda.synchronize()
                    e0.record()
                    for _ in range(args.steps):
                        gr.replay()
                    e1.record()
                    torch.cuda.synchronize()
                    ms_graph = e0.elapsed_time(e1) / args.steps
                    del gr
                except Exception as e:   # noqa: BLE001
                    print(f"[bench] sweep graph timing skipped: {e}", file=sys.stderr)
            toks = int((acc + 1).sum().item())
            N = b.N
            t_star = max(2.0 * N * V_Q * D_Q / (tf_burst * 1e12), (2.0 * V_Q * D_Q + 2 * N * D_Q) / (hbm * 1e9))
            t_sus = max(2.0 * N * V_Q * D_Q / (tf_sust * 1e12), (2.0 * V_Q * D_Q + 2 * N * D_Q) / (hbm * 1e9))
            emit({"config": f"B{B}_g{g}", "B": B, "gamma": g, "N": N, "path": PATH_NAMES[path],
                              "us_per_step": ms * 1e3, "positions_per_s": N / (ms / 1e3),
                              "accepted_tokens_per_s": toks / (ms / 1e3), "roofline_us": t_star * 1e6,
                              "frac_of_roofline": t_star / (ms / 1e3), "roofline_us_sustained": t_sus * 1e6,
                              "frac_of_roofline_sustained": t_sus / (ms / 1e3),
                              "us_per_step_graph": ms_graph * 1e3 if ms_graph else None,
                              "frac_of_roofline_graph": t_star / (ms_graph / 1e3) if ms_graph else None,
                              "frac_of_roofline_sustained_graph": t_sus / (ms_graph / 1e3) if ms_graph else None,
                              "dominant_kernel_us": kms / max(kn, 1) * 1e3,
                              "launches": launches})
            del v


def _cpu_batch(b):
    import torch
    from synth.inputs import Batch
    return Batch(b.hidden.cpu(), b.W.cpu(), b.draft_tokens.cpu(), b.draft_probs.cpu(), b.gamma, b.uniforms.cpu())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="nj", choices=["nj", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(set(CONFIGS) | {"c4", "c5", "propose", "greedy_c2", "greedy_b256g5"}))
    ap.add_argument("--path", default=None, choices=[None] + PATH_NAMES)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager nj_verify launches only")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--sweep", action="store_true", help="C3 grid: one JSON line per (B, gamma) point")
    ap.add_argument("--sweep-B", default="1,2,4,8,16,32,48,64,96,128,192,256")
    ap.add_argument("--sweep-gamma", default="0,1,2,3,4,5,mixed:5")
    ap.add_argument("--trace-steps", type=int, default=4000)
    ap.add_argument("--c4-buckets", default="graph", choices=["graph", "none"],
                    help="C4: pad B_t up to the CUDA-graph batch buckets (graph) or not (none)")
    ap.add_argument("--cprefill-b200-scale", type=float, default=0.07,
                    help="C4: factor on the B200 c_prefill table (verification step / full step time)")
    ap.add_argument("--cprefill-table1", action="store_true",
                    help="C4: use PAPER Table 1 x --cprefill-scale even if a B200 measurement exists")
    ap.add_argument("--cprefill-scale", type=float, default=0.01)
    ap.add_argument("--temperature", type=float, default=1.0, help="target temperature (nj_set_temperature)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak = every rank its own batch; strong = one global batch split by rows")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    _claim_stdout()
    ws, rank, local = dist_setup()
    if ws != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
    if args.sweep:
        bench_sweep(args, ws, rank, local)
        return
    if args.config == "c4" and args.impl != "reference":
        bench_c4(args, ws, rank, local)
        return
    if args.config == "c5" and args.impl != "reference":
        bench_c5(args, ws, rank, local)
        return
    if args.config.startswith("greedy") and args.impl != "reference":
        bench_greedy(args, ws, rank, local)
        return
    if args.config == "propose" and args.impl != "reference":
        bench_propose(args, ws, rank, local)
        return
    if args.impl == "reference":
        bench_reference(args, ws, rank)
    else:
        bench_nj(args, ws, rank, local)


if __name__ == "__main__":
    sys.exit(main() or 0)
