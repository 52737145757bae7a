"""Plain-Python reference of Nightjar's arm selection (Algorithm 1 + Eq. 3).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Written line by line from
PAPER.md, independently of the C++ bandit in libnj:

  Eq. 3:  gamma* = argmin_g 1/g~_{B,g} + 1(g_{t-1}=0 and g>0) c_prefill / g
  CMA update: g~^(n) = g~^(n-1) + (r - g~^(n-1)) / n,  g~^(0) = 0
  Algorithm 1: per-B state j_B=H_B=b_B=tau_B=1; at tau_B = 1 the bin
      is Exploration w.p. 1/sqrt(b_B) (line 179); explore -> gamma ~ U{0..Gmax}
      (line 183), exploit -> Eq. 3 (line 187); play, observe, update (line 190);
      tau_B += 1; if tau_B > sqrt(H_B): b_B += 1, tau_B = 1; if b_B > sqrt(H_B):
      j_B += 1, H_B = 2^(j_B - 1), b_B = 1 (lines 191-199).
  c_prefill lookup (Table 1): L_max = max_i L_i, ceiling
      bucket with clamp, ms -> s.
Gap readings (R13, R14 = SPEC ledger S:112-119): unvisited arms are
excluded from the argmin, all unvisited -> 0; ties -> smallest gamma;
gamma_{t-1} is global; bin type drawn lazily at the first select of a bin;
RNG draws in the order bin-type then arm; sqrt comparisons real-valued.

RNG: SplitMix64 evaluated at (seed, counter) -- a counter-based generator that
the C++ side implements independently (R14), so both consume the same
random numbers without sharing code.
"""
from __future__ import annotations

import math

_M64 = (1 << 64) - 1


def splitmix64(seed: int, k: int) -> int:
    z = (seed + (k + 1) * 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


class Rng:
    def __init__(self, seed: int):
        self.seed = seed & _M64
        self.k = 0

    def uniform(self) -> float:
        v = splitmix64(self.seed, self.k)
        self.k += 1
        return (v >> 11) * (1.0 / (1 << 53))


class PrefillTable:
    def __init__(self, len_buckets, batch_buckets, cost_ms):
        self.L = list(len_buckets)
        self.B = list(batch_buckets)
        self.c = [list(r) for r in cost_ms]  # [len][batch] ms

    def cost_ms(self, l_max: int, batch: int) -> float:
        if l_max <= 0 or not self.L:
            return 0.0
        i = next((k for k, v in enumerate(self.L) if v >= l_max), len(self.L) - 1)
        j = next((k for k, v in enumerate(self.B) if v >= batch), len(self.B) - 1)
        return self.c[i][j]


class Hier:
    def __init__(self, arms: int):
        self.j, self.H, self.b, self.tau = 1, 1, 1, 1
        self.bin_type = None  # None unset, "explore", "exploit"
        self.mean = [0.0] * arms
        self.n = [0] * arms


class Nightjar:
    def __init__(self, gamma_max: int, batch_max: int, seed: int, table: PrefillTable | None = None):
        if gamma_max < 1 or batch_max < 1:
            raise ValueError("gamma_max and batch_max must be >= 1")
        self.G = gamma_max
        self.Bmax = batch_max
        self.rng = Rng(seed)
        self.table = table
        self.h = {B: Hier(gamma_max + 1) for B in range(1, batch_max + 1)}
        self.last_gamma = 0  # gamma_{t-1}, global (R14)

    def c_prefill_s(self, l_max: int, B: int) -> float:
        return 0.0 if self.table is None else self.table.cost_ms(l_max, B) / 1000.0

    def score(self, B: int, gamma_prev: int, g: int, l_max: int) -> float:
        h = self.h[B]
        if h.n[g] == 0:
            return float("nan")
        inv = math.inf if h.mean[g] == 0.0 else 1.0 / h.mean[g]
        sw = self.c_prefill_s(l_max, B) / g if (gamma_prev == 0 and g > 0) else 0.0
        return inv + sw

    def select(self, B: int, l_max: int = 0) -> int:
        if not (1 <= B <= self.Bmax):
            raise ValueError("batch size out of range")
        h = self.h[B]
        if h.tau == 1 and h.bin_type is None:              # line 177-179
            h.bin_type = "explore" if self.rng.uniform() < 1.0 / math.sqrt(h.b) else "exploit"
        if h.bin_type == "explore":                        # line 181-183
            return min(int(self.rng.uniform() * (self.G + 1)), self.G)
        best, best_s = 0, None                             # line 185-187, Eq. 3
        for g in range(self.G + 1):
            s = self.score(B, self.last_gamma, g, l_max)
            if math.isnan(s):
                continue
            if best_s is None or s < best_s:
                best, best_s = g, s
        return best

    def observe(self, B: int, g: int, r: float) -> None:
        if r < 0:
            raise ValueError("negative reward")
        h = self.h[B]
        h.n[g] += 1                                         # line 190 + P:120
        h.mean[g] += (r - h.mean[g]) / h.n[g]
        self.last_gamma = g
        h.tau += 1                                          # line 191
        if h.tau > math.sqrt(h.H):                          # line 193
            h.b += 1
            h.tau = 1
            h.bin_type = None
            if h.b > math.sqrt(h.H):                        # line 196
                h.j += 1
                h.H = 2 ** (h.j - 1)
                h.b = 1


# Table 1: c_prefill (ms), 7B on RTX 4090, by input length x batch size.
TABLE1_LEN = [128, 256, 512]
TABLE1_BATCH = [32, 64]
TABLE1_MS = [[17.87, 28.53], [20.65, 22.33], [24.30, 102.03]]
