// nj_bandit.cpp — Nightjar speculative-length bandit (host side of libnj).
//
// PAPER.md P:113-118 (Eq. 3 cost-aware exploitation), P:120 (incremental
// cumulative moving average), P:125-133 and Algorithm 1 P:164-203 (per-batch-
// size block / bin / round hierarchy, exploration probability 1/sqrt(b_B),
// block growth H_B <- 2^(j_B-1)), P:135-162 (c_prefill(L_max, B) lookup of
// Table 1).  Gaps are resolved as DESIGN.md R13/R14 (SPEC ledger S:112-119).
//
// Selection is O(Gamma_max) with no allocation: the paper reports ~1e-5 s per
// decision; this implementation targets < 1 us.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <new>
#include <string>
#include <vector>

#include "nj.h"

namespace {

// Counter-based SplitMix64: draw k of stream `seed` (R14).
inline uint64_t mix64(uint64_t seed, uint64_t k) {
    uint64_t z = seed + (k + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

enum BinType : int32_t { kUnset = -1, kExploit = 0, kExplore = 1 };

struct BatchState {           // D1 / D2: one per batch size B (Algorithm 1)
    int32_t j = 1;            // block index j_B
    int64_t H = 1;            // block size  H_B = 2^(j_B-1)
    int64_t bin = 1;          // bin index   b_B
    int64_t tau = 1;          // round       tau_B
    int32_t bin_type = kUnset;
    double sqrtH = 1.0;       // sqrt(H_B), recomputed when H changes
};

}  // namespace

struct nj_bandit {
    int32_t gamma_max = 0;
    int32_t batch_max = 0;
    uint64_t seed = 0;
    uint64_t draws = 0;                  // RNG counter
    int32_t last_gamma = 0;              // gamma_{t-1}, global engine state (R14)
    std::vector<BatchState> st;          // [batch_max]
    std::vector<double> mean;            // [batch_max][gamma_max+1]  g~_{B,gamma}
    std::vector<int64_t> count;          // visit counts n
    std::vector<int32_t> len_b, batch_b; // c_prefill buckets
    std::vector<double> cost_ms;         // [n_len][n_batch]

    double uniform() { return double(mix64(seed, draws++) >> 11) * (1.0 / 9007199254740992.0); }
    size_t arm(int32_t B, int32_t g) const { return size_t(B - 1) * size_t(gamma_max + 1) + size_t(g); }
};

static double prefill_ms(const nj_bandit* b, int32_t l_max, int32_t B) {
    if (l_max <= 0 || b->len_b.empty()) return 0.0;
    size_t i = 0;
    while (i + 1 < b->len_b.size() && b->len_b[i] < l_max) ++i;   // ceiling, clamp to last
    size_t k = 0;
    while (k + 1 < b->batch_b.size() && b->batch_b[k] < B) ++k;
    return b->cost_ms[i * b->batch_b.size() + k];
}

// Eq. 3 score in seconds; NaN for an unvisited arm.
static double score(const nj_bandit* b, int32_t B, int32_t gprev, int32_t g, double cpre_s) {
    size_t a = b->arm(B, g);
    if (b->count[a] == 0) return std::numeric_limits<double>::quiet_NaN();
    double inv = b->mean[a] == 0.0 ? std::numeric_limits<double>::infinity() : 1.0 / b->mean[a];
    double sw = (gprev == 0 && g > 0) ? cpre_s / double(g) : 0.0;
    return inv + sw;
}

extern "C" {

nj_status nj_bandit_create(int32_t gamma_max, int32_t batch_max, uint64_t seed,
                           const int32_t* len_buckets, int32_t n_len,
                           const int32_t* batch_buckets, int32_t n_batch,
                           const double* cost_ms, nj_bandit** out) {
    if (!out) return NJ_EINVAL;
    *out = nullptr;
    if (gamma_max < 1 || batch_max < 1 || gamma_max > 64 || batch_max > (1 << 20)) return NJ_EINVAL;
    if (cost_ms) {
        if (!len_buckets || !batch_buckets || n_len < 1 || n_batch < 1) return NJ_EINVAL;
        for (int32_t i = 1; i < n_len; ++i) if (len_buckets[i] <= len_buckets[i - 1]) return NJ_EINVAL;
        for (int32_t i = 1; i < n_batch; ++i) if (batch_buckets[i] <= batch_buckets[i - 1]) return NJ_EINVAL;
        for (int32_t i = 0; i < n_len * n_batch; ++i) if (!(cost_ms[i] > 0.0)) return NJ_EINVAL;
    }
    nj_bandit* b = new (std::nothrow) nj_bandit();
    if (!b) return NJ_ENOMEM;
    b->gamma_max = gamma_max;
    b->batch_max = batch_max;
    b->seed = seed;
    b->st.resize(size_t(batch_max));
    b->mean.assign(size_t(batch_max) * size_t(gamma_max + 1), 0.0);
    b->count.assign(size_t(batch_max) * size_t(gamma_max + 1), 0);
    if (cost_ms) {
        b->len_b.assign(len_buckets, len_buckets + n_len);
        b->batch_b.assign(batch_buckets, batch_buckets + n_batch);
        b->cost_ms.assign(cost_ms, cost_ms + size_t(n_len) * size_t(n_batch));
    }
    *out = b;
    return NJ_OK;
}

void nj_bandit_destroy(nj_bandit* b) { delete b; }

int32_t nj_select_gamma(nj_bandit* b, int32_t B, int32_t l_max) {
    if (!b || B < 1 || B > b->batch_max || l_max < 0) return -NJ_EINVAL;
    BatchState& s = b->st[size_t(B - 1)];
    if (s.tau == 1 && s.bin_type == kUnset)                                // lines 177-179
        s.bin_type = (b->uniform() < 1.0 / std::sqrt(double(s.bin))) ? kExplore : kExploit;
    if (s.bin_type == kExplore) {                                          // lines 181-183
        int32_t g = int32_t(b->uniform() * double(b->gamma_max + 1));
        return g > b->gamma_max ? b->gamma_max : g;
    }
    const double cpre_s = prefill_ms(b, l_max, B) * 1e-3;                 // ms -> s
    int32_t best = 0;                                                      // all unvisited -> 0
    double best_s = std::numeric_limits<double>::quiet_NaN();
    for (int32_t g = 0; g <= b->gamma_max; ++g) {                          // lines 185-187
        double sc = score(b, B, b->last_gamma, g, cpre_s);
        if (std::isnan(sc)) continue;                                      // unvisited excluded
        if (std::isnan(best_s) || sc < best_s) { best = g; best_s = sc; }  // ties -> smallest
    }
    return best;
}

nj_status nj_observe(nj_bandit* b, int32_t B, int32_t g, double r) {
    if (!b || B < 1 || B > b->batch_max || g < 0 || g > b->gamma_max) return NJ_EINVAL;
    if (!(r >= 0.0) || std::isinf(r)) return NJ_EINVAL;
    size_t a = b->arm(B, g);
    b->count[a] += 1;
    b->mean[a] += (r - b->mean[a]) / double(b->count[a]);
    b->last_gamma = g;
    BatchState& s = b->st[size_t(B - 1)];
    s.tau += 1;                                                            // line 191
    if (double(s.tau) > s.sqrtH) {                                         // line 193
        s.bin += 1;
        s.tau = 1;
        s.bin_type = kUnset;
        if (double(s.bin) > s.sqrtH) {                                     // line 196
            s.j += 1;
            s.H = (s.j - 1) >= 62 ? (int64_t(1) << 62) : (int64_t(1) << (s.j - 1));
            s.sqrtH = std::sqrt(double(s.H));
            s.bin = 1;
        }
    }
    return NJ_OK;
}

double nj_exploitation_score(const nj_bandit* b, int32_t B, int32_t gprev, int32_t g, int32_t l_max) {
    if (!b || B < 1 || B > b->batch_max || g < 0 || g > b->gamma_max)
        return std::numeric_limits<double>::quiet_NaN();
    return score(b, B, gprev, g, prefill_ms(b, l_max, B) * 1e-3);
}

double nj_prefill_cost_ms(const nj_bandit* b, int32_t l_max, int32_t B) {
    if (!b) return std::numeric_limits<double>::quiet_NaN();
    return prefill_ms(b, l_max, B);
}

nj_status nj_bandit_state(const nj_bandit* b, int32_t B, int32_t* j, int64_t* H, int64_t* bin,
                          int64_t* tau, int32_t* bin_type) {
    if (!b || B < 1 || B > b->batch_max) return NJ_EINVAL;
    const BatchState& s = b->st[size_t(B - 1)];
    if (j) *j = s.j;
    if (H) *H = s.H;
    if (bin) *bin = s.bin;
    if (tau) *tau = s.tau;
    if (bin_type) *bin_type = s.bin_type;
    return NJ_OK;
}

nj_status nj_bandit_arm(const nj_bandit* b, int32_t B, int32_t g, double* mean, int64_t* count) {
    if (!b || B < 1 || B > b->batch_max || g < 0 || g > b->gamma_max) return NJ_EINVAL;
    size_t a = b->arm(B, g);
    if (mean) *mean = b->mean[a];
    if (count) *count = b->count[a];
    return NJ_OK;
}

int32_t nj_bandit_last_gamma(const nj_bandit* b) { return b ? b->last_gamma : -NJ_EINVAL; }

nj_status nj_bandit_snapshot_json(const nj_bandit* b, char* buf, size_t cap, size_t* needed) {
    if (!b) return NJ_EINVAL;
    std::string s;
    char tmp[160];
    std::snprintf(tmp, sizeof tmp,
                  "{\"gamma_max\":%d,\"batch_max\":%d,\"seed\":%llu,\"draws\":%llu,\"last_gamma\":%d,\"batches\":[",
                  b->gamma_max, b->batch_max, (unsigned long long)b->seed,
                  (unsigned long long)b->draws, b->last_gamma);
    s += tmp;
    bool first = true;
    for (int32_t B = 1; B <= b->batch_max; ++B) {
        const BatchState& st = b->st[size_t(B - 1)];
        bool touched = st.j != 1 || st.tau != 1 || st.bin != 1 || st.bin_type != kUnset;
        for (int32_t g = 0; g <= b->gamma_max && !touched; ++g) touched = b->count[b->arm(B, g)] != 0;
        if (!touched) continue;
        if (!first) s += ",";
        first = false;
        std::snprintf(tmp, sizeof tmp, "{\"B\":%d,\"j\":%d,\"H\":%lld,\"b\":%lld,\"tau\":%lld,\"bin_type\":%d,\"arms\":[",
                      B, st.j, (long long)st.H, (long long)st.bin, (long long)st.tau, st.bin_type);
        s += tmp;
        for (int32_t g = 0; g <= b->gamma_max; ++g) {
            std::snprintf(tmp, sizeof tmp, "%s{\"gamma\":%d,\"mean\":%.17g,\"n\":%lld}", g ? "," : "", g,
                          b->mean[b->arm(B, g)], (long long)b->count[b->arm(B, g)]);
            s += tmp;
        }
        s += "]}";
    }
    s += "]}";
    if (needed) *needed = s.size() + 1;
    if (!buf || cap < s.size() + 1) return NJ_ESHAPE;
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return NJ_OK;
}

}  // extern "C"
