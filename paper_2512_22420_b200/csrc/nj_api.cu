// nj_api.cu — host side of libnj: the C ABI of include/nj.h.
//
// Validation, workspace ownership, TMA tensor-map encoding, path planning and
// launch sequencing for nj_verify (BJ steps 1-3), plus the
// test-only stage exports.  No device->host synchronisation happens inside
// nj_verify: gamma_per_req is a host array, so every shape (N, G, row offsets)
// is known here and passed to the kernels by value (graph capturable).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "nj.h"
#include "nj_gemm.cuh"
#include "nj_sampler.cuh"
#include "nj_shard.cuh"

#include <dlfcn.h>

using namespace nj;

namespace {

thread_local std::string g_create_error;

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// 2-D bf16 K-major tensor [rows, d], box {64, box_rows}, SWIZZLE_128B.
bool encode_2d(CUtensorMap* m, const void* base, int64_t rows, int64_t d, int box_rows) {
    EncodeTiledFn fn = get_encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)d * 2};
    cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 2-D fp32 row-major tensor [rows][cols] with row pitch ld (elements), box {16, 32},
// SWIZZLE_64B: k_lmhead's logits stores (nj_lmhead.cuh)
bool encode_out(CUtensorMap* m, const float* base, int64_t rows, int64_t cols, int64_t ld) {
    EncodeTiledFn fn = get_encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
    cuuint32_t box[2] = {16, 32};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

constexpr int kStagedMaxN = kBigMaxRowG;   // staged path on k_gemm_big (NJ_LM=0): rows of one GEMM pass
constexpr int kFusedAutoMaxN = 24;          // AUTO takes the fused kernel up to this many rows
constexpr int kInlineLseRows = 64;          // staged path: N up to which k_accept merges row statistics inline
constexpr int kStagedMaxRows = 2048;        // staged path on k_lmhead: rows of one GEMM pass (logits_st rows)
constexpr int kPhaseTsN = 24 * 1024;     // debug timeline entries (NJ_PHASE_TS): k_lmhead [0, 18K) CTA 0 + [20K, 20.5K) per-CTA end, k_sample_small [18K, 20K)

inline int round16(int x) { return (x + 15) & ~15; }
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// device smem carve-up mirror (must match nj_fused.cuh)
size_t fused_tail(int NPAD, int S) {
    const int kMaxT = 16;
    size_t t = 0;
    t += 4 * NPAD * sizeof(float2);
    t += NPAD * sizeof(double);
    t += NPAD * sizeof(ReqInfo);
    t += (size_t)NPAD * kMaxT * 4 * sizeof(float);
    t += (size_t)NPAD * (kMaxT + 1) * sizeof(double);
    t += NPAD * sizeof(double);
    t += 5 * NPAD * sizeof(int32_t) + 4 * sizeof(int32_t) + 2 * NPAD * sizeof(float);
    t = align_up(t, 8);
    t += (size_t)(2 * S + 16) * 8 + 8;
    return t;
}

// Tuning / probe knobs (DESIGN.md §8 "knobs"): read from the environment ONCE
// at nj_create (never per launch); -1 = unset (the measured defaults apply).
struct Knobs {
    int fgroups = -1, kpd = -1, sacc = -1, kgroup = -1, phase_ts = 0;       // fused kernel
    int big_gk = -1, big_nbuf = -1, big_dbg = 0, spin = 0, stats = 1, sleep_ns = 0, big_s = -1;   // k_gemm_big
    int w_evict_first = -1, mass_probe = 0;
    int lm = 1, lm_cg = 0, lm_tw = 256, lm_gk = 0, lm_s = 0, lm_dbg = 0, lm_nbuf = 0, lm_ks = 0, lm_tma_out = 1, lm_pf = -1, lm_mb = 0, lm_ost = 1, lm_ks0 = 0, lm_arv1 = 0, lm_w = 0, lm_fence = 0, lm_mma4 = 0, small = 1, small_pdl = 1, small_cl16 = 1, qpf = 0, small_pf = 0, lm_sleep = 0, small_bmax = 12, inline_lse = kInlineLseRows, small_trig = 0, lm_pdl = 0, small_cl12 = 1, small_reuse = 1, small_cl = 0, qstage_gbs = 50, pdl_chain = 0, small_flat = 1, hostq_fused = 0, small_coop = 1, lm_out_keep = 0, lm_zero = 1;   // k_lmhead; k_sample_small
};
int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return (e && *e) ? atoi(e) : dflt;
}
Knobs read_knobs() {
    Knobs k;
    k.fgroups = env_int("NJ_FGROUPS", -1);
    k.kpd = env_int("NJ_KPD", -1);
    k.sacc = env_int("NJ_SACC", -1);
    k.kgroup = env_int("NJ_KGROUP", -1);
    k.phase_ts = env_int("NJ_PHASE_TS", 0) == 1;
    k.big_gk = env_int("NJ_BIG_GK", -1);
    k.big_nbuf = env_int("NJ_BIG_NBUF", -1);
    k.big_dbg = env_int("NJ_BIG_DBG", 0);
    k.spin = env_int("NJ_SPIN", 0);
    k.stats = env_int("NJ_STATS", 1);
    k.sleep_ns = env_int("NJ_SLEEP", 0);
    k.big_s = env_int("NJ_BIG_S", -1);
    k.w_evict_first = env_int("NJ_W_EVICT_FIRST", -1);
    k.mass_probe = env_int("NJ_MASS_PROBE", 0);
    k.lm = env_int("NJ_LM", 1);
    k.lm_cg = env_int("NJ_LM_CG", 0);
    k.lm_tw = std::min(256, std::max(16, env_int("NJ_LM_TW", 256) & ~15));
    k.lm_gk = env_int("NJ_LM_GK", 0);
    k.lm_s = env_int("NJ_LM_S", 0);
    k.lm_dbg = env_int("NJ_LM_DBG", 0);
    k.lm_nbuf = env_int("NJ_LM_NBUF", 0);   // probes only (TMEM holds 512 / stride buffers)
    k.lm_ks = env_int("NJ_LM_KS", 0);
    k.lm_tma_out = env_int("NJ_LM_TMA_OUT", 1);
    k.lm_pf = env_int("NJ_LM_PF", -1);
    k.lm_mb = env_int("NJ_LM_MB", 0);
    k.lm_ks0 = env_int("NJ_LM_KS0", 0);
    k.lm_arv1 = env_int("NJ_LM_ARV1", 0);
    k.lm_w = std::min(256, env_int("NJ_LM_W", 0) & ~15);   // probe: fixed tile width (ragged last tile)
    k.lm_fence = env_int("NJ_LM_FENCE", 0);
    k.lm_mma4 = env_int("NJ_LM_MMA4", 0);
    k.small = env_int("NJ_SMALL", 1);
    k.small_pdl = env_int("NJ_SMALL_PDL", 1);
    k.small_cl16 = env_int("NJ_SMALL_CL16", 1);
    k.small_pf = env_int("NJ_SMALL_PF", 0);          // measured slower (C2 204.7 vs 200.5 us)
    k.lm_sleep = env_int("NJ_LM_SLEEP", 0);
    k.small_flat = env_int("NJ_SMALL_FLAT", 1);     // k_sample_small<FLAT> (no cluster, PDL dependent of k_lmhead)
    // batch limit of the one-launch sampler: flat mode beats the multi-kernel sampler up to
    // B = 32 (sweep at gamma 2 / 3: -2..-4 % at B = 16-24, -1 % at 32, +1 % at 40-48), the
    // cluster mode up to 12
    k.small_bmax = env_int("NJ_SMALL_BMAX", k.small_flat ? 32 : 12);
    k.inline_lse = env_int("NJ_INLINE_LSE", kInlineLseRows);
    k.lm_pdl = env_int("NJ_LM_PDL", 0);             // k_lmhead triggers its dependents' launch at its start:
                                                    // k_sample_small still starts ~4 us after the last GEMM CTA (no gain)
    k.small_cl12 = env_int("NJ_SMALL_CL12", 1);     // 12-CTA clusters between 16 and 8
    k.small_reuse = env_int("NJ_SMALL_REUSE", 1);   // owner CTA reads the located chunk from its staging buffer
    k.small_cl = env_int("NJ_SMALL_CL", 0);
    k.qstage_gbs = env_int("NJ_QSTAGE_GBS", 50);
    // host-resident q (nj_verify_host): 1 = the fused kernel up to 48 rows; 0 (default) = the
    // device-q rule -- the staged step above 24 rows, whose flat sampler reads q_i(x_i) during
    // the GEMM's tail and the rejected rows' chunks from ~144 CTAs at once (e2e +13..19 % at
    // B = 8-16, scripts/e2e_path.py)
    k.hostq_fused = env_int("NJ_HOSTQ_FUSED", 0);
    k.lm_out_keep = env_int("NJ_LM_OUT_KEEP", 0);
    k.lm_zero = env_int("NJ_LM_ZERO", 1);           // staged step: k_lmhead zeroes the fallback block   // evict_last hint on small staged logits stores
    k.small_coop = env_int("NJ_SMALL_COOP", 1);     // flat sampler launched cooperatively (co-residency guaranteed)
    k.pdl_chain = env_int("NJ_PDL_CHAIN", 0);       // staged multi-kernel sampler as a PDL chain (no gain measured:
                                                    // B = 16 / 64 / 256 equal within the box's noise)    // host-link GB/s assumed by the q-row staging budget         // tests: force the cluster size (2, 4, 8, 12, 16; 0 = auto)
    k.small_trig = env_int("NJ_SMALL_TRIG", 0);   // early PDL trigger of the fallback launch (no gain measured)   // larger B: 2-4 CTA clusters measured slower than the 4-5 launches
    k.qpf = env_int("NJ_QPF", 0);   // measured slower (the prefetch competes with the W stream)
    k.lm_ost = std::min(2, std::max(1, env_int("NJ_LM_OST", 1)));
    return k;
}

}  // namespace

struct nj_ctx {
    nj_config cfg{};
    Knobs kn;
    int V_local = 0;
    int num_sms = 0;
    int grid = 0;       // persistent grid (CTAs)
    int pld = 0;        // row stride of the per-CTA softmax partials (>= every GEMM grid)
    int gemm_ks = 4;    // k_gemm_big: k-blocks per accumulator restart
    int gemm_ks_ka = 8; // two-pass K-A (acceptance statistics only, certified): restart period
    int gemm_cg = 0;    // k_gemm_big CTA group: 0 auto, 1 single CTA, 2 CTA pair (NJ_CG)
    int gemm_pf = 0;    // k_gemm_big: W k-blocks prefetched into L2 ahead of the ring (NJ_PF)
    int gemm_maxt = 256;  // k_gemm_big: max token chunk (NJ_BIG_MAXT)
    int gemm_teams = -1;  // k_gemm_big: two alternating epilogue teams (NJ_TEAMS; -1 auto)
    int U = 0;          // 16-row vocab units
    int max_tiles = 0;  // max 128-row tiles per CTA
    int nchunks = 0;    // sampler chunks
    int Nmax = 0, Gmax = 0;
    // options
    int path_opt = NJ_PATH_AUTO;
    int certify = 1;
    int force_fb = 0;
    double temperature = 1.0;   // target temperature T (nj_set_temperature); logits l / T
    double inv_t = 1.0;
    int profile = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;   // recorded, not yet harvested
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_free;
    double prof_ms = 0.0;
    int64_t prof_n = 0;
    unsigned long long* phase_ts = nullptr;   // debug (NJ_PHASE_TS=1)
    // certificate margins: fused path logits err <= 6e-7 (ln p);
    // two-pass path (restarted accumulators, fp32 RN running sums) ln p err ~1e-6
    // Draws carry no certificate (eps_draw = 0): at V = 152064 the CDF breakpoints
    // are ~6.6e-6 apart, so any band comparable to them would fire on most draws;
    // the GEMMs are instead accurate enough that the draw CDF error stays far
    // below the 1e-6 tie band (tests/test_gpu_parity.py uncertified).
    float eps_acc_fused = 2e-6f, eps_draw_fused = 0.f;
    // acceptance certificates = ~2x the measured max |d ln p| over every vocabulary
    // entry with p > 1e-6 (profiles/r02_ks_accuracy.json: restart every 4 / 8 / 14
    // k-blocks -> 6.8e-6 / 1.03e-5 / 1.9e-5)
    float eps_acc = 1.5e-5f;      // k_gemm_big, restart every 4 k-blocks (staged, K-C)
    float eps_acc_ka = 2.5e-5f;   // two-pass K-A, restart every 8 k-blocks (certificate off)
    float eps_acc_ka_cert = 4e-5f;   // two-pass / sharded K-A with the certificate on (14 k-blocks)
    int gemm_ks_ka_cert = 14;     // K-A restart period when certified: acceptance-only rows,
                                  // every near-tie recomputed in fp64 (-9 % K-A time at B=256 gamma=5)
    float eps_draw = 0.f;
    std::string err;
    // workspace
    std::vector<void*> allocs;
    float *part_m = nullptr, *part_s = nullptr, *part2_m = nullptr, *part2_s = nullptr;
    double* dl = nullptr;
    double* row_lse = nullptr;   // [max(Nmax, Gmax)] k_lse_rows output
    double *wpart = nullptr, *s_lse = nullptr, *cmass = nullptr, *fb_logits = nullptr, *lse_tmp = nullptr;
    uint16_t *hd = nullptr, *hs = nullptr;
    float* logits_s = nullptr;
    float* logits_st = nullptr;    // staged path: [staged_rows][V_local]
    int32_t *s_resid = nullptr, *s_qrow = nullptr;
    int32_t* fb_block = nullptr;   // [0] count, [1..MB] list, [1+MB..] req_flags, [1+2MB..] k_sample_small<FLAT> arrivals
    uint32_t* bar = nullptr;       // count, gen
    int32_t* fb_done = nullptr;    // k_fb completion counter
    unsigned long long* amax = nullptr;   // nj_verify_greedy: per-row argmax keys [Nmax]
    int mass_nst = 2;                 // k_mass cp.async ring stages (NJ_MASS_NST: 2..4; 2 = 3 CTAs / SM)
    int mass_occ = 1;                 // resident k_mass CTAs per SM at mass_nst
    int small_maxcl[17] = {};         // k_sample_small: co-resident clusters of 2 / 4 / 8 / 12 / 16 CTAs (0: unknown)
    int32_t* scratch_i = nullptr;  // [MB]
    int32_t* s_row = nullptr;      // [MB] staged path: sample row of each request
    int32_t* g2row = nullptr;      // [Gmax] staged sharded step: packed row of each draft row
    // vocab-sharded mode (nj_shard.cuh): rank / ranks, NCCL comm or nj_group member
    int nranks = 1, rank = 0;
    void* ncomm = nullptr;
    bool in_group = false;
    bool sharded() const { return ncomm != nullptr || in_group; }
    double *xs1 = nullptr, *xr1 = nullptr, *xs2 = nullptr, *xr2 = nullptr, *xs3 = nullptr, *xr3 = nullptr;
    double* fblse = nullptr;
    int32_t *x6 = nullptr, *fbn = nullptr;
    // host-API staging (lazy)
    uint16_t* st_hidden = nullptr;
    int32_t* st_tok = nullptr;
    float *st_q = nullptr, *st_u = nullptr;
    int32_t *st_acc = nullptr, *st_next = nullptr;
    int64_t st_ldq = 0;
    int q_zero_copy = 1;   // nj_verify_host: read mapped pinned q in place (NJ_OPT_Q_ZERO_COPY)
    int q_remote = 0;      // the current call's q lives in host memory (no bulk q prefetch)
    // nj_verify_host, zero-copy q: the likely sample rows staged into st_q over a copy
    // stream while the GEMM runs (NJ_OPT_Q_STAGE_ROWS; -1 auto budget, 0 off = default)
    int q_stage_opt = 0;   // off by default: on this pool's hosts a pinned 608-KB copy takes ~50 us
                           // (12.6 GB/s; 40 GB/s for 8 MB), so staging gains <= 6 % of a C2 call, noisily
    cudaStream_t cstream = nullptr;
    cudaEvent_t ev_qstage = nullptr;
    int qstage_active = 0;              // the current call staged rows (the sampler waits for ev_qstage)
    uint64_t qstage_mask[4] = {};       // staged draft rows (bit g), G <= 256
    std::vector<int32_t> qstage_rows;   // the last call's staged rows (nj_host_staged_rows)
    // W tensor-map cache
    const void* w_cached = nullptr;
    CUtensorMap tmW128{}, tmW16{};
    const void* lm_w_cached = nullptr;   // k_lmhead W map (box rows vary with the tile width)
    int lm_wbox = 0;
    CUtensorMap tmWlm{};
    int staged_rows = 0;                 // rows of logits_st

    int32_t* fb_count() { return fb_block; }
    int32_t* fb_list() { return fb_block + 1; }
    int32_t* req_flags() { return fb_block + 1 + cfg.max_batch; }
    int32_t* small_cnt() { return fb_block + 1 + 2 * cfg.max_batch; }
};

namespace {

nj_status set_err(nj_ctx* c, nj_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf; else g_create_error = buf;
    return st;
}

// NJ_TRACE=1: synchronise after every launch and report it on stderr (debug).
bool trace_on() {
    static int on = -1;
    if (on < 0) { const char* e = getenv("NJ_TRACE"); on = (e && *e == '1') ? 1 : 0; }
    return on == 1;
}
// NJ_LAUNCH_TIMES=1 (measurement): an event after every launch; at exit, per kernel
// name the mean GPU time between its event and the previous launch's event on the same
// stream (the kernel's duration in an eager back-to-back pipeline, no profiler attached),
// printed to stderr.  Production runs leave it off (one getenv at first launch).
struct LaunchTimes {
    struct Rec { const char* name; cudaStream_t st; cudaEvent_t ev; };
    std::vector<Rec> recs;
    std::mutex mu;
    ~LaunchTimes() {
        if (recs.empty()) return;
        cudaDeviceSynchronize();
        std::unordered_map<std::string, std::pair<double, int64_t>> agg;
        std::vector<std::string> order;
        std::unordered_map<cudaStream_t, cudaEvent_t> last;
        for (auto& r : recs) {
            auto it = last.find(r.st);
            if (it != last.end()) {
                float ms = 0.f;
                if (cudaEventElapsedTime(&ms, it->second, r.ev) == cudaSuccess) {
                    auto& a = agg[r.name];
                    if (a.second == 0) order.push_back(r.name);
                    a.first += ms;
                    a.second += 1;
                }
            }
            last[r.st] = r.ev;
        }
        for (auto& n : order)
            fprintf(stderr, "[nj-launch-times] %s n=%lld mean_us=%.2f\n", n.c_str(), (long long)agg[n].second,
                    agg[n].first * 1e3 / agg[n].second);
    }
};
LaunchTimes& launch_times() { static LaunchTimes lt; return lt; }
bool launch_times_on() {
    static int on = -1;
    if (on < 0) { const char* e = getenv("NJ_LAUNCH_TIMES"); on = (e && *e == '1') ? 1 : 0; }
    return on == 1;
}
cudaError_t trace(const char* what, cudaStream_t st) {
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess && launch_times_on()) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone) {
            cudaEvent_t ev;
            if (cudaEventCreate(&ev) == cudaSuccess) {
                std::lock_guard<std::mutex> g(launch_times().mu);
                if (cudaEventRecord(ev, st) == cudaSuccess) launch_times().recs.push_back({what, st, ev});
            }
        }
    }
    if (!trace_on() || e != cudaSuccess) return e;
    e = cudaStreamSynchronize(st);
    fprintf(stderr, "[nj] %s -> %s\n", what, cudaGetErrorString(e));
    return e;
}
#define NJ_LAUNCHED(ctx, name, st) NJ_CUDA(ctx, trace(name, st))

#define NJ_CUDA(ctx, call)                                                                          \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess)                                                                      \
            return set_err(ctx, NJ_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),   \
                           __FILE__, __LINE__);                                                     \
    } while (0)

template <typename T>
nj_status alloc(nj_ctx* c, T** p, size_t n) {
    void* q = nullptr;
    if (n == 0) n = 1;
    cudaError_t e = cudaMalloc(&q, n * sizeof(T));
    if (e != cudaSuccess) return set_err(c, NJ_ENOMEM, "cudaMalloc(%zu) failed: %s", n * sizeof(T), cudaGetErrorString(e));
    c->allocs.push_back(q);
    *p = reinterpret_cast<T*>(q);
    return NJ_OK;
}

template <typename K>
cudaError_t set_smem_attr(K kernel) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
}

nj_status ensure_w_maps(nj_ctx* c, const uint16_t* W) {
    if (c->w_cached == W) return NJ_OK;
    if (!encode_2d(&c->tmW128, W, c->V_local, c->cfg.d, 128) || !encode_2d(&c->tmW16, W, c->V_local, c->cfg.d, 16))
        return set_err(c, NJ_ECUDA, "cuTensorMapEncodeTiled failed for W_lm");
    c->w_cached = W;
    return NJ_OK;
}

struct Plan {
    int B, N, G;
    int path;
    int npad;
    std::vector<int32_t> row_off;
};

nj_status make_plan(nj_ctx* c, const int32_t* gamma, int32_t B, Plan& pl) {
    if (!gamma) return set_err(c, NJ_EINVAL, "gamma_per_req is NULL");
    if (B < 1 || B > c->cfg.max_batch) return set_err(c, NJ_ESHAPE, "B=%d outside [1, max_batch=%d]", B, c->cfg.max_batch);
    pl.B = B;
    pl.row_off.assign((size_t)B + 1, 0);
    for (int b = 0; b < B; ++b) {
        if (gamma[b] < 0 || gamma[b] > c->cfg.gamma_max)
            return set_err(c, NJ_EINVAL, "gamma_per_req[%d]=%d outside [0, gamma_max=%d]", b, gamma[b], c->cfg.gamma_max);
        pl.row_off[b + 1] = pl.row_off[b] + gamma[b] + 1;
    }
    pl.N = pl.row_off[B];
    pl.G = pl.N - B;
    pl.npad = round16(pl.N);
    const bool fused_ok = pl.N <= kFusedMaxN && c->max_tiles <= 16 && (c->max_tiles + 1) * pl.npad <= 512 &&
                          !c->sharded();
    // staged: unsharded, or the vocab-sharded step on k_lmhead (one W-shard pass, §9)
    const bool staged_ok = pl.N <= c->staged_rows && c->logits_st != nullptr && (!c->sharded() || c->kn.lm);
    int path = c->path_opt;
    if (c->sharded() && path == NJ_PATH_AUTO) path = staged_ok ? NJ_PATH_STAGED : NJ_PATH_TWOPASS;   // phased driver
    // k_gemm_big's cost is ~per (vocab tile, token chunk) item whatever the chunk
    // width (<= 256): staged (ceil(N/256) chunks in one pass) wins only when it
    // needs fewer chunks than K-A + K-C (ceil(G/256) + ceil(B/256))
    const auto nch = [](int r) { return (r + kBigMaxT - 1) / kBigMaxT; };
    // k_lmhead (default): one pass over all rows always beats streaming W twice
    const bool staged_pays = c->kn.lm || pl.N <= kBigMaxT || nch(pl.N) < nch(pl.G) + nch(pl.B);
    if (path == NJ_PATH_AUTO)
        // fused for the smallest batches only: above kFusedAutoMaxN rows k_lmhead + the sampler
        // kernels are faster (B200: N = 32 203-208 vs 207-210 us, N = 48 210-215 vs 240-248 us;
        // N = 4 fused 193 vs 203 us)
        // q read in place from host memory (nj_verify_host, zero-copy): the staged step at
        // every size (its flat sampler reads q_i(x_i) during the GEMM's tail and a rejected
        // row's chunks from ~144 CTAs at once: N = 4 / 16 / 24 / 32 266 / 296 / 309 / 314 us
        // per call vs the fused kernel's 278 / 335 / 351 / 354, scripts/e2e_*path.py);
        // NJ_HOSTQ_FUSED=1: the fused kernel up to 48 rows (round-2 second session's rule)
        path = (c->q_remote && !c->kn.hostq_fused && staged_ok && c->kn.lm) ? NJ_PATH_STAGED
               : (fused_ok && (pl.N <= kFusedAutoMaxN || !staged_ok || !c->kn.lm ||
                               (c->q_remote && !c->qstage_active && c->kn.hostq_fused)))
                   ? NJ_PATH_FUSED
               : (staged_ok && staged_pays) ? NJ_PATH_STAGED : NJ_PATH_TWOPASS;
    if (path == NJ_PATH_FUSED && !fused_ok)
        return set_err(c, NJ_EUNSUPPORTED, "fused path needs N <= %d and TMEM room (N=%d)", kFusedMaxN, pl.N);
    if (path == NJ_PATH_STAGED && !staged_ok)
        return set_err(c, NJ_EUNSUPPORTED, "staged path needs N <= %d (N=%d)", c->staged_rows, pl.N);
    pl.path = path;
    return NJ_OK;
}

// k_sample_small (nj_sampler.cuh) takes the unsharded staged path's sampler when
// one cluster of kSmallCl CTAs per request fits the SMs
// cluster size: 16 CTAs per request for B <= 8 (one cluster per GPC at a time), 8 up to
// B = 12 (16 clusters of 8 did not all fit at once), then 4 / 2 while B * cluster <= SMs
// -- but only a size of which all B clusters are co-resident on this device (the
// driver's cudaOccupancyMaxActiveClusters at nj_create): the GPCs' SM counts differ
// between B200 parts, and a request whose cluster waits for a second wave doubles the
// sampler's time (measured 20 -> 34 us at B = 8 on a box where 16-CTA clusters did
// not all fit); a smaller cluster then takes over in one wave
int small_sampler_cl(const nj_ctx* c, int B) {
    const int f = c->kn.small_cl;
    if ((f == 2 || f == 4 || f == 8 || f == 12 || f == 16) && B * f <= c->num_sms) return f;   // tests
    int cl = (B <= 8 && c->kn.small_cl16) ? 16 : B <= 12 ? kSmallCl : (B * 4 <= c->num_sms ? 4 : 2);
    auto fits = [&](int n) { return c->small_maxcl[n] == 0 || c->small_maxcl[n] >= B; };
    if (cl == 16 && !fits(16) && c->kn.small_cl12 && fits(12)) return 12;
    while (cl > 2 && !fits(cl)) cl >>= 1;
    return cl;
}
int small_pb_for(int nchunks, int cl) {   // chunks per staged batch (two buffers)
    return std::max(1, std::min(3, (nchunks + cl - 1) / cl));
}
// NJ_SMALL_FLAT: k_sample_small<FLAT> -- no cluster, num_sms / B CTAs per request (<= 32),
// chunk masses exchanged through global memory, the request's last CTA draws; launched as
// a programmatic dependent of k_lmhead (which then triggers at its start), so its CTAs
// take the SMs the GEMM's CTAs free during the GEMM's tail
int small_flat_cpr(const nj_ctx* c, int B) { return std::max(1, std::min(32, c->num_sms / std::max(B, 1))); }
bool small_flat_on(const nj_ctx* c) { return c->kn.small_flat && c->kn.small_cl == 0; }   // NJ_SMALL_CL: clusters
int small_sampler_ctas(const nj_ctx* c, int B) { return small_flat_on(c) ? small_flat_cpr(c, B) : small_sampler_cl(c, B); }
int small_sampler_pb(const nj_ctx* c, int B) { return small_pb_for(c->nchunks, small_sampler_ctas(c, B)); }
size_t small_sampler_smem(const nj_ctx* c, int B) {   // two batch buffers of logits + q chunks
    return (size_t)2 * small_sampler_pb(c, B) * 2 * kChunk * sizeof(float);
}
bool small_sampler_ok(const nj_ctx* c, const Plan& pl) {
    const int cl = small_sampler_ctas(c, pl.B);
    return c->kn.small && pl.path == NJ_PATH_STAGED && !c->sharded() && pl.B <= c->kn.small_bmax &&
           pl.B * cl <= c->num_sms && c->nchunks <= kSmallMaxChunks && c->cfg.gamma_max + 1 <= kSmallMaxRows &&
           small_sampler_smem(c, pl.B) <= 200 * 1024;
}

ReqMeta make_meta(const Plan& pl) {
    ReqMeta m;
    m.B = pl.B;
    for (int b = 0; b <= pl.B; ++b) m.row_off[b] = pl.row_off[b];
    return m;
}

// dominant-kernel event bracket (NJ_OPT_PROFILE)
nj_status prof_begin(nj_ctx* c, cudaStream_t st, std::pair<cudaEvent_t, cudaEvent_t>& e) {
    if (!c->profile) return NJ_OK;
    if (c->ev_free.empty()) {
        cudaEvent_t a, b;
        NJ_CUDA(c, cudaEventCreate(&a));
        NJ_CUDA(c, cudaEventCreate(&b));
        c->ev_free.push_back({a, b});
    }
    e = c->ev_free.back();
    c->ev_free.pop_back();
    NJ_CUDA(c, cudaEventRecord(e.first, st));
    return NJ_OK;
}
nj_status prof_end(nj_ctx* c, cudaStream_t st, std::pair<cudaEvent_t, cudaEvent_t>& e) {
    if (!c->profile) return NJ_OK;
    NJ_CUDA(c, cudaEventRecord(e.second, st));
    c->ev.push_back(e);
    return NJ_OK;
}

template <int NPAD>
nj_status launch_fused(nj_ctx* c, cudaStream_t st, const Plan& pl, const CUtensorMap& tmH, FusedParams& fp) {
    // ring stages of GK k-blocks: one barrier round trip per GK x 16 KB of W keeps
    // the TMA stream at HBM speed (scripts/stream_test*.py: 16-KB stages reach
    // 4.75 TB/s, 48-64-KB stages 6.3-6.8 TB/s on B200).  The k-block partials of a
    // stage are drained with ONE handshake into double-buffered scratch groups,
    // which must fit in TMEM next to the resident logits (max_tiles x NPAD).
    fp.scratch_col = c->max_tiles * NPAD;
    const int spare = 512 - fp.scratch_col;
    // One accumulator partial per 4-k-block ring stage (restart every 16 MMAs,
    // the k_gemm_big accuracy) needs two NPAD-column groups of
    // scratch TMEM; without room for them (NPAD = 48) a single buffer takes
    // partials of 4 k-blocks with a per-partial handshake.
    int GK = 4;
    fp.kpd = 1;
    fp.sacc = 1;
    if (spare >= 2 * NPAD) {
        // as many one-partial groups as the spare TMEM holds: the MMAs run that
        // many stages ahead of the epilogue's per-tile work
        fp.ngroups = std::max(2, std::min(8, spare / NPAD));
        if (c->kn.fgroups > 0) fp.ngroups = std::max(2, std::min(fp.ngroups, c->kn.fgroups));
        fp.nbuf = fp.ngroups;
    } else {
        fp.ngroups = 0;
        fp.nbuf = std::max(1, std::min(8, spare / NPAD));
        fp.kpd = 4;
    }
    if (c->kn.kpd > 0) fp.kpd = c->kn.kpd;   // tuning knobs
    if (c->kn.sacc >= 0) fp.sacc = c->kn.sacc;
    if (!fp.sacc && fp.ngroups > 0) {   // one partial per k-block: GK partial slots per group
        GK = std::max(1, std::min(4, spare / (2 * NPAD)));
        fp.ngroups = 2;
        fp.nbuf = 2 * GK;
    }
    if (c->kn.kgroup > 0) GK = c->kn.kgroup;
    const size_t stage2 = (size_t)GK * (kTileBytesA + NPAD * 128);
    const int S = (int)std::min<size_t>(8, (kSmemLimit - fused_tail(NPAD, 8) - 1024) / stage2);
    fp.nstages = S;
    fp.kgroup = GK;
    // accuracy of the partials: restart every k-block -> 2e-6;
    // every 2 -> 4e-6; every 3-4 k-blocks (<= 16 MMAs) -> the k_gemm_big margin
    const int kspan = (fp.ngroups > 0 && fp.sacc) ? GK : fp.kpd;
    fp.eps_acc = (kspan == 1 ? c->eps_acc_fused : kspan == 2 ? 2.0f * c->eps_acc_fused : c->eps_acc) *
                 (float)std::max(1.0, c->inv_t);
    if (c->kn.phase_ts) {
        if (!c->phase_ts) NJ_CUDA(c, cudaMalloc(&c->phase_ts, kPhaseTsN * sizeof(unsigned long long)));
        fp.phase_ts = c->phase_ts;
    }
    const size_t smem = (size_t)S * stage2 + fused_tail(NPAD, S);
    // post-GEMM scratch in the idle ring: q slices [G (prefetch) or nq][rows_cap] fp32,
    // then partials [N][grid] float2 (phase 2) and masses [B][grid] fp64 (phase 4)
    fp.rows_cap = c->max_tiles * kTileV;
    const size_t ring = (size_t)S * stage2;
    const size_t all_q = align_up((size_t)pl.G * fp.rows_cap * 4, 16);
    fp.q_prefetch = (all_q <= ring && !c->q_remote) ? 1 : 0;
    const int nq = std::min(pl.B, pl.G);
    fp.q_bytes_cap = (int)(fp.q_prefetch ? all_q : align_up((size_t)nq * fp.rows_cap * 4, 16));
    const size_t tailb = 0;
    fp.q_vec16 = (fp.ldq % 4 == 0 && c->cfg.v_begin % 4 == 0 &&
                  (reinterpret_cast<uintptr_t>(fp.q) & 15) == 0) ? 1 : 0;
    if ((size_t)fp.q_bytes_cap + tailb > ring)
        return set_err(c, NJ_EUNSUPPORTED, "fused path: post-GEMM scratch %zu > ring %zu",
                       (size_t)fp.q_bytes_cap + tailb, ring);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c->grid);
    cfg.blockDim = dim3(kFusedThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    std::pair<cudaEvent_t, cudaEvent_t> ev;
    nj_status ps = prof_begin(c, st, ev);
    if (ps != NJ_OK) return ps;
    NJ_CUDA(c, cudaLaunchKernelEx(&cfg, k_fused_verify<NPAD>, c->tmW128, c->tmW16, tmH, fp));
    NJ_LAUNCHED(c, "k_fused_verify", st);
    return prof_end(c, st, ev);
    return NJ_OK;
}

// LM-head GEMM of the staged / two-pass paths over R contiguous rows of h
// (k_gemm_big).  rr: deal (tile, chunk) items round-robin over
// grid_rr = min(SMs, tiles) CTAs; otherwise the tile-balanced vocab split
// over c->grid (CG = 1).  CTA pairs (CG = 2) always deal (tile pair, chunk)
// items round-robin.  grid_force > 0: use that grid (several launches that
// write one partial layout).  *grid_used = CTAs that wrote partials.
template <bool WRITE, bool STATS, bool CAPTURE>
nj_status launch_lmhead(nj_ctx* c, cudaStream_t st, const uint16_t* h, int R, const GemmBigParams& in, bool rr,
                        int* grid_used, int grid_force = 0) {
    if (R <= 0) return NJ_OK;
    GemmBigParams gp = in;
    gp.R = R;
    if (gp.inv_t == 0.f) gp.inv_t = (float)c->inv_t;   // 0: the context's temperature
    const int CG = c->gemm_cg == 2 ? 2 : 1;
    // two epilogue teams (alternate items) need chunks of <= 128 columns: 2 teams x
    // 2 buffers x 128 TMEM columns
    // (on by default only when the chunks are that narrow anyway: halving 256-wide
    // chunks doubles the per-item costs, which outweighs the overlap)
    gp.nchunks = (R + c->gemm_maxt - 1) / c->gemm_maxt;
    const bool narrow = (R + gp.nchunks - 1) / gp.nchunks <= 128;
    gp.teams = (CG == 1 && (c->gemm_teams == 1 || (c->gemm_teams < 0 && narrow))) ? 2 : 1;
    if (gp.teams == 2) gp.nchunks = (R + std::min(128, c->gemm_maxt) - 1) / std::min(128, c->gemm_maxt);
    gp.chunk = (R + gp.nchunks - 1) / gp.nchunks;
    gp.chunk = CG == 2 ? (gp.chunk + 31) & ~31 : round16(gp.chunk);   // pair: each CTA a multiple-of-16 half
    gp.V_local = c->V_local;
    gp.U = c->U;
    gp.num_kb = (c->cfg.d + kBK - 1) / kBK;
    gp.v_begin = c->cfg.v_begin;
    gp.part_ld = c->pld;
    gp.ntiles_g = (c->V_local + kTileV - 1) / kTileV;
    gp.rr = (rr || gp.nchunks > 1) ? 1 : 0;
    int grid;
    if (CG == 2) {
        // pairs take (tile pair, chunk) items round-robin; as few pairs as give the same max load
        const int items = (gp.ntiles_g + 1) / 2 * gp.nchunks;
        const int np0 = std::max(1, std::min(c->num_sms / 2, items));
        const int ipp = (items + np0 - 1) / np0;
        grid = 2 * ((items + ipp - 1) / ipp);
    } else {
        grid = gp.rr ? std::max(1, std::min(c->num_sms, gp.ntiles_g)) : c->grid;
    }
    // several launches writing one partial layout share the first launch's grid
    // (CTAs without items write (-inf, 0) partials)
    if (grid_force > 0) grid = CG == 2 ? (grid_force + 1) & ~1 : grid_force;
    // ring stages of several k-blocks: the single-thread producer / MMA loops cost
    // ~600 cycles per stage, so a stage must carry more MMA work than
    // that -- 4 / 3 / 2 k-blocks for chunks of <= 64 / <= 128 / more columns (~96 KB stages)
    gp.gk = gp.chunk <= 64 ? 4 : gp.chunk <= 128 ? 3 : 2;
    if (c->kn.big_gk > 0) gp.gk = c->kn.big_gk;
    gp.ks = in.ks > 0 ? in.ks : c->gemm_ks;   // accumulator groups are counted per k-block, not per stage
    // as many accumulator buffers as TMEM holds: small chunks let the MMAs run
    // further ahead of the epilogue's per-item output
    gp.bstride = std::max(32, (gp.chunk + 31) & ~31);
    gp.nbuf = std::max(2, std::min(kBigMaxBuf, 512 / gp.bstride));
    if (gp.teams == 2) gp.nbuf &= ~1;   // an even split between the teams
    if (c->kn.big_nbuf > 0) gp.nbuf = std::max(2, std::min(gp.nbuf, c->kn.big_nbuf));
    gp.pf = c->gemm_pf;
    gp.dbg = c->kn.big_dbg;
    gp.spin = c->kn.spin;
    gp.stats_mode = c->kn.stats;
    gp.sleep_ns = c->kn.sleep_ns;
    gp.ts = nullptr;
    if (c->kn.phase_ts) {
        if (!c->phase_ts) NJ_CUDA(c, cudaMalloc(&c->phase_ts, kPhaseTsN * sizeof(unsigned long long)));
        gp.ts = c->phase_ts;
    }
    CUtensorMap tmH;
    if (!encode_2d(&tmH, h, R, c->cfg.d, gp.chunk / CG))
        return set_err(c, NJ_ECUDA, "cuTensorMapEncodeTiled failed (H)");
    const size_t stage = (size_t)gp.gk * (kTileBytesA + (size_t)(gp.chunk / CG) * 128);
    size_t tail = 4 * 4 * kBigNC * sizeof(float2) + (STATS ? (size_t)gp.teams * R * 8 : 0) +
                  (CAPTURE ? (size_t)R * 4 : 0);
    tail = align_up(tail, 8) + (2 * 8 + 2 * kBigMaxBuf) * 8 + 8;
    int S = (int)std::min<size_t>(8, (kSmemLimit - tail - 1024) / stage);
    if (c->kn.big_s > 0) S = (gp.dbg & 4) ? std::min(64, c->kn.big_s) : std::min(S, std::max(2, c->kn.big_s));
    if (S < 2) return set_err(c, NJ_EUNSUPPORTED, "k_gemm_big: not enough shared memory (R=%d)", R);
    gp.nstages = S;
    const size_t smem = ((gp.dbg & 4) ? 0 : (size_t)S * stage) + tail + ((gp.dbg & 4) ? (size_t)S * 16 : 0);
    if (CG == 2) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kBigThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        NJ_CUDA(c, cudaLaunchKernelEx(&cfg, k_gemm_big<WRITE, STATS, CAPTURE, 2>, c->tmW128, c->tmW16, tmH, gp));
    } else {
        k_gemm_big<WRITE, STATS, CAPTURE, 1><<<grid, kBigThreads, smem, st>>>(c->tmW128, c->tmW16, tmH, gp);
    }
    NJ_LAUNCHED(c, "k_gemm_big", st);
    if (grid_used) *grid_used = grid;
    return NJ_OK;
}

// k_lmhead (nj_lmhead.cuh): CTA group from the measured per-chunk cost (B200, Qwen
// shape, scripts/time_lm.py): a CTA-pair chunk of 256 token rows costs ~255 us, a
// single-CTA chunk of 128 rows ~145 us (more operand bytes per FLOP), whatever the
// number of chunks; R <= 128 is W-stream bound and single-CTA (226 vs 264 us at
// R = 128).  The tile width is the balanced width of the largest vocabulary range.
struct LmPlan {
    int cg, tile_w, w, nunits, nchunks;
};
LmPlan lm_plan(const nj_ctx* c, int R) {
    int cg = R <= kLmTok ? 1 : (1.13 * kLmTok * ((R + kLmTok - 1) / kLmTok) < 2.0 * kLmTok * ((R + 2 * kLmTok - 1) / (2 * kLmTok)) ? 1 : 2);
    if (c->kn.lm_cg == 1 || c->kn.lm_cg == 2) cg = c->kn.lm_cg;
    const int nch = (R + kLmTok * cg - 1) / (kLmTok * cg);
    const int ngroups = std::max(1, std::min(c->num_sms / cg / nch, c->U));   // units = groups x chunks
    const int upu = (c->U + ngroups - 1) / ngroups;   // 16-id units of the largest range
    const int rows = std::min(upu * kUnit, c->V_local);
    const int ntile = (rows + c->kn.lm_tw - 1) / c->kn.lm_tw;
    const int w = c->kn.lm_w > 0 ? c->kn.lm_w : ((rows + ntile - 1) / ntile + 15) & ~15;
    return LmPlan{cg, w, w, ngroups * nch, nch};
}

template <int MODE>
nj_status launch_lm(nj_ctx* c, cudaStream_t st, const uint16_t* h, const uint16_t* W, int R, LmheadParams& p,
                    int* nparts) {
    if (R <= 0) return NJ_OK;
    const LmPlan pl = lm_plan(c, R);
    const int CG = pl.cg;
    p.R = R;
    p.nchunks = pl.nchunks;
    p.V_local = c->V_local;
    p.U = c->U;
    p.num_kb = (c->cfg.d + kBK - 1) / kBK;
    p.v_begin = c->cfg.v_begin;
    p.part_ld = c->pld;
    if (p.inv_t == 0.f) p.inv_t = (float)c->inv_t;
    if (p.ks <= 0) p.ks = c->gemm_ks;
    p.tile_w = pl.tile_w;
    p.wbox = (pl.w + CG - 1) / CG;
    p.bstride = std::max(32, (pl.w + 31) & ~31);
    p.nbuf = std::max(2, std::min(kLmMaxBuf, 512 / p.bstride));
    if (c->kn.lm_nbuf > 0) p.nbuf = std::min(kLmMaxBuf, c->kn.lm_nbuf);
    if (c->kn.lm_ks > 0) p.ks = c->kn.lm_ks;
    // first accumulator group of an item: ks (NJ_LM_KS0 = 8 lets the MMAs run 12 k-blocks
    // ahead of the per-item output, -3..-4 %, but its larger CDF error put one of 10 240
    // uncertified B = 256 gamma = 5 draws outside the 1e-6 band, DESIGN.md §6 / §17)
    p.ks0 = std::max(p.ks, c->kn.lm_ks0 > 0 ? c->kn.lm_ks0 : p.ks);
    p.arv1 = c->kn.lm_arv1;
    p.sleep_ns = c->kn.lm_sleep;
    p.fence_full = c->kn.lm_fence;
    p.mma4 = c->kn.lm_mma4;
    p.pdl = (c->kn.lm_pdl || p.pdl) ? 1 : 0;   // the caller asks for it when a PDL dependent follows
    // NJ_LM_OUT_KEEP: the staged logits of a one-chunk launch (R <= 128 rows, <= 78 MB) stored with
    // an L2 evict_last hint so that the sampler's re-read hits L2
    p.out_keep = (c->kn.lm_out_keep && pl.nchunks == 1 && CG == 1) ? 1 : 0;
    p.dbg = c->kn.lm_dbg;
    p.ts = nullptr;
    if (c->kn.phase_ts) {
        if (!c->phase_ts) NJ_CUDA(c, cudaMalloc(&c->phase_ts, kPhaseTsN * sizeof(unsigned long long)));
        NJ_CUDA(c, cudaMemsetAsync(c->phase_ts, 0, kPhaseTsN * sizeof(unsigned long long), st));
        p.ts = c->phase_ts;
    }
    // one chunk: W is streamed once (evict_first); several: the other chunks of a
    // tile re-read it from L2 one item later (evict_last)
    p.w_evict_first = pl.nchunks == 1 ? 1 : 0;
    p.pf = c->kn.lm_pf >= 0 ? c->kn.lm_pf : 0;
    if (c->kn.w_evict_first >= 0) p.w_evict_first = c->kn.w_evict_first;
    if (c->lm_w_cached != W || c->lm_wbox != p.wbox) {
        if (!encode_2d(&c->tmWlm, W, c->V_local, c->cfg.d, p.wbox))
            return set_err(c, NJ_ECUDA, "cuTensorMapEncodeTiled failed (W, k_lmhead)");
        c->lm_w_cached = W;
        c->lm_wbox = p.wbox;
    }
    p.hbox = (CG == 1 && pl.nchunks == 1) ? std::min(kLmTok, (R + 7) & ~7) : kLmTok;
    CUtensorMap tmH, tmL{};
    if (!encode_2d(&tmH, h, R, c->cfg.d, p.hbox)) return set_err(c, NJ_ECUDA, "cuTensorMapEncodeTiled failed (H)");
    constexpr bool STATE = (MODE & (LM_STATS | LM_ARGMAX)) != 0, CAP = (MODE & LM_CAPTURE) != 0,
                   WR = (MODE & LM_WRITE) != 0;
    p.tma_out = WR && c->kn.lm_tma_out && (p.ld_out & 3) == 0 && (reinterpret_cast<uintptr_t>(p.logits) & 15) == 0;
    if (p.tma_out && !encode_out(&tmL, p.logits, R, c->V_local, p.ld_out))
        return set_err(c, NJ_ECUDA, "cuTensorMapEncodeTiled failed (logits)");
    const size_t nloc = kLmTok;
    p.ost_n = c->kn.lm_ost;
    size_t tail = (p.tma_out ? (size_t)kLmEpiWarps * p.ost_n * 2048 : 0) + (STATE ? 4 * nloc * 8 : 0) + (CAP ? nloc * 8 : 0);
    tail = align_up(tail, 8) + (2 * 8 + 2 * kLmMaxBuf) * 8 + 8;
    const size_t kb_bytes = (size_t)p.hbox * 128 + (size_t)p.wbox * 128;
    // CTA pairs: 2-k-block ring stages.  Every ring stage costs one tcgen05.commit, and
    // each commit stalls the tensor pipe: with no loads at all, 1-k-block stages run
    // 1.26x slower than no ring, 2-k-block stages as fast (R = 1536, interleaved A/B:
    // full kernel -7 % at R = 1536, -4 % at 768, -7 % at R = 256).
    // Single CTAs, one chunk (R <= 128, HBM-bound: C2): 2-k-block stages as well (fewer,
    // larger stages stream W faster: C2 214.1 -> 210.4 us/step, same-box
    // A/B); several single-CTA chunks too, although two 92-KB stages are all that fit
    // (interleaved A/B: R = 160 / 192 / 288 / 320 / 384 -8 / -6 / -9 / -7 / -7 %)
    p.gk = c->kn.lm_gk > 0 ? c->kn.lm_gk : 2;
    while (p.gk > 1 && (kSmemLimit - tail - 1024) / ((size_t)p.gk * kb_bytes) < 2) --p.gk;
    const size_t stage = (size_t)p.gk * kb_bytes;
    int S = (int)std::min<size_t>(8, (kSmemLimit - tail - 1024) / stage);
    if (c->kn.lm_s > 0) S = std::min(S, std::max(2, c->kn.lm_s));
    if (S < 2) return set_err(c, NJ_EUNSUPPORTED, "k_lmhead: not enough shared memory (R=%d)", R);
    p.nstages = S;
    p.nstages_mem = 0;
    if ((p.dbg & 48) == 48 && c->kn.lm_s > S) {   // probe without loads: more barrier stages than memory
        p.nstages_mem = S;
        p.nstages = std::min(c->kn.lm_s, 8);
    }
    // the MMA warp takes two 1-k-block stages per operand wait (sweep: -2..-6 % vs one)
    p.mb = c->kn.lm_mb > 0 ? std::min(c->kn.lm_mb, S - 1) : std::max(1, std::min(2, S - 2));
    const size_t smem = (size_t)(p.nstages_mem > 0 ? p.nstages_mem : p.nstages) * stage + tail;
    const int grid = pl.nunits * CG;
    if (CG == 2) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kLmThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        NJ_CUDA(c, cudaLaunchKernelEx(&cfg, k_lmhead<MODE, 2>, c->tmWlm, tmH, tmL, p));
    } else {
        k_lmhead<MODE, 1><<<grid, kLmThreads, smem, st>>>(c->tmWlm, tmH, tmL, p);
    }
    NJ_LAUNCHED(c, "k_lmhead", st);
    if (nparts) *nparts = pl.nunits / pl.nchunks;   // one partial per group and row
    return NJ_OK;
}

template <typename K, typename... Args>
cudaError_t launch_pdl_smem(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}
template <typename K, typename... Args>
cudaError_t launch_pdl(K kernel, dim3 grid, dim3 block, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// K-D: [k_sample_lse when some sample-row lse is still NaN] + k_mass over a
// grid of num_sms x resident CTAs taking (request, chunk) items round-robin.
nj_status launch_mass(nj_ctx* c, cudaStream_t st, const MassParams& mp, int B, bool need_lse, bool pdl = false) {
    if (B <= 0) return NJ_OK;
    if (need_lse) {
        k_sample_lse<<<(B + 7) / 8, 256, 0, st>>>(mp, B, const_cast<double*>(mp.s_lse));   // ctx-owned s_lse
        NJ_LAUNCHED(c, "k_sample_lse", st);
    }
    const int total = B * c->nchunks;
    const int grid = std::max(1, std::min(total, c->num_sms * c->mass_occ));
    const_cast<MassParams&>(mp).probe = c->kn.mass_probe;
    const size_t sm = mass_smem(c->mass_nst, B);
    if (pdl) {
        auto km = c->mass_nst == 2 ? k_mass<2> : c->mass_nst == 4 ? k_mass<4> : k_mass<3>;
        NJ_CUDA(c, launch_pdl_smem(km, dim3(grid), dim3(kSampThreads), sm, st, mp, B));
    } else if (c->mass_nst == 2) k_mass<2><<<grid, kSampThreads, sm, st>>>(mp, B);
    else if (c->mass_nst == 4) k_mass<4><<<grid, kSampThreads, sm, st>>>(mp, B);
    else k_mass<3><<<grid, kSampThreads, sm, st>>>(mp, B);
    NJ_LAUNCHED(c, "k_mass", st);
    return NJ_OK;
}

FbParams fb_params(nj_ctx* c, const uint16_t* hidden, const uint16_t* W, const int32_t* tok, const float* q,
                   int64_t ldq, const float* u, int32_t* acc, int32_t* nxt, const nj_debug* dbg) {
    FbParams f{};
    f.inv_t = c->inv_t;
    f.hidden = hidden;
    f.W = W;
    f.d = c->cfg.d;
    f.V_local = c->V_local;
    f.v_begin = c->cfg.v_begin;
    f.fb_count = c->fb_count();
    f.fb_list = c->fb_list();
    f.req_flags = c->req_flags();
    f.fb_logits = c->fb_logits;
    f.fb_done = c->fb_done;
    f.draft_tokens = tok;
    f.q = q;
    f.ldq = ldq;
    f.u = u;
    f.accept_len = acc;
    f.next_token = nxt;
    f.dbg_mass = dbg ? dbg->mass : nullptr;
    f.dbg_flags = dbg ? dbg->flags : nullptr;
    return f;
}

// launch with programmatic stream serialization (PDL): the kernel may start
// before its predecessor finishes and waits in-kernel (griddepcontrol.wait)
nj_status launch_fallback(nj_ctx* c, cudaStream_t st, const FbParams& f, const ReqMeta& m) {
    NJ_CUDA(c, launch_pdl(k_fb, dim3(c->num_sms * 2), dim3(256), st, f, m));
    NJ_LAUNCHED(c, "k_fb", st);
    return NJ_OK;
}


// ---------------------------------------------------------------------------
// Vocab-sharded mode (BJ config 5): host driver.
// nj_verify runs 4 phases (8 with the certified fallback) separated by small
// exchanges (nj_shard.cuh): over NCCL for one process per GPU, or as device
// copies between the members of an nj_group (single process, tests).
// ---------------------------------------------------------------------------

// NCCL is loaded at runtime (the process's libnccl.so.2 -- torch's, when torch
// is imported -- else the system one); only these entry points are used.
struct NcclId { char b[128]; };
struct NcclApi {
    int (*GetUniqueId)(NcclId*) = nullptr;
    int (*CommInitRank)(void**, int, NcclId, int) = nullptr;
    int (*CommDestroy)(void*) = nullptr;
    int (*CommCount)(const void*, int*) = nullptr;
    int (*CommUserRank)(const void*, int*) = nullptr;
    int (*AllGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
    int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(int) = nullptr;
    bool ok = false;
};
constexpr int kNcclInt8 = 0, kNcclInt32 = 2, kNcclMax = 2;

NcclApi* nccl_api() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = nullptr;
        const char* env = getenv("NJ_NCCL_LIB");
        if (env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
#define S(f, name) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, name))
        S(GetUniqueId, "ncclGetUniqueId");
        S(CommInitRank, "ncclCommInitRank");
        S(CommDestroy, "ncclCommDestroy");
        S(CommCount, "ncclCommCount");
        S(CommUserRank, "ncclCommUserRank");
        S(AllGather, "ncclAllGather");
        S(AllReduce, "ncclAllReduce");
        S(GetErrorString, "ncclGetErrorString");
#undef S
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.CommCount && api.CommUserRank &&
                 api.AllGather && api.AllReduce && api.GetErrorString;
    });
    return api.ok ? &api : nullptr;
}

// contiguous 128-row-aligned shard of rank r (rank order = ascending ids, R5)
void shard_range(int V, int n, int r, int& vb, int& ve) {
    const int64_t T = (V + kTileV - 1) / kTileV;
    vb = (int)std::min<int64_t>(V, (T * r / n) * kTileV);
    ve = (int)std::min<int64_t>(V, (T * (r + 1) / n) * kTileV);
}

// Exchange buffers of the sharded step (nj_shard.cuh): per rank
//   X2: [MB x 3 doubles (lse used, W_r, lse_r(n))] ++ [MB x slots x 2 doubles fallback stats]
//   X3: [MB int32 tokens | MB int32 flags] ++ [MB x 2 doubles fallback masses]  (3 MB doubles)
//   X4: [MB int32 tokens | MB int32 flags] (in-place MAX)
int64_t x2_stride(const nj_ctx* c) {
    const int64_t MB = c->cfg.max_batch, slots = c->cfg.gamma_max + 1;
    return 3 * MB + 2 * MB * slots;
}
int64_t x3_stride(const nj_ctx* c) { return 3 * (int64_t)c->cfg.max_batch; }

nj_status alloc_shard_ws(nj_ctx* c) {
    const int MB = c->cfg.max_batch, n = c->nranks;
    nj_status s;
    if ((s = alloc(c, &c->xs1, (size_t)c->Gmax * 2)) != NJ_OK) return s;
    if ((s = alloc(c, &c->xr1, (size_t)n * c->Gmax * 2)) != NJ_OK) return s;
    if ((s = alloc(c, &c->xs2, (size_t)x2_stride(c))) != NJ_OK) return s;
    if ((s = alloc(c, &c->xr2, (size_t)n * x2_stride(c))) != NJ_OK) return s;
    if ((s = alloc(c, &c->xs3, (size_t)x3_stride(c))) != NJ_OK) return s;
    if ((s = alloc(c, &c->xr3, (size_t)n * x3_stride(c))) != NJ_OK) return s;
    if ((s = alloc(c, &c->x6, (size_t)2 * MB)) != NJ_OK) return s;
    if ((s = alloc(c, &c->fbn, (size_t)MB)) != NJ_OK) return s;
    if ((s = alloc(c, &c->fblse, (size_t)MB)) != NJ_OK) return s;
    // the exchanges have fixed sizes (max_batch-based); entries a step does not
    // fill (unused fallback slots) are exchanged too, so start them defined
    if (cudaMemset(c->xs2, 0, sizeof(double) * (size_t)x2_stride(c)) != cudaSuccess ||
        cudaMemset(c->xs3, 0, sizeof(double) * (size_t)x3_stride(c)) != cudaSuccess ||
        cudaMemset(c->x6, 0, sizeof(int32_t) * 2 * (size_t)MB) != cudaSuccess)
        return set_err(c, NJ_ECUDA, "cudaMemset failed (exchange buffers)");
    return NJ_OK;
}

struct ShardCall {
    Plan pl;
    ReqMeta meta;
    const uint16_t* hidden;
    const uint16_t* W;
    const int32_t* tok;
    const float* q;
    int64_t ldq;
    const float* u;
    int32_t* acc;
    int32_t* nxt;
    const nj_debug* dbg;
    int certify;
    int gridA, gridC;
    MassParams mp;
};

struct XSpec {
    void* send;
    void* recv;
    size_t bytes;
    int max_i32;   // 1: in-place allreduce-MAX over bytes/4 int32
};

int shard_nphases(const ShardCall&) { return 5; }

// exchange after phase ph (false: none): X1-X3 allgather, X4 allreduce-MAX
bool shard_xchg(nj_ctx* c, const ShardCall& a, int ph, XSpec& x) {
    const size_t MB = (size_t)c->cfg.max_batch;
    switch (ph) {
        case 0: if (a.pl.G == 0) return false; x = {c->xs1, c->xr1, (size_t)a.pl.G * 16, 0}; return true;
        case 1: x = {c->xs2, c->xr2, (size_t)x2_stride(c) * 8, 0}; return true;
        case 2: x = {c->xs3, c->xr3, (size_t)x3_stride(c) * 8, 0}; return true;
        case 3: x = {c->x6, c->x6, MB * 8, 1}; return true;
        default: return false;
    }
}

nj_status shard_phase(nj_ctx* c, cudaStream_t st, ShardCall& a, int ph) {
    nj_status s = NJ_OK;
    const Plan& pl = a.pl;
    const int MB = c->cfg.max_batch, slots = c->cfg.gamma_max + 1;
    const nj_debug* dbg = a.dbg;
    FbParams f = fb_params(c, a.hidden, a.W, a.tok, a.q, a.ldq, a.u, a.acc, a.nxt, dbg);
    int32_t* x3i = reinterpret_cast<int32_t*>(c->xs3);   // [MB tokens | MB flags] of this rank
    switch (ph) {
    case 0: {   // K-A on the shard, X1 pack
        NJ_CUDA(c, cudaMemsetAsync(c->fb_block, 0, (1 + 2 * (size_t)MB) * sizeof(int32_t), st));
        if (dbg && dbg->lse) NJ_CUDA(c, cudaMemsetAsync(dbg->lse, 0xFF, (size_t)pl.N * sizeof(float), st));
        a.gridA = c->grid;
        if (pl.path == NJ_PATH_STAGED) {
            // staged step (k_lmhead over all N rows of the shard: logits, per-row statistics,
            // owned draft logits), then X1 from the draft rows' statistics
            if (pl.G > 0) NJ_CUDA(c, cudaMemsetAsync(c->dl, 0xFF, (size_t)pl.G * sizeof(double), st));   // NaN: not owned
            LmheadParams lp{};
            lp.logits = c->logits_st; lp.ld_out = c->V_local;
            lp.part_m = c->part_m; lp.part_s = c->part_s;
            lp.tok = a.tok; lp.dl = c->dl;
            lp.cap_staged = 1;
            lp.pdl = (small_flat_on(c) && small_sampler_ok(c, pl)) ? 1 : 0;   // k_sample_small<FLAT> follows
            lp.B = pl.B;
            for (int b = 0; b <= pl.B; ++b) lp.row_off[b] = pl.row_off[b];
            std::pair<cudaEvent_t, cudaEvent_t> ev;
            if ((s = prof_begin(c, st, ev)) != NJ_OK) return s;
            if ((s = launch_lm<LM_WRITE | LM_STATS | LM_CAPTURE>(c, st, a.hidden, a.W, pl.N, lp, &a.gridA)) != NJ_OK)
                return s;
            if ((s = prof_end(c, st, ev)) != NJ_OK) return s;
            if (pl.G > 0) {
                k_draft_rows<<<(pl.B + 127) / 128, 128, 0, st>>>(a.meta, c->g2row);
                NJ_LAUNCHED(c, "k_draft_rows", st);
                k_xpack1<<<(pl.G + 7) / 8, 256, 0, st>>>(c->part_m, c->part_s, c->pld, a.gridA, c->dl, pl.G, c->xs1,
                                                          c->g2row);
                NJ_LAUNCHED(c, "k_xpack1", st);
            }
            return NJ_OK;
        }
        if (pl.G > 0) {
            NJ_CUDA(c, cudaMemsetAsync(c->dl, 0xFF, (size_t)pl.G * sizeof(double), st));   // NaN: not owned
            k_gather_drafts<<<pl.G, 128, 0, st>>>(a.hidden, c->cfg.d, a.meta, c->hd);
            NJ_LAUNCHED(c, "k_gather_drafts", st);
            const bool rrA = pl.G > kBigMaxT;
            for (int r0 = 0; r0 < pl.G; r0 += kMaxStatRows) {
                const int R = std::min(kMaxStatRows, pl.G - r0);
                GemmBigParams gp{};
                gp.part_m = c->part_m + (size_t)r0 * c->pld;
                gp.part_s = c->part_s + (size_t)r0 * c->pld;
                gp.tok = a.tok + r0;
                gp.dl = c->dl + r0;
                gp.ks = c->gemm_ks_ka_cert;   // acceptance only, always certified here
                std::pair<cudaEvent_t, cudaEvent_t> ev;
                if ((s = prof_begin(c, st, ev)) != NJ_OK) return s;
                if ((s = launch_lmhead<false, true, true>(c, st, c->hd + (size_t)r0 * c->cfg.d, R, gp, rrA,
                                                          &a.gridA, r0 > 0 ? a.gridA : 0)) != NJ_OK)
                    return s;
                if ((s = prof_end(c, st, ev)) != NJ_OK) return s;
            }
            k_xpack1<<<(pl.G + 7) / 8, 256, 0, st>>>(c->part_m, c->part_s, c->pld, a.gridA, c->dl, pl.G, c->xs1,
                                                      nullptr);
            NJ_LAUNCHED(c, "k_xpack1", st);
        }
        return NJ_OK;
    }
    case 1: {   // K-B (merged lse, identical on every rank) + canonical fallback queue, K-C on the
                // shard, local masses, X2 pack, and the queued requests' fp64 logits / local stats
        AcceptParams ap{};
        ap.part_m = c->part_m; ap.part_s = c->part_s; ap.grid = a.gridA; ap.pld = c->pld; ap.dl = c->dl;
        ap.draft_tokens = a.tok; ap.q = a.q; ap.ldq = a.ldq; ap.u = a.u;
        ap.hidden = a.hidden; ap.d = c->cfg.d; ap.hs = c->hs;
        ap.accept_len = a.acc; ap.s_resid = c->s_resid; ap.s_qrow = c->s_qrow; ap.s_lse = c->s_lse;
        ap.fb_count = c->fb_count(); ap.fb_list = c->fb_list(); ap.req_flags = c->req_flags();
        ap.dbg_lse = dbg ? dbg->lse : nullptr; ap.dbg_pdraft = dbg ? dbg->p_draft : nullptr;
        ap.certify = a.certify; ap.force_fallback = c->force_fb;
        ap.eps_acc = c->eps_acc_ka_cert * (float)std::max(1.0, c->inv_t);
        ap.xr1 = c->xr1; ap.nranks = c->nranks; ap.xld = pl.G;
        const bool staged = pl.path == NJ_PATH_STAGED;
        if (staged) {   // sample row of request b = row s_row[b] of the staged logits (no K-C);
                        // a residual row keeps X1's merged lse, a bonus row this rank's lse from its
                        // own row statistics (rescaled across ranks by X2, R15)
            ap.staged = 1; ap.s_row = c->s_row; ap.hs = nullptr;
        }
        k_accept<<<(pl.B + 7) / 8, 256, 0, st>>>(ap, a.meta);
        NJ_LAUNCHED(c, "k_accept", st);
        k_qcanon<<<1, 1024, 0, st>>>(c->req_flags(), pl.B, c->fb_count(), c->fb_list(), c->force_fb);
        NJ_LAUNCHED(c, "k_qcanon", st);
        a.gridC = c->grid;
        if (!staged) {
            GemmBigParams gp{};
            gp.logits = c->logits_s; gp.ld_out = c->V_local;
            gp.part_m = c->part2_m; gp.part_s = c->part2_s;
            const bool rrC = pl.B > kBigMaxT;
            if ((s = launch_lmhead<true, true, false>(c, st, c->hs, pl.B, gp, rrC, &a.gridC)) != NJ_OK) return s;
        }
        MassParams& mp = a.mp;
        mp = MassParams{};
        mp.logits = c->logits_s; mp.ld = c->V_local; mp.V_local = c->V_local; mp.v_begin = c->cfg.v_begin;
        mp.nchunks = c->nchunks; mp.s_resid = c->s_resid; mp.s_qrow = c->s_qrow; mp.s_lse = c->s_lse;
        mp.part2_m = c->part2_m; mp.part2_s = c->part2_s; mp.grid2 = a.gridC; mp.pld2 = c->pld;
        if (staged) {
            mp.logits = c->logits_st; mp.s_row = c->s_row;
            mp.part2_m = c->part_m; mp.part2_s = c->part_s; mp.grid2 = a.gridA; mp.part2_by_row = 1;
        }
        mp.q = a.q; mp.ldq = a.ldq; mp.u = a.u; mp.stage_mode = 0; mp.cmass = c->cmass;
        mp.accept_len = a.acc; mp.next_token = x3i;
        mp.fb_count = c->fb_count(); mp.fb_list = c->fb_list(); mp.req_flags = c->req_flags();
        mp.dbg_mass = dbg ? dbg->mass : nullptr; mp.dbg_flags = nullptr;
        mp.dbg_lse = dbg ? dbg->lse : nullptr;
        mp.certify = a.certify; mp.eps_draw = c->eps_draw;
        mp.xr2 = c->xr2; mp.xstride = x2_stride(c); mp.nranks = c->nranks; mp.rank = c->rank;
        mp.xflags = x3i + MB;
        if ((s = launch_mass(c, st, mp, pl.B, true)) != NJ_OK) return s;
        k_xpack2<<<(pl.B + 7) / 8, 256, 0, st>>>(mp, pl.B, c->xs2);
        NJ_LAUNCHED(c, "k_xpack2", st);
        NJ_CUDA(c, cudaMemsetAsync(x3i + MB, 0, (size_t)MB * sizeof(int32_t), st));   // X3 flags
        k_fb_logits<<<c->num_sms * 2, 256, 0, st>>>(f, a.meta);
        NJ_LAUNCHED(c, "k_fb_logits", st);
        k_fbx_stats<<<std::min(MB, c->num_sms), 256, 0, st>>>(f, a.meta, slots, c->xs2 + 3 * (size_t)MB);
        NJ_LAUNCHED(c, "k_fbx_stats", st);
        return NJ_OK;
    }
    case 2:     // owner rank of each draw locates its token (others write -1); fp64 fallback
                // acceptance + local masses of the queued requests (X2's second part)
        k_locate<<<pl.B, kSampThreads, 0, st>>>(a.mp, a.meta);
        NJ_LAUNCHED(c, "k_locate", st);
        k_fbx_accept<<<std::min(MB, c->num_sms), 256, 0, st>>>(f, a.meta, c->xr2 + 3 * (size_t)MB, x2_stride(c),
                                                                c->nranks, slots, c->xs3 + MB, c->fbn, c->fblse);
        NJ_LAUNCHED(c, "k_fbx_accept", st);
        return NJ_OK;
    case 3:     // outputs = max over the gathered X3 tokens; the fallback's owner-rank draw
        k_xfinish2<<<1, 256, 0, st>>>(reinterpret_cast<const int32_t*>(c->xr3), c->nranks, 2 * x3_stride(c), MB,
                                      pl.B, a.nxt, dbg ? dbg->flags : nullptr);
        NJ_LAUNCHED(c, "k_xfinish2", st);
        k_fbx_locate<<<std::min(MB, c->num_sms), 256, 0, st>>>(f, a.meta, c->xr3 + MB, x3_stride(c), c->nranks,
                                                                c->rank, MB, c->fbn, c->fblse, c->x6);
        NJ_LAUNCHED(c, "k_fbx_locate", st);
        return NJ_OK;
    case 4:
        k_fbx_write<<<1, 256, 0, st>>>(f, c->fbn, c->x6, MB);
        NJ_LAUNCHED(c, "k_fbx_write", st);
        return NJ_OK;
    }
    return NJ_OK;
}

nj_status shard_call(nj_ctx* c, ShardCall& a, const uint16_t* hidden, const uint16_t* W, const int32_t* tok,
                     const float* q, int64_t ldq, const int32_t* gamma, const float* u, int32_t B, int32_t* acc,
                     int32_t* nxt, const nj_debug* dbg) {
    nj_status s = make_plan(c, gamma, B, a.pl);
    if (s != NJ_OK) return s;
    if (!hidden || !W || !u || !acc || !nxt) return set_err(c, NJ_EINVAL, "NULL device pointer");
    if (a.pl.G > 0 && (!tok || !q)) return set_err(c, NJ_EINVAL, "NULL draft buffers with G=%d", a.pl.G);
    if (ldq < c->cfg.V) return set_err(c, NJ_ESHAPE, "ldq=%lld must be >= V", (long long)ldq);
    if ((reinterpret_cast<uintptr_t>(hidden) | reinterpret_cast<uintptr_t>(W)) & 15)
        return set_err(c, NJ_ESHAPE, "hidden / W_lm must be 16-byte aligned");
    if ((s = ensure_w_maps(c, W)) != NJ_OK) return s;
    a.meta = make_meta(a.pl);
    a.hidden = hidden; a.W = W; a.tok = tok; a.q = q; a.ldq = ldq; a.u = u; a.acc = acc; a.nxt = nxt; a.dbg = dbg;
    // the sharded driver always runs its fallback phases: they also carry the
    // zero-residual-mass draws (R6), which no single rank can redo alone
    a.certify = 1;
    return NJ_OK;
}

nj_status nccl_exchange(nj_ctx* c, cudaStream_t st, const XSpec& x) {
    NcclApi* api = nccl_api();
    if (!api) return set_err(c, NJ_ENCCL, "libnccl.so.2 not loadable");
    const int r = x.max_i32 ? api->AllReduce(x.send, x.recv, x.bytes / 4, kNcclInt32, kNcclMax, c->ncomm, st)
                            : api->AllGather(x.send, x.recv, x.bytes, kNcclInt8, c->ncomm, st);
    if (r != 0) return set_err(c, NJ_ENCCL, "NCCL %s failed: %s", x.max_i32 ? "allreduce" : "allgather",
                               api->GetErrorString(r));
    return NJ_OK;
}

nj_status verify_sharded_nccl(nj_ctx* c, cudaStream_t st, const uint16_t* hidden, const uint16_t* W,
                              const int32_t* tok, const float* q, int64_t ldq, const int32_t* gamma, const float* u,
                              int32_t B, int32_t* acc, int32_t* nxt, const nj_debug* dbg) {
    ShardCall a{};
    nj_status s = shard_call(c, a, hidden, W, tok, q, ldq, gamma, u, B, acc, nxt, dbg);
    if (s != NJ_OK) return s;
    for (int ph = 0; ph < shard_nphases(a); ++ph) {
        if ((s = shard_phase(c, st, a, ph)) != NJ_OK) return s;
        XSpec x;
        if (shard_xchg(c, a, ph, x) && (s = nccl_exchange(c, st, x)) != NJ_OK) return s;
    }
    return NJ_OK;
}

}  // namespace

struct nj_group {
    std::vector<nj_ctx*> mem;
    int32_t* scratch = nullptr;   // [n][2 * max_batch] for the MAX exchange
    std::string err;
};

extern "C" {

nj_status nj_create(const nj_config* cfg, nj_ctx** out) {
    if (!cfg || !out) return set_err(nullptr, NJ_EINVAL, "NULL argument");
    *out = nullptr;
    if (cfg->d < 8 || cfg->d % 8 != 0) return set_err(nullptr, NJ_ESHAPE, "d=%d must be a positive multiple of 8", cfg->d);
    if (cfg->V < 1) return set_err(nullptr, NJ_ESHAPE, "V=%d", cfg->V);
    if (cfg->max_batch < 1 || cfg->max_batch > kMaxB)
        return set_err(nullptr, NJ_ESHAPE, "max_batch=%d outside [1, %d]", cfg->max_batch, kMaxB);
    if (cfg->gamma_max < 0 || cfg->gamma_max > 15) return set_err(nullptr, NJ_ESHAPE, "gamma_max=%d outside [0,15]", cfg->gamma_max);
    if (cfg->v_begin < 0 || cfg->v_end > cfg->V || cfg->v_begin >= cfg->v_end)
        return set_err(nullptr, NJ_ESHAPE, "bad shard [%d,%d) of V=%d", cfg->v_begin, cfg->v_end, cfg->V);
    int nranks = 1, rank = 0;
    if (cfg->nccl_comm) {
        NcclApi* api = nccl_api();
        if (!api) return set_err(nullptr, NJ_ENCCL, "vocab-sharded mode: libnccl.so.2 not loadable");
        if (api->CommCount(cfg->nccl_comm, &nranks) != 0 || api->CommUserRank(cfg->nccl_comm, &rank) != 0)
            return set_err(nullptr, NJ_ENCCL, "ncclCommCount / ncclCommUserRank failed");
        int vb, ve;
        shard_range(cfg->V, nranks, rank, vb, ve);
        if (vb != cfg->v_begin || ve != cfg->v_end)
            return set_err(nullptr, NJ_ESHAPE, "rank %d of %d must own [%d,%d) (nj_shard_range), got [%d,%d)", rank,
                           nranks, vb, ve, cfg->v_begin, cfg->v_end);
    }
    // (the fused kernel keeps every lane's CTA partials in registers: grid <= 160)
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return set_err(nullptr, NJ_ECUDA, "no CUDA device visible (libnj has no CPU fallback)");
    if (cfg->device < 0 || cfg->device >= ndev) return set_err(nullptr, NJ_EINVAL, "device %d of %d", cfg->device, ndev);
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, cfg->device) != cudaSuccess) return set_err(nullptr, NJ_ECUDA, "cudaGetDeviceProperties failed");
    if (prop.major != 10 || prop.minor != 0)
        return set_err(nullptr, NJ_ECUDA, "device %d is sm_%d%d; libnj is built for sm_100a only", cfg->device, prop.major, prop.minor);
    if (cudaSetDevice(cfg->device) != cudaSuccess) return set_err(nullptr, NJ_ECUDA, "cudaSetDevice failed");
    if (!get_encode_fn()) return set_err(nullptr, NJ_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");

    nj_ctx* c = new nj_ctx();
    c->cfg = *cfg;
    c->kn = read_knobs();
    c->nranks = nranks;
    c->rank = rank;
    c->ncomm = cfg->nccl_comm;
    c->V_local = cfg->v_end - cfg->v_begin;
    c->num_sms = prop.multiProcessorCount;
    c->U = (c->V_local + kUnit - 1) / kUnit;
    // tile-balanced persistent grid: every CTA gets ceil(T/grid) or fewer whole
    // 128-row tiles (V = 152064 -> 132 CTAs x 9 tiles; a ragged 148-CTA split
    // leaves 16-row tail tiles that run latency-bound and finish last)
    {
        const int T = (c->V_local + kTileV - 1) / kTileV;
        const int tpc = (T + c->num_sms - 1) / c->num_sms;
        c->grid = std::max(1, std::min(c->U, (T + tpc - 1) / tpc));
        if (const char* e = getenv("NJ_GRID")) c->grid = std::max(1, std::min(c->U, atoi(e)));
    }
    const int upc = (c->U + c->grid - 1) / c->grid;
    c->max_tiles = (upc * kUnit + kTileV - 1) / kTileV;
    c->nchunks = (c->V_local + kChunk - 1) / kChunk;
    const int MB = cfg->max_batch, GM = cfg->gamma_max;
    c->Nmax = MB * (GM + 1);
    c->Gmax = std::max(1, MB * GM);
    nj_status s = NJ_OK;
    c->pld = std::max(c->grid, c->num_sms);
    if (const char* e = getenv("NJ_KS")) c->gemm_ks = std::max(1, atoi(e));
    if (const char* e = getenv("NJ_KS_KA")) c->gemm_ks_ka = std::max(1, atoi(e));
    if (const char* e = getenv("NJ_KS_KA_CERT")) c->gemm_ks_ka_cert = std::max(1, atoi(e));
    if (const char* e = getenv("NJ_CG")) c->gemm_cg = atoi(e);
    if (const char* e = getenv("NJ_PF")) c->gemm_pf = std::max(0, atoi(e));
    if (const char* e = getenv("NJ_BIG_MAXT")) c->gemm_maxt = std::min(256, std::max(32, atoi(e)));
    if (const char* e = getenv("NJ_TEAMS")) c->gemm_teams = atoi(e) != 0;
    const size_t g = (size_t)c->grid, gp_ = (size_t)c->pld;
#define A(ptr, n) if ((s = alloc(c, &c->ptr, (n))) != NJ_OK) { nj_destroy(c); return s; }
    A(part_m, (size_t)c->Nmax * gp_);
    A(part_s, (size_t)c->Nmax * gp_);
    A(part2_m, (size_t)MB * gp_);
    A(part2_s, (size_t)MB * gp_);
    A(dl, (size_t)c->Gmax);
    A(row_lse, (size_t)std::max(c->Nmax, c->Gmax));
    A(wpart, (size_t)MB * g);
    A(s_lse, (size_t)MB);
    A(lse_tmp, (size_t)MB);
    A(cmass, (size_t)MB * c->nchunks);
    A(fb_logits, (size_t)c->Nmax * c->V_local);
    A(hd, (size_t)c->Gmax * cfg->d);
    A(hs, (size_t)MB * cfg->d);
    A(logits_s, (size_t)MB * c->V_local);
    c->staged_rows = std::min(c->Nmax, c->kn.lm ? kStagedMaxRows : kStagedMaxN);
    A(logits_st, (size_t)c->staged_rows * c->V_local);
    A(s_resid, (size_t)MB);
    A(s_qrow, (size_t)MB);
    A(fb_block, (size_t)1 + 3 * MB);
    A(bar, 2);
    A(fb_done, 1);
    A(scratch_i, (size_t)MB);
    A(s_row, (size_t)MB);
    A(amax, (size_t)c->Nmax);
    A(g2row, (size_t)c->Gmax);
#undef A
    if (c->ncomm && (s = alloc_shard_ws(c)) != NJ_OK) { nj_destroy(c); return s; }
    if (cudaMemset(c->bar, 0, 2 * sizeof(uint32_t)) != cudaSuccess || cudaMemset(c->fb_done, 0, sizeof(int32_t)) != cudaSuccess ||
        cudaMemset(c->fb_block, 0, (1 + 3 * MB) * sizeof(int32_t)) != cudaSuccess) {
        nj_destroy(c);
        return set_err(nullptr, NJ_ECUDA, "cudaMemset failed");
    }
    cudaError_t e = cudaSuccess;
    e = e ? e : set_smem_attr(k_fused_verify<16>);
    e = e ? e : set_smem_attr(k_fused_verify<32>);
    e = e ? e : set_smem_attr(k_fused_verify<48>);
    e = e ? e : set_smem_attr(k_gemm_big<false, true, true, 1>);
    e = e ? e : set_smem_attr(k_gemm_big<true, true, false, 1>);
    e = e ? e : set_smem_attr(k_gemm_big<true, true, true, 1>);
    e = e ? e : set_smem_attr(k_gemm_big<false, true, true, 2>);
    e = e ? e : set_smem_attr(k_gemm_big<true, true, false, 2>);
    e = e ? e : set_smem_attr(k_gemm_big<true, true, true, 2>);
    e = e ? e : set_smem_attr(k_lmhead<LM_WRITE | LM_STATS | LM_CAPTURE, 1>);
    e = e ? e : set_smem_attr(k_lmhead<LM_WRITE | LM_STATS | LM_CAPTURE, 2>);
    e = e ? e : set_smem_attr(k_lmhead<LM_WRITE | LM_STATS, 1>);
    e = e ? e : set_smem_attr(k_lmhead<LM_WRITE | LM_STATS, 2>);
    e = e ? e : set_smem_attr(k_lmhead<LM_ARGMAX, 1>);
    e = e ? e : cudaFuncSetAttribute(k_sample_small<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    e = e ? e : cudaFuncSetAttribute(k_sample_small<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    e = e ? e : cudaFuncSetAttribute(k_sample_small<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cl : {2, 4, 8, 12, 16}) {
        if (e) break;
        cudaLaunchConfig_t oc = {};
        oc.gridDim = dim3(cl);
        oc.blockDim = dim3(kSampThreads);
        oc.dynamicSmemBytes = (size_t)2 * small_pb_for(c->nchunks, cl) * 2 * kChunk * sizeof(float);
        cudaLaunchAttribute oa[1];
        oa[0].id = cudaLaunchAttributeClusterDimension;
        oa[0].val.clusterDim.x = cl;
        oa[0].val.clusterDim.y = 1;
        oa[0].val.clusterDim.z = 1;
        oc.attrs = oa;
        oc.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, k_sample_small<false>, &oc) == cudaSuccess) c->small_maxcl[cl] = n;
        else (void)cudaGetLastError();   // unknown: keep the measured default size
    }
    if (getenv("NJ_SMALL_INFO"))
        fprintf(stderr, "[nj] k_sample_small co-resident clusters: 2:%d 4:%d 8:%d 12:%d 16:%d\n", c->small_maxcl[2],
                c->small_maxcl[4], c->small_maxcl[8], c->small_maxcl[12], c->small_maxcl[16]);
    e = e ? e : set_smem_attr(k_lmhead<LM_ARGMAX, 2>);
    if (const char* ev = getenv("NJ_MASS_NST")) c->mass_nst = std::min(4, std::max(2, atoi(ev)));
    e = e ? e : cudaFuncSetAttribute(k_mass<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mass_smem(2, c->cfg.max_batch));
    e = e ? e : cudaFuncSetAttribute(k_mass<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mass_smem(3, c->cfg.max_batch));
    e = e ? e : cudaFuncSetAttribute(k_mass<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mass_smem(4, c->cfg.max_batch));
    e = e ? e : cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                    &c->mass_occ, c->mass_nst == 2 ? k_mass<2> : c->mass_nst == 4 ? k_mass<4> : k_mass<3>, kSampThreads,
                    mass_smem(c->mass_nst, c->cfg.max_batch));
    if (e != cudaSuccess) {
        nj_destroy(c);
        return set_err(nullptr, NJ_ECUDA, "cudaFuncSetAttribute failed: %s", cudaGetErrorString(e));
    }
    if (const char* ev = getenv("NJ_MASS_OCC")) c->mass_occ = std::max(1, atoi(ev));
    c->mass_occ = std::max(1, c->mass_occ);
    *out = c;
    return NJ_OK;
}

void nj_destroy(nj_ctx* c) {
    if (!c) return;
    for (auto& e : c->ev) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
    for (auto& e : c->ev_free) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
    if (c->ev_qstage) cudaEventDestroy(c->ev_qstage);
    if (c->cstream) cudaStreamDestroy(c->cstream);
    for (void* p : c->allocs) cudaFree(p);
    delete c;
}

const char* nj_last_error(const nj_ctx* c) { return c ? c->err.c_str() : g_create_error.c_str(); }

nj_status nj_set_option(nj_ctx* c, nj_option opt, int64_t v) {
    if (!c) return NJ_EINVAL;
    switch (opt) {
        case NJ_OPT_PATH:
            if (v < NJ_PATH_AUTO || v > NJ_PATH_STAGED) return set_err(c, NJ_EINVAL, "bad path %lld", (long long)v);
            c->path_opt = (int)v;
            return NJ_OK;
        case NJ_OPT_CERTIFY: c->certify = v != 0; return NJ_OK;
        case NJ_OPT_FORCE_FALLBACK: c->force_fb = v != 0; return NJ_OK;
        case NJ_OPT_PROFILE: c->profile = v != 0; return NJ_OK;
        case NJ_OPT_Q_ZERO_COPY: c->q_zero_copy = v != 0; return NJ_OK;
        case NJ_OPT_Q_STAGE_ROWS: c->q_stage_opt = (int)std::max<int64_t>(-1, std::min<int64_t>(v, 256)); return NJ_OK;
    }
    return set_err(c, NJ_EINVAL, "unknown option %d", (int)opt);
}

nj_status nj_set_temperature(nj_ctx* c, double temperature) {
    if (!c) return NJ_EINVAL;
    if (!(temperature > 0.0) || !(temperature <= 1e6))
        return set_err(c, NJ_EINVAL, "temperature %g outside (0, 1e6] (T -> 0 is nj_verify_greedy)", temperature);
    c->temperature = temperature;
    c->inv_t = 1.0 / temperature;
    return NJ_OK;
}

nj_status nj_debug_phase_times(nj_ctx* c, unsigned long long* host_out, int32_t n) {
    if (!c || !c->phase_ts) return NJ_EINVAL;
    NJ_CUDA(c, cudaMemcpy(host_out, c->phase_ts, sizeof(unsigned long long) * std::min(n, kPhaseTsN), cudaMemcpyDeviceToHost));
    return NJ_OK;
}

nj_status nj_kernel_time(nj_ctx* c, double* ms_total, int64_t* launches, int32_t reset) {
    if (!c) return NJ_EINVAL;
    for (auto& e : c->ev) {
        NJ_CUDA(c, cudaEventSynchronize(e.second));
        float ms = 0.f;
        NJ_CUDA(c, cudaEventElapsedTime(&ms, e.first, e.second));
        c->prof_ms += ms;
        c->prof_n += 1;
        c->ev_free.push_back(e);
    }
    c->ev.clear();
    if (ms_total) *ms_total = c->prof_ms;
    if (launches) *launches = c->prof_n;
    if (reset) { c->prof_ms = 0.0; c->prof_n = 0; }
    return NJ_OK;
}

nj_status nj_plan(nj_ctx* c, const int32_t* gamma, int32_t B, int32_t* path_out, int32_t* launches_out) {
    if (!c) return NJ_EINVAL;
    Plan pl;
    nj_status s = make_plan(c, gamma, B, pl);
    if (s != NJ_OK) return s;
    int n = 0;
    if (c->sharded()) {
        // gather + K-A + pack1; accept, qcanon, K-C, sample_lse, mass, pack2, fb_logits, fbx_stats;
        // locate, fbx_accept; xfinish2, fbx_locate; fbx_write
        if (pl.path == NJ_PATH_STAGED)   // k_lmhead (+ draft_rows + pack1); accept, qcanon, sample_lse,
                                         // mass, pack2, fb_logits, fbx_stats; ...
            n = 1 + (pl.G > 0 ? 2 : 0) + 7 + 2 + 2 + 1;
        else
            n = (pl.G > 0 ? 1 + ((pl.G + kMaxStatRows - 1) / kMaxStatRows) + 1 : 0) + 8 + 2 + 2 + 1;
        if (path_out) *path_out = pl.path;
        if (launches_out) *launches_out = n;
        return NJ_OK;
    }
    if (pl.path == NJ_PATH_FUSED) n = 1;
    else if (pl.path == NJ_PATH_STAGED)   // GEMM, [row lse,] accept, mass, locate | GEMM, k_sample_small
        n = small_sampler_ok(c, pl) ? 2 : pl.N > c->kn.inline_lse ? 5 : 4;
    else n = (pl.G > 0 ? 2 * ((pl.G + kMaxStatRows - 1) / kMaxStatRows) + 1 : 0) + 4;   // gather+KA, row lse, KB, KC, KD1, KD2
    n += 1;   // k_fb (every call; exits at once on an empty queue)
    if (path_out) *path_out = pl.path;
    if (launches_out) *launches_out = n;
    return NJ_OK;
}

nj_status nj_verify(nj_ctx* c, void* stream, const uint16_t* hidden, const uint16_t* W_lm,
                    const int32_t* draft_tokens, const float* draft_probs, int64_t ldq,
                    const int32_t* gamma_per_req, const float* uniforms, int32_t B,
                    int32_t* accept_len, int32_t* next_token, const nj_debug* dbg) {
    if (!c) return NJ_EINVAL;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (c->in_group) return set_err(c, NJ_EINVAL, "nj_group member: call nj_group_verify");
    if (c->ncomm)
        return verify_sharded_nccl(c, st, hidden, W_lm, draft_tokens, draft_probs, ldq, gamma_per_req, uniforms, B,
                                   accept_len, next_token, dbg);
    Plan pl;
    nj_status s = make_plan(c, gamma_per_req, B, pl);
    if (s != NJ_OK) return s;
    if (!hidden || !W_lm || !uniforms || !accept_len || !next_token)
        return set_err(c, NJ_EINVAL, "NULL device pointer");
    if (pl.G > 0 && (!draft_tokens || !draft_probs)) return set_err(c, NJ_EINVAL, "NULL draft buffers with G=%d", pl.G);
    if (ldq < c->cfg.V) return set_err(c, NJ_ESHAPE, "ldq=%lld must be >= V", (long long)ldq);
    if ((reinterpret_cast<uintptr_t>(hidden) | reinterpret_cast<uintptr_t>(W_lm)) & 15)
        return set_err(c, NJ_ESHAPE, "hidden / W_lm must be 16-byte aligned");
    if ((s = ensure_w_maps(c, W_lm)) != NJ_OK) return s;
    const ReqMeta meta = make_meta(pl);
    const int certify = c->certify || c->force_fb;

    if (pl.path == NJ_PATH_FUSED) {
        CUtensorMap tmH;
        if (!encode_2d(&tmH, hidden, pl.N, c->cfg.d, pl.npad))
            return set_err(c, NJ_ECUDA, "cuTensorMapEncodeTiled failed (hidden)");
        FusedParams fp{};
        fp.B = pl.B; fp.N = pl.N; fp.G = pl.G;
        fp.V_local = c->V_local; fp.v_begin = c->cfg.v_begin; fp.U = c->U;
        fp.num_kb = (c->cfg.d + kBK - 1) / kBK;
        fp.draft_tokens = draft_tokens; fp.q = draft_probs; fp.ldq = ldq; fp.u = uniforms;
        fp.accept_len = accept_len; fp.next_token = next_token;
        fp.part_m = c->part_m; fp.part_s = c->part_s; fp.dl = c->dl; fp.wpart = c->wpart;
        fp.bar = c->bar;
        fp.fb_count = c->fb_count(); fp.fb_list = c->fb_list(); fp.req_flags = c->req_flags();
        fp.dbg_lse = dbg ? dbg->lse : nullptr; fp.dbg_pdraft = dbg ? dbg->p_draft : nullptr;
        fp.dbg_mass = dbg ? dbg->mass : nullptr; fp.dbg_flags = dbg ? dbg->flags : nullptr;
        fp.certify = certify; fp.force_fallback = c->force_fb;
        fp.eps_acc = c->eps_acc_fused * (float)std::max(1.0, c->inv_t); fp.eps_draw = c->eps_draw_fused;
        fp.inv_t = c->inv_t;
        for (int b = 0; b <= pl.B; ++b) fp.row_off[b] = pl.row_off[b];
        if (pl.npad == 16) s = launch_fused<16>(c, st, pl, tmH, fp);
        else if (pl.npad == 32) s = launch_fused<32>(c, st, pl, tmH, fp);
        else s = launch_fused<48>(c, st, pl, tmH, fp);
        if (s != NJ_OK) return s;
    } else if (pl.path == NJ_PATH_STAGED) {
        // one GEMM pass over all N rows: per-row stats, draft-logit capture, and every
        // row's fp32 logits stored with an L2 evict_last policy (W streams evict_first)
        // the fallback block (queue, flags, the flat sampler's arrival counters) is zeroed by
        // k_lmhead's first CTA (NJ_LM_ZERO; no memset node in the step) or by a memset
        const bool zero_in_lm = c->kn.lm && c->kn.lm_zero;
        if (!zero_in_lm)
            NJ_CUDA(c, cudaMemsetAsync(c->fb_block, 0, (1 + 3 * (size_t)c->cfg.max_batch) * sizeof(int32_t), st));
        if (dbg && dbg->lse) NJ_CUDA(c, cudaMemsetAsync(dbg->lse, 0xFF, (size_t)pl.N * sizeof(float), st));
        GemmBigParams gp{};
        gp.logits = c->logits_st; gp.ld_out = c->V_local;
        gp.part_m = c->part_m; gp.part_s = c->part_s;
        gp.tok = draft_tokens; gp.dl = c->dl;
        gp.use_row_g = 1;
        gp.w_evict_first = pl.N <= kBigMaxT ? 1 : 0;   // two chunks re-read W tiles from L2
        if (c->kn.w_evict_first >= 0) gp.w_evict_first = c->kn.w_evict_first;
        if (!c->kn.lm)
            for (int b = 0; b < pl.B; ++b)
                for (int r = pl.row_off[b]; r < pl.row_off[b + 1]; ++r)
                    gp.row_g[r] = r + 1 < pl.row_off[b + 1] ? r - b : -1;
        std::pair<cudaEvent_t, cudaEvent_t> ev;
        if ((s = prof_begin(c, st, ev)) != NJ_OK) return s;
        int gridA = c->grid;
        if (c->kn.lm) {
            LmheadParams lp{};
            lp.logits = c->logits_st; lp.ld_out = c->V_local;
            lp.part_m = c->part_m; lp.part_s = c->part_s;
            lp.tok = draft_tokens; lp.dl = c->dl;
            lp.cap_staged = 1;
            lp.pdl = (small_flat_on(c) && small_sampler_ok(c, pl)) ? 1 : 0;   // k_sample_small<FLAT> follows
            if (zero_in_lm) {
                lp.zero_ptr = c->fb_block;
                lp.zero_n = 1 + 3 * c->cfg.max_batch;
            }
            lp.B = pl.B;
            for (int b = 0; b <= pl.B; ++b) lp.row_off[b] = pl.row_off[b];
            // small batches: the q rows into L2 during the GEMM (the sampler reads the rejected
            // ones right after); device-resident q of a 16-byte-aligned pitch only
            if (c->kn.qpf && small_sampler_ok(c, pl) && pl.G > 0 && !c->q_remote && (ldq & 3) == 0 &&
                (reinterpret_cast<uintptr_t>(draft_probs) & 15) == 0 && (size_t)pl.G * ldq * 4 <= (32u << 20)) {
                lp.qpf = draft_probs + c->cfg.v_begin; lp.qpf_ld = ldq; lp.qpf_rows = pl.G; lp.qpf_cols = c->V_local;
            }
            if ((s = launch_lm<LM_WRITE | LM_STATS | LM_CAPTURE>(c, st, hidden, W_lm, pl.N, lp, &gridA)) != NJ_OK)
                return s;
        } else if ((s = launch_lmhead<true, true, true>(c, st, hidden, pl.N, gp, false, &gridA)) != NJ_OK) {
            return s;
        }
        if ((s = prof_end(c, st, ev)) != NJ_OK) return s;
        AcceptParams ap{};
        ap.part_m = c->part_m; ap.part_s = c->part_s; ap.grid = gridA; ap.pld = c->pld; ap.dl = c->dl;
        ap.draft_tokens = draft_tokens; ap.q = draft_probs; ap.ldq = ldq; ap.u = uniforms;
        ap.hidden = hidden; ap.d = c->cfg.d; ap.hs = nullptr;
        ap.accept_len = accept_len; ap.s_resid = c->s_resid; ap.s_qrow = c->s_qrow; ap.s_lse = c->s_lse;
        ap.fb_count = c->fb_count(); ap.fb_list = c->fb_list(); ap.req_flags = c->req_flags();
        ap.dbg_lse = dbg ? dbg->lse : nullptr; ap.dbg_pdraft = dbg ? dbg->p_draft : nullptr;
        ap.certify = certify; ap.force_fallback = c->force_fb; ap.eps_acc = c->eps_acc * (float)std::max(1.0, c->inv_t);
        ap.staged = 1; ap.s_row = c->s_row;
        if (small_sampler_ok(c, pl)) {
            // small batch: acceptance, chunk masses and the draw in one clustered launch
            MassParams mp{};
            mp.logits = c->logits_st; mp.ld = c->V_local; mp.V_local = c->V_local; mp.v_begin = c->cfg.v_begin;
            mp.nchunks = c->nchunks; mp.q = draft_probs; mp.ldq = ldq; mp.u = uniforms;
            mp.accept_len = accept_len; mp.next_token = next_token;
            mp.fb_count = c->fb_count(); mp.fb_list = c->fb_list(); mp.req_flags = c->req_flags();
            mp.dbg_mass = dbg ? dbg->mass : nullptr; mp.dbg_flags = dbg ? dbg->flags : nullptr;
            mp.dbg_lse = dbg ? dbg->lse : nullptr;
            mp.certify = certify; mp.eps_draw = c->eps_draw;
            mp.small_pb = small_sampler_pb(c, pl.B);
            mp.ts = c->kn.phase_ts ? c->phase_ts : nullptr;   // cleared with k_lmhead's stamps (a memset
                                                                  // here would break the PDL edge)
            mp.pdl_trigger = c->kn.small_trig;
            mp.small_reuse = c->kn.small_reuse;
            if (c->qstage_active) {
                // nj_verify_host staged the likely sample rows over the copy stream during the GEMM
                NJ_CUDA(c, cudaStreamWaitEvent(st, c->ev_qstage, 0));
                mp.q_loc = c->st_q;
                for (int i = 0; i < 4; ++i) mp.q_loc_mask[i] = c->qstage_mask[i];
            }
            // NJ_SMALL_PF: 1 candidate logits + q rows into L2 after the wait, 2 (flat sampler) the
            // candidate q rows before it (device-resident q of a 16-byte-aligned pitch only)
            mp.pf_rows = (!c->q_remote && (ldq & 3) == 0 && (c->V_local & 3) == 0 &&
                          (reinterpret_cast<uintptr_t>(draft_probs) & 15) == 0) ? c->kn.small_pf : 0;
            if (small_flat_on(c)) {
                mp.flat_cpr = small_flat_cpr(c, pl.B);
                mp.cm_glob = c->cmass;
                mp.cm_cnt = c->small_cnt();
                if (c->kn.small_coop) {
                    // cooperative: the runtime guarantees the B x CL CTAs are co-resident (the
                    // per-request barrier of the flat mode relies on it); PDL as above
                    cudaLaunchConfig_t cfg = {};
                    cfg.gridDim = dim3(pl.B * mp.flat_cpr);
                    cfg.blockDim = dim3(kSampThreads);
                    cfg.dynamicSmemBytes = small_sampler_smem(c, pl.B);
                    cfg.stream = st;
                    cudaLaunchAttribute at[2];
                    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                    at[0].val.programmaticStreamSerializationAllowed = 1;
                    at[1].id = cudaLaunchAttributeCooperative;
                    at[1].val.cooperative = 1;
                    cfg.attrs = at;
                    cfg.numAttrs = 2;
                    NJ_CUDA(c, cudaLaunchKernelEx(&cfg, k_sample_small<true>, ap, mp, meta));
                } else {
                    NJ_CUDA(c, launch_pdl_smem(k_sample_small<true>, dim3(pl.B * mp.flat_cpr), dim3(kSampThreads),
                                               small_sampler_smem(c, pl.B), st, ap, mp, meta));
                }
                NJ_LAUNCHED(c, "k_sample_small", st);
                goto fallback;
            }
            cudaLaunchConfig_t cfg = {};
            const int cl = small_sampler_cl(c, pl.B);
            cfg.gridDim = dim3(pl.B * cl);
            cfg.blockDim = dim3(kSampThreads);
            cfg.dynamicSmemBytes = small_sampler_smem(c, pl.B);
            cfg.stream = st;
            cudaLaunchAttribute at[2];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cl;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[1].val.programmaticStreamSerializationAllowed = c->kn.small_pdl ? 1 : 0;
            cfg.attrs = at;
            cfg.numAttrs = 2;
            NJ_CUDA(c, cudaLaunchKernelEx(&cfg, k_sample_small<false>, ap, mp, meta));
            NJ_LAUNCHED(c, "k_sample_small", st);
            goto fallback;
        }
        // small batches: k_accept merges its rows' statistics itself (one launch fewer)
        // (NJ_PDL_CHAIN: the sampler kernels launched as programmatic dependents, pdl_enter)
        const bool pdl = c->kn.pdl_chain != 0;
        if (pl.N > c->kn.inline_lse) {
            if (pdl) NJ_CUDA(c, launch_pdl(k_lse_rows, dim3((pl.N + 7) / 8), dim3(256), st, (const float*)c->part_m,
                                           (const float*)c->part_s, c->pld, gridA, pl.N, c->row_lse));
            else k_lse_rows<<<(pl.N + 7) / 8, 256, 0, st>>>(c->part_m, c->part_s, c->pld, gridA, pl.N, c->row_lse);
            NJ_LAUNCHED(c, "k_lse_rows", st);
            ap.pre_lse = c->row_lse;
        }
        if (pdl) NJ_CUDA(c, launch_pdl(k_accept, dim3((pl.B + 7) / 8), dim3(256), st, ap, meta));
        else k_accept<<<(pl.B + 7) / 8, 256, 0, st>>>(ap, meta);
        NJ_LAUNCHED(c, "k_accept", st);
        MassParams mp{};
        mp.logits = c->logits_st; mp.ld = c->V_local; mp.s_row = c->s_row;
        mp.V_local = c->V_local; mp.v_begin = c->cfg.v_begin;
        mp.nchunks = c->nchunks; mp.s_resid = c->s_resid; mp.s_qrow = c->s_qrow; mp.s_lse = c->s_lse;
        mp.part2_m = c->part_m; mp.part2_s = c->part_s; mp.grid2 = gridA; mp.pld2 = c->pld;
        mp.q = draft_probs; mp.ldq = ldq; mp.u = uniforms; mp.stage_mode = 0; mp.cmass = c->cmass;
        mp.accept_len = accept_len; mp.next_token = next_token;
        mp.fb_count = c->fb_count(); mp.fb_list = c->fb_list(); mp.req_flags = c->req_flags();
        mp.dbg_mass = dbg ? dbg->mass : nullptr; mp.dbg_flags = dbg ? dbg->flags : nullptr;
        mp.dbg_lse = dbg ? dbg->lse : nullptr;
        mp.certify = certify; mp.eps_draw = c->eps_draw;
        if ((s = launch_mass(c, st, mp, pl.B, false, pdl)) != NJ_OK) return s;
        if (pdl) NJ_CUDA(c, launch_pdl(k_locate, dim3(pl.B), dim3(kSampThreads), st, mp, meta));
        else k_locate<<<pl.B, kSampThreads, 0, st>>>(mp, meta);
        NJ_LAUNCHED(c, "k_locate", st);
    } else {
        NJ_CUDA(c, cudaMemsetAsync(c->fb_block, 0, (1 + 2 * (size_t)c->cfg.max_batch) * sizeof(int32_t), st));
        if (dbg && dbg->lse) NJ_CUDA(c, cudaMemsetAsync(dbg->lse, 0xFF, (size_t)pl.N * sizeof(float), st));
        // K-A: stats GEMM over the draft rows (gathered contiguous), draft-logit capture;
        // all K-A launches share one partial layout (round-robin mode when G > 256)
        const bool rrA = pl.G > kBigMaxT;
        int gridA = c->grid;
        if (pl.G > 0) {
            k_gather_drafts<<<pl.G, 128, 0, st>>>(hidden, c->cfg.d, meta, c->hd);
            NJ_LAUNCHED(c, "k_gather_drafts", st);
            for (int r0 = 0; r0 < pl.G; r0 += kMaxStatRows) {
                const int R = std::min(kMaxStatRows, pl.G - r0);
                GemmBigParams gp{};
                gp.part_m = c->part_m + (size_t)r0 * c->pld;
                gp.part_s = c->part_s + (size_t)r0 * c->pld;
                gp.tok = draft_tokens + r0;
                gp.dl = c->dl + r0;
                // acceptance only: cheaper drains; with the certificate on,
                // a longer restart period whose error the wider certificate covers
                gp.ks = certify ? c->gemm_ks_ka_cert : c->gemm_ks_ka;
                std::pair<cudaEvent_t, cudaEvent_t> ev;
                if ((s = prof_begin(c, st, ev)) != NJ_OK) return s;
                if ((s = launch_lmhead<false, true, true>(c, st, c->hd + (size_t)r0 * c->cfg.d, R, gp, rrA,
                                                          &gridA, r0 > 0 ? gridA : 0)) != NJ_OK)
                    return s;
                if ((s = prof_end(c, st, ev)) != NJ_OK) return s;
            }
        }
        // K-B: acceptance, first rejection, sample-row gather
        AcceptParams ap{};
        ap.part_m = c->part_m; ap.part_s = c->part_s; ap.grid = gridA; ap.pld = c->pld; ap.dl = c->dl;
        ap.draft_tokens = draft_tokens; ap.q = draft_probs; ap.ldq = ldq; ap.u = uniforms;
        ap.hidden = hidden; ap.d = c->cfg.d; ap.hs = c->hs;
        ap.accept_len = accept_len; ap.s_resid = c->s_resid; ap.s_qrow = c->s_qrow; ap.s_lse = c->s_lse;
        ap.fb_count = c->fb_count(); ap.fb_list = c->fb_list(); ap.req_flags = c->req_flags();
        ap.dbg_lse = dbg ? dbg->lse : nullptr; ap.dbg_pdraft = dbg ? dbg->p_draft : nullptr;
        ap.certify = certify; ap.force_fallback = c->force_fb;
        ap.eps_acc = (certify ? c->eps_acc_ka_cert : c->eps_acc_ka) * (float)std::max(1.0, c->inv_t);
        ap.lse_sample_from_c = 1;
        if (pl.G > 0) {
            k_lse_rows<<<(pl.G + 7) / 8, 256, 0, st>>>(c->part_m, c->part_s, c->pld, gridA, pl.G, c->row_lse);
            NJ_LAUNCHED(c, "k_lse_rows", st);
            ap.pre_lse = c->row_lse;
        }
        k_accept<<<(pl.B + 7) / 8, 256, 0, st>>>(ap, meta);
        NJ_LAUNCHED(c, "k_accept", st);
        // K-C: sample-row GEMM -> fp32 logits [B, V_local] + stats (bonus-row lse)
        int gridC = c->grid;
        {
            GemmBigParams gp{};
            gp.logits = c->logits_s; gp.ld_out = c->V_local;
            gp.part_m = c->part2_m; gp.part_s = c->part2_s;
            const bool rrC = pl.B > kBigMaxT;
            if ((s = launch_lmhead<true, true, false>(c, st, c->hs, pl.B, gp, rrC, &gridC)) != NJ_OK) return s;
        }
        // K-D: residual / bonus masses and the inverse-CDF draw
        MassParams mp{};
        mp.logits = c->logits_s; mp.ld = c->V_local; mp.V_local = c->V_local; mp.v_begin = c->cfg.v_begin;
        mp.nchunks = c->nchunks; mp.s_resid = c->s_resid; mp.s_qrow = c->s_qrow; mp.s_lse = c->s_lse;
        mp.part2_m = c->part2_m; mp.part2_s = c->part2_s; mp.grid2 = gridC; mp.pld2 = c->pld;
        mp.q = draft_probs; mp.ldq = ldq; mp.u = uniforms; mp.stage_mode = 0; mp.cmass = c->cmass;
        mp.accept_len = accept_len; mp.next_token = next_token;
        mp.fb_count = c->fb_count(); mp.fb_list = c->fb_list(); mp.req_flags = c->req_flags();
        mp.dbg_mass = dbg ? dbg->mass : nullptr; mp.dbg_flags = dbg ? dbg->flags : nullptr;
        mp.dbg_lse = dbg ? dbg->lse : nullptr;
        mp.certify = certify; mp.eps_draw = c->eps_draw;
        if ((s = launch_mass(c, st, mp, pl.B, true)) != NJ_OK) return s;
        k_locate<<<pl.B, kSampThreads, 0, st>>>(mp, meta);
        NJ_LAUNCHED(c, "k_locate", st);
    }
fallback:
    // the fp64 fallback runs on every call (an empty queue exits at once): with
    // certification it recomputes flagged decisions, and it always takes the
    // zero-residual-mass draws (R6), which must come from p_n
    {
        FbParams f = fb_params(c, hidden, W_lm, draft_tokens, draft_probs, ldq, uniforms, accept_len, next_token, dbg);
        if ((s = launch_fallback(c, st, f, meta)) != NJ_OK) return s;
    }
    return NJ_OK;
}

nj_status nj_verify_host(nj_ctx* c, void* stream, const uint16_t* hidden_h, const uint16_t* W_lm,
                         const int32_t* tok_h, const float* q_h, int64_t ldq, const int32_t* gamma,
                         const float* u_h, int32_t B, int32_t* acc_h, int32_t* next_h) {
    if (!c) return NJ_EINVAL;
    Plan pl;
    nj_status s = make_plan(c, gamma, B, pl);
    if (s != NJ_OK) return s;
    if (!hidden_h || !u_h || !acc_h || !next_h || (pl.G > 0 && (!tok_h || !q_h)))
        return set_err(c, NJ_EINVAL, "NULL host pointer");
    if (ldq < c->cfg.V) return set_err(c, NJ_ESHAPE, "ldq=%lld must be >= V", (long long)ldq);
    if (!c->st_hidden || c->st_ldq < ldq) {
        if (c->st_q) { cudaFree(c->st_q); c->allocs.erase(std::find(c->allocs.begin(), c->allocs.end(), (void*)c->st_q)); }
        if (!c->st_hidden) {
            if ((s = alloc(c, &c->st_hidden, (size_t)c->Nmax * c->cfg.d)) != NJ_OK) return s;
            if ((s = alloc(c, &c->st_tok, (size_t)c->Gmax)) != NJ_OK) return s;
            if ((s = alloc(c, &c->st_u, (size_t)c->Nmax)) != NJ_OK) return s;
            if ((s = alloc(c, &c->st_acc, (size_t)c->cfg.max_batch)) != NJ_OK) return s;
            if ((s = alloc(c, &c->st_next, (size_t)c->cfg.max_batch)) != NJ_OK) return s;
        }
        if ((s = alloc(c, &c->st_q, (size_t)c->Gmax * ldq)) != NJ_OK) return s;
        c->st_ldq = ldq;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    NJ_CUDA(c, cudaMemcpyAsync(c->st_hidden, hidden_h, (size_t)pl.N * c->cfg.d * 2, cudaMemcpyHostToDevice, st));
    NJ_CUDA(c, cudaMemcpyAsync(c->st_u, u_h, (size_t)pl.N * 4, cudaMemcpyHostToDevice, st));
    // The draft rows q are read zero-copy when the host buffer is pinned and
    // mapped (UVA): the path touches only q_i(x_i) and the sample row of each
    // rejected request (<= B of the G rows), so copying all G x V floats would
    // move ~G/R times the bytes the method reads.
    const float* qd = c->st_q;
    c->q_remote = 0;
    c->qstage_active = 0;
    c->qstage_rows.clear();
    for (auto& w : c->qstage_mask) w = 0;
    if (pl.G > 0) {
        NJ_CUDA(c, cudaMemcpyAsync(c->st_tok, tok_h, (size_t)pl.G * 4, cudaMemcpyHostToDevice, st));
        cudaPointerAttributes at{};
        if (c->q_zero_copy && cudaPointerGetAttributes(&at, q_h) == cudaSuccess && at.type == cudaMemoryTypeHost &&
            at.devicePointer) {
            qd = static_cast<const float*>(at.devicePointer);
            c->q_remote = 1;
            // The kernels read only q_i(x_i) and each rejected request's row n_b, known after
            // the GEMM.  When the one-launch small-batch sampler will run, the rows of the
            // likely first-rejection positions (position 0 of every request, then 1, ...:
            // P(n_b = i) falls geometrically with i) are copied to st_q over a second
            // stream while the GEMM streams W, as many as the host link moves in the GEMM's
            // time; the sampler waits for them and reads the rest in place.
            if (c->q_stage_opt != 0 && pl.path == NJ_PATH_STAGED && small_sampler_ok(c, pl) && pl.G <= 256) {
                const double rowb = (double)c->cfg.V * 4.0;
                const double t_gemm = std::max(2.0 * c->cfg.V * c->cfg.d / 6.5e12, 2.0 * pl.N * c->cfg.V * c->cfg.d / 1.35e15);
                int budget = c->q_stage_opt > 0 ? c->q_stage_opt : (int)(t_gemm * c->kn.qstage_gbs * 1e9 / rowb);
                budget = std::min(budget, pl.G);
                for (int pos = 0; (int)c->qstage_rows.size() < budget && pos < c->cfg.gamma_max; ++pos)
                    for (int b = 0; b < pl.B && (int)c->qstage_rows.size() < budget; ++b)
                        if (pos < pl.row_off[b + 1] - pl.row_off[b] - 1) c->qstage_rows.push_back(pl.row_off[b] - b + pos);
                if (!c->qstage_rows.empty()) {
                    if (!c->cstream) NJ_CUDA(c, cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
                    if (!c->ev_qstage) NJ_CUDA(c, cudaEventCreateWithFlags(&c->ev_qstage, cudaEventDisableTiming));
                    for (int g : c->qstage_rows) {
                        NJ_CUDA(c, cudaMemcpyAsync(c->st_q + (size_t)g * ldq, q_h + (size_t)g * ldq, (size_t)c->cfg.V * 4,
                                                   cudaMemcpyHostToDevice, c->cstream));
                        c->qstage_mask[g >> 6] |= 1ull << (g & 63);
                    }
                    NJ_CUDA(c, cudaEventRecord(c->ev_qstage, c->cstream));
                    c->qstage_active = 1;
                }
            }
        } else {
            (void)cudaGetLastError();
            NJ_CUDA(c, cudaMemcpyAsync(c->st_q, q_h, (size_t)pl.G * ldq * 4, cudaMemcpyHostToDevice, st));
        }
    }
    s = nj_verify(c, stream, c->st_hidden, W_lm, c->st_tok, qd, ldq, gamma, c->st_u, B, c->st_acc,
                  c->st_next, nullptr);
    c->q_remote = 0;
    c->qstage_active = 0;
    if (s != NJ_OK) return s;
    NJ_CUDA(c, cudaMemcpyAsync(acc_h, c->st_acc, (size_t)B * 4, cudaMemcpyDeviceToHost, st));
    NJ_CUDA(c, cudaMemcpyAsync(next_h, c->st_next, (size_t)B * 4, cudaMemcpyDeviceToHost, st));
    NJ_CUDA(c, cudaStreamSynchronize(st));
    return NJ_OK;
}

nj_status nj_host_staged_rows(nj_ctx* c, int32_t* rows_out, int32_t max_rows, int32_t* n_out) {
    if (!c || !n_out || (max_rows > 0 && !rows_out)) return NJ_EINVAL;
    *n_out = (int32_t)c->qstage_rows.size();
    for (int i = 0; i < std::min<int>(max_rows, (int)c->qstage_rows.size()); ++i) rows_out[i] = c->qstage_rows[i];
    return NJ_OK;
}

nj_status nj_verify_greedy(nj_ctx* c, void* stream, const uint16_t* hidden, const uint16_t* W_lm,
                           const int32_t* draft_tokens, const int32_t* gamma_per_req, int32_t B, int32_t* accept_len,
                           int32_t* next_token) {
    if (!c) return NJ_EINVAL;
    Plan pl;
    nj_status s = make_plan(c, gamma_per_req, B, pl);
    if (s != NJ_OK) return s;
    if (!hidden || !W_lm || !accept_len || !next_token || (pl.G > 0 && !draft_tokens))
        return set_err(c, NJ_EINVAL, "NULL device pointer");
    if (c->V_local != c->cfg.V || c->ncomm || !c->logits_st)
        return set_err(c, NJ_EUNSUPPORTED, "nj_verify_greedy is unsharded only");
    if ((reinterpret_cast<uintptr_t>(hidden) | reinterpret_cast<uintptr_t>(W_lm)) & 15)
        return set_err(c, NJ_ESHAPE, "hidden / W_lm must be 16-byte aligned");
    if ((s = ensure_w_maps(c, W_lm)) != NJ_OK) return s;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    // all N rows through the LM-head GEMM in blocks of the staged logits buffer
    // (one W stream per block), fp32 logits -> row argmax
    if (c->kn.lm) {
        // k_lmhead with the row argmax in its epilogue (no logits written), blocks of
        // kStagedMaxRows rows, per-group partials merged into the argmax keys
        for (int r0 = 0; r0 < pl.N; r0 += kStagedMaxRows) {
            const int R = std::min(kStagedMaxRows, pl.N - r0);
            LmheadParams lp{};
            lp.part_m = c->part_m;
            lp.part_s = c->part_s;
            lp.inv_t = 1.f;
            int np = 0;
            std::pair<cudaEvent_t, cudaEvent_t> ev;
            if ((s = prof_begin(c, st, ev)) != NJ_OK) return s;
            if ((s = launch_lm<LM_ARGMAX>(c, st, hidden + (size_t)r0 * c->cfg.d, W_lm, R, lp, &np)) != NJ_OK) return s;
            if ((s = prof_end(c, st, ev)) != NJ_OK) return s;
            k_argmax_merge<<<(R + 7) / 8, 256, 0, st>>>(c->part_m, c->part_s, c->pld, np, R, c->amax + r0);
            NJ_LAUNCHED(c, "k_argmax_merge", st);
        }
        const ReqMeta meta = make_meta(pl);
        k_greedy_decide<<<(B + 127) / 128, 128, 0, st>>>(meta, draft_tokens, c->amax, accept_len, next_token);
        NJ_LAUNCHED(c, "k_greedy_decide", st);
        return NJ_OK;
    }
    const int cap = std::min(c->Nmax, kStagedMaxN);   // k_gemm_big blocks
    NJ_CUDA(c, cudaMemsetAsync(c->amax, 0, (size_t)pl.N * sizeof(unsigned long long), st));
    for (int r0 = 0; r0 < pl.N; r0 += cap) {
        const int R = std::min(cap, pl.N - r0);
        GemmBigParams gp{};
        gp.logits = c->logits_st; gp.ld_out = c->V_local;
        gp.part_m = c->part_m; gp.part_s = c->part_s;   // statistics unused
        int grid = c->grid;
        std::pair<cudaEvent_t, cudaEvent_t> ev;
        if ((s = prof_begin(c, st, ev)) != NJ_OK) return s;
        if ((s = launch_lmhead<true, true, false>(c, st, hidden + (size_t)r0 * c->cfg.d, R, gp, false, &grid)) != NJ_OK)
            return s;
        if ((s = prof_end(c, st, ev)) != NJ_OK) return s;
        const int nsplit = std::max(1, std::min((c->V_local + 2047) / 2048, (c->num_sms * 4 + R - 1) / R));
        k_argmax_rows<<<dim3(nsplit, R), 256, 0, st>>>(c->logits_st, c->V_local, c->V_local, c->amax + r0);
        NJ_LAUNCHED(c, "k_argmax_rows", st);
    }
    const ReqMeta meta = make_meta(pl);
    k_greedy_decide<<<(B + 127) / 128, 128, 0, st>>>(meta, draft_tokens, c->amax, accept_len, next_token);
    NJ_LAUNCHED(c, "k_greedy_decide", st);
    return NJ_OK;
}

nj_status nj_propose(nj_ctx* c, void* stream, const uint16_t* hidden, const uint16_t* W_lm, const float* u,
                     int32_t B, int32_t* tokens, float* q_out, int64_t ldq) {
    if (!c) return NJ_EINVAL;
    if (!hidden || !W_lm || !u || !tokens || !q_out) return set_err(c, NJ_EINVAL, "NULL device pointer");
    if (B < 1 || B > c->cfg.max_batch) return set_err(c, NJ_ESHAPE, "B=%d outside [1, max_batch=%d]", B, c->cfg.max_batch);
    if (ldq < c->V_local) return set_err(c, NJ_ESHAPE, "ldq=%lld < V", (long long)ldq);
    if (c->V_local != c->cfg.V || c->ncomm) return set_err(c, NJ_EUNSUPPORTED, "nj_propose is unsharded only");
    if ((reinterpret_cast<uintptr_t>(hidden) | reinterpret_cast<uintptr_t>(W_lm)) & 15)
        return set_err(c, NJ_ESHAPE, "hidden / W_lm must be 16-byte aligned");
    nj_status s;
    if ((s = ensure_w_maps(c, W_lm)) != NJ_OK) return s;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    // draft LM head: fp32 logits straight into q_out + per-CTA (max, sum) partials
    int grid = c->grid;
    {
        std::pair<cudaEvent_t, cudaEvent_t> ev;
        if ((s = prof_begin(c, st, ev)) != NJ_OK) return s;
        if (c->kn.lm) {
            LmheadParams lp{};
            lp.logits = q_out; lp.ld_out = ldq;
            lp.part_m = c->part2_m; lp.part_s = c->part2_s;
            if ((s = launch_lm<LM_WRITE | LM_STATS>(c, st, hidden, W_lm, B, lp, &grid)) != NJ_OK) return s;
        } else {
            GemmBigParams gp{};
            gp.logits = q_out; gp.ld_out = ldq;
            gp.part_m = c->part2_m; gp.part_s = c->part2_s;
            const bool rr = B > kBigMaxT;
            if ((s = launch_lmhead<true, true, false>(c, st, hidden, B, gp, rr, &grid)) != NJ_OK) return s;
        }
        if ((s = prof_end(c, st, ev)) != NJ_OK) return s;
    }
    k_lse_rows<<<(B + 7) / 8, 256, 0, st>>>(c->part2_m, c->part2_s, c->pld, grid, B, c->row_lse);
    NJ_LAUNCHED(c, "k_lse_rows", st);
    NJ_CUDA(c, cudaMemsetAsync(c->s_resid, 0, (size_t)B * sizeof(int32_t), st));   // every row: w = q
    MassParams mp{};
    mp.logits = q_out; mp.ld = ldq; mp.V_local = c->V_local; mp.v_begin = 0; mp.nchunks = c->nchunks;
    mp.s_resid = c->s_resid; mp.s_qrow = c->scratch_i; mp.s_lse = c->row_lse;
    mp.q = q_out; mp.ldq = ldq; mp.u = u; mp.stage_mode = 1; mp.cmass = c->cmass;
    mp.next_token = tokens;
    mp.fb_count = c->fb_count(); mp.fb_list = c->fb_list(); mp.req_flags = c->req_flags();
    mp.certify = 0; mp.eps_draw = 0.f;
    mp.w_inplace = 1;   // k_mass leaves q = exp(l - lse) in q_out; k_locate reads it
    if ((s = launch_mass(c, st, mp, B, false)) != NJ_OK) return s;
    ReqMeta meta;
    meta.B = B;
    k_locate<<<B, kSampThreads, 0, st>>>(mp, meta);
    NJ_LAUNCHED(c, "k_locate", st);
    return NJ_OK;
}

nj_status nj_lmhead_logits(nj_ctx* c, void* stream, const uint16_t* hidden, const uint16_t* W_lm,
                           const int32_t* rows, int32_t n_rows, float* logits, int64_t ld_out, int32_t ks) {
    if (!c) return NJ_EINVAL;
    if (!hidden || !W_lm || !rows || !logits) return set_err(c, NJ_EINVAL, "NULL device pointer");
    if (n_rows < 1 || n_rows > std::min(c->Gmax, kMaxStatRows))
        return set_err(c, NJ_ESHAPE, "n_rows=%d outside [1, %d]", n_rows, std::min(c->Gmax, kMaxStatRows));
    if (ld_out < c->V_local) return set_err(c, NJ_ESHAPE, "ld_out=%lld < V_local", (long long)ld_out);
    if (ks < 0) return set_err(c, NJ_EINVAL, "ks=%d", ks);
    nj_status s;
    if ((s = ensure_w_maps(c, W_lm)) != NJ_OK) return s;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    k_gather_rows<<<n_rows, 128, 0, st>>>(hidden, c->cfg.d, rows, c->hd);
    NJ_LAUNCHED(c, "k_gather_rows", st);
    // the production LM-head GEMM (k_lmhead as the staged path launches it; k_gemm_big
    // with NJ_LM=0, as the two-pass path and nj_propose launch it) writing fp32
    // logits; statistics go to scratch partials
    if (c->kn.lm) {
        LmheadParams lp{};
        lp.logits = logits;
        lp.ld_out = ld_out;
        lp.part_m = c->part_m;
        lp.part_s = c->part_s;
        lp.ks = ks;
        lp.inv_t = 1.f;
        int np = 0;
        return launch_lm<LM_WRITE | LM_STATS>(c, st, c->hd, W_lm, n_rows, lp, &np);
    }
    GemmBigParams gp{};
    gp.logits = logits;
    gp.ld_out = ld_out;
    gp.part_m = c->part_m;
    gp.part_s = c->part_s;
    gp.ks = ks;
    gp.inv_t = 1.f;   // raw logits (no temperature)
    int grid = c->grid;
    return launch_lmhead<true, true, false>(c, st, c->hd, n_rows, gp, n_rows > kBigMaxT, &grid);
}

nj_status nj_sample_from_logits(nj_ctx* c, void* stream, const float* logits, int64_t ld_l, const int32_t* residual,
                                const float* q, int64_t ldq, const float* u, int32_t B, int32_t* next_token,
                                double* mass) {
    if (!c) return NJ_EINVAL;
    if (!logits || !residual || !q || !u || !next_token) return set_err(c, NJ_EINVAL, "NULL device pointer");
    if (B < 1 || B > c->cfg.max_batch) return set_err(c, NJ_ESHAPE, "B=%d", B);
    if (c->V_local != c->cfg.V) return set_err(c, NJ_EUNSUPPORTED, "stage export is unsharded only");
    if (ld_l < c->V_local || ldq < c->V_local) return set_err(c, NJ_ESHAPE, "pitch < V");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    NJ_CUDA(c, cudaMemsetAsync(c->fb_block, 0, (1 + 2 * (size_t)c->cfg.max_batch) * sizeof(int32_t), st));
    k_row_lse<<<B, 256, 0, st>>>(logits, ld_l, c->V_local, c->lse_tmp);
    NJ_LAUNCHED(c, "k_row_lse", st);
    k_iota<<<(B + 255) / 256, 256, 0, st>>>(c->scratch_i, B);
    NJ_LAUNCHED(c, "k_iota", st);
    MassParams mp{};
    mp.logits = logits; mp.ld = ld_l; mp.V_local = c->V_local; mp.v_begin = 0; mp.nchunks = c->nchunks;
    mp.s_resid = residual; mp.s_qrow = c->scratch_i; mp.s_lse = c->lse_tmp;
    mp.q = q; mp.ldq = ldq; mp.u = u; mp.stage_mode = 1; mp.cmass = c->cmass;
    mp.next_token = next_token;
    mp.fb_count = c->fb_count(); mp.fb_list = c->fb_list(); mp.req_flags = c->req_flags();
    mp.dbg_mass = mass;
    mp.certify = c->certify; mp.eps_draw = 4e-6f;
    ReqMeta meta;
    meta.B = B;
    if (nj_status s2 = launch_mass(c, st, mp, B, false)) return s2;
    k_locate<<<B, kSampThreads, 0, st>>>(mp, meta);
    NJ_LAUNCHED(c, "k_locate", st);
    {   // certified draws (certify on) and zero-mass draws (R6, always)
        FbParams f{};
        f.V_local = c->V_local;
        f.fb_count = c->fb_count(); f.fb_list = c->fb_list(); f.req_flags = c->req_flags();
        f.q = q; f.ldq = ldq; f.u = u; f.next_token = next_token; f.dbg_mass = mass;
        f.st_logits = logits; f.st_ld = ld_l; f.st_resid = residual; f.stage_mode = 1;
        k_fb_decide<<<std::min(B, c->num_sms), 256, 0, st>>>(f, meta);
        NJ_LAUNCHED(c, "k_fb_decide", st);
    }
    return NJ_OK;
}


/* ------------------------------------------------------- vocab-sharded mode */

nj_status nj_shard_range(int32_t V, int32_t nranks, int32_t rank, int32_t* v_begin, int32_t* v_end) {
    if (V < 1 || nranks < 1 || rank < 0 || rank >= nranks || !v_begin || !v_end) return NJ_EINVAL;
    if ((V + kTileV - 1) / kTileV < nranks) return NJ_ESHAPE;
    int vb, ve;
    shard_range(V, nranks, rank, vb, ve);
    *v_begin = vb;
    *v_end = ve;
    return NJ_OK;
}

nj_status nj_nccl_get_unique_id(void* id_out) {
    if (!id_out) return NJ_EINVAL;
    NcclApi* api = nccl_api();
    if (!api) return NJ_ENCCL;
    NcclId id;
    if (api->GetUniqueId(&id) != 0) return NJ_ENCCL;
    memcpy(id_out, &id, sizeof id);
    return NJ_OK;
}

nj_status nj_nccl_comm_init(int32_t nranks, const void* id, int32_t rank, int32_t device, void** comm_out) {
    if (!id || !comm_out || nranks < 1 || rank < 0 || rank >= nranks) return NJ_EINVAL;
    NcclApi* api = nccl_api();
    if (!api) return NJ_ENCCL;
    if (cudaSetDevice(device) != cudaSuccess) return NJ_ECUDA;
    NcclId nid;
    memcpy(&nid, id, sizeof nid);
    void* comm = nullptr;
    if (api->CommInitRank(&comm, nranks, nid, rank) != 0) return NJ_ENCCL;
    *comm_out = comm;
    return NJ_OK;
}

void nj_nccl_comm_destroy(void* comm) {
    NcclApi* api = nccl_api();
    if (api && comm) api->CommDestroy(comm);
}

nj_status nj_group_create(const nj_config* cfg, int32_t nshards, nj_group** out) {
    if (!cfg || !out || nshards < 1) return set_err(nullptr, NJ_EINVAL, "NULL argument / nshards < 1");
    *out = nullptr;
    if ((cfg->V + kTileV - 1) / kTileV < nshards) return set_err(nullptr, NJ_ESHAPE, "V=%d too small for %d shards", cfg->V, nshards);
    nj_group* g = new nj_group();
    for (int r = 0; r < nshards; ++r) {
        nj_config cr = *cfg;
        cr.nccl_comm = nullptr;
        int vb, ve;
        shard_range(cfg->V, nshards, r, vb, ve);
        cr.v_begin = vb;
        cr.v_end = ve;
        nj_ctx* c = nullptr;
        nj_status s = nj_create(&cr, &c);
        if (s == NJ_OK) {
            c->in_group = true;
            c->nranks = nshards;
            c->rank = r;
            s = alloc_shard_ws(c);
            if (s != NJ_OK) g_create_error = c->err;
        }
        if (s != NJ_OK) {
            if (c) nj_destroy(c);
            nj_group_destroy(g);
            return s;
        }
        g->mem.push_back(c);
    }
    if (cudaMalloc(&g->scratch, (size_t)nshards * 2 * cfg->max_batch * sizeof(int32_t)) != cudaSuccess) {
        nj_group_destroy(g);
        return set_err(nullptr, NJ_ENOMEM, "cudaMalloc failed (group scratch)");
    }
    *out = g;
    return NJ_OK;
}

void nj_group_destroy(nj_group* g) {
    if (!g) return;
    for (nj_ctx* c : g->mem) nj_destroy(c);
    if (g->scratch) cudaFree(g->scratch);
    delete g;
}

nj_ctx* nj_group_member(nj_group* g, int32_t r) {
    return (g && r >= 0 && r < (int)g->mem.size()) ? g->mem[r] : nullptr;
}

nj_status nj_group_verify(nj_group* g, void* stream, const uint16_t* hidden, const uint16_t* const* W_shards,
                          const int32_t* draft_tokens, const float* draft_probs, int64_t ldq,
                          const int32_t* gamma_per_req, const float* uniforms, int32_t B, int32_t* accept_len,
                          int32_t* next_token, const nj_debug* dbg) {
    if (!g || !W_shards) return NJ_EINVAL;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int n = (int)g->mem.size();
    std::vector<ShardCall> calls(n);
    for (int r = 0; r < n; ++r) {
        nj_status s = shard_call(g->mem[r], calls[r], hidden, W_shards[r], draft_tokens, draft_probs, ldq,
                                 gamma_per_req, uniforms, B, accept_len, next_token, r == 0 ? dbg : nullptr);
        if (s != NJ_OK) return s;
    }
    for (int ph = 0; ph < shard_nphases(calls[0]); ++ph) {
        for (int r = 0; r < n; ++r) {
            nj_status s = shard_phase(g->mem[r], st, calls[r], ph);
            if (s != NJ_OK) return s;
        }
        XSpec x0;
        if (!shard_xchg(g->mem[0], calls[0], ph, x0)) continue;
        nj_ctx* c0 = g->mem[0];
        if (x0.max_i32) {
            const int len = (int)(x0.bytes / 4);
            for (int r = 0; r < n; ++r) {
                XSpec xr;
                shard_xchg(g->mem[r], calls[r], ph, xr);
                NJ_CUDA(c0, cudaMemcpyAsync(g->scratch + (size_t)r * len, xr.send, x0.bytes, cudaMemcpyDeviceToDevice, st));
            }
            for (int i = 0; i < n; ++i) {
                XSpec xi;
                shard_xchg(g->mem[i], calls[i], ph, xi);
                k_imax<<<(len + 255) / 256, 256, 0, st>>>(g->scratch, n, len, static_cast<int32_t*>(xi.recv));
                NJ_CUDA(c0, cudaGetLastError());
            }
        } else {
            for (int i = 0; i < n; ++i) {
                XSpec xi;
                shard_xchg(g->mem[i], calls[i], ph, xi);
                for (int r = 0; r < n; ++r) {
                    XSpec xr;
                    shard_xchg(g->mem[r], calls[r], ph, xr);
                    NJ_CUDA(c0, cudaMemcpyAsync(static_cast<char*>(xi.recv) + (size_t)r * x0.bytes, xr.send, x0.bytes,
                                                cudaMemcpyDeviceToDevice, st));
                }
            }
        }
    }
    return NJ_OK;
}

const char* nj_group_last_error(const nj_group* g) {
    if (!g) return g_create_error.c_str();
    for (nj_ctx* c : g->mem)
        if (!c->err.empty()) return c->err.c_str();
    return "";
}


}  // extern "C"
