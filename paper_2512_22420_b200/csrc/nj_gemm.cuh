// nj_gemm.cuh — LM-head GEMM kernels for sm_100a (tcgen05 + TMEM + TMA).
//
// BJ step (1): l_j(x) = sum_k W[x,k] h_j[k] ("the target model then
// verifies in parallel"), with BJ step (2) online-softmax statistics fused in
// the epilogue so the logits of verified rows never go to HBM.
//
// Layout ("swap-AB"): the MMA M dimension is 128 VOCAB rows of W (operand A,
// K-major, SWIZZLE_128B, TMA box 64x128 or 64x16), the N dimension is the
// token rows of H (operand B, 16..256 rows).  Accumulator D[vocab, token] lives
// in TMEM: lane = vocab row, column = token.  Small token counts therefore cost
// no MMA padding (N is any multiple of 16), and the vocabulary runs across
// TMEM lanes / threads, which makes the sampler's reads of q coalesced.
//
// Vocabulary split: V_local is cut into 16-row units balanced over the grid
// (one CTA per SM): at V = 152064 on 148 SMs every CTA owns 1024 or 1040 rows =
// 8 full 128-row tiles + at most one 16-row tile (98.8% balance).
//
// Warp roles (256 threads): warp 0 TMA producer, warp 1 MMA issuer, warp 2
// TMEM allocator, warps 4-7 epilogue (warp w reads TMEM lanes 32*(w%4)..+31).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "nj_ptx.cuh"

namespace nj {

constexpr int kThreads = 256;
constexpr int kTileV = 128;                     // vocab rows per tile (UMMA M)
constexpr int kBK = 64;                         // K per stage (one 128-B swizzle row)
constexpr int kTileBytesA = kTileV * kBK * 2;   // 16 KB
constexpr int kUnit = 16;                       // vocab split granularity
constexpr int kMaxB = 1024;                     // requests passed by value
constexpr int kMaxStatRows = 1536;              // rows per k_gemm_rows launch (STATS)
constexpr int kFusedMaxN = 48;                  // fused path: N <= 48 tokens
constexpr int kSmemLimit = 227 * 1024;

__device__ __forceinline__ void vocab_range(int U, int grid, int c, int V_local, int& r0, int& rows) {
    const int base = U / grid, rem = U % grid;
    const int u0 = c * base + (c < rem ? c : rem);
    const int nu = base + (c < rem ? 1 : 0);
    r0 = u0 * kUnit;
    rows = V_local - r0;
    if (rows > nu * kUnit) rows = nu * kUnit;
    if (rows < 0) rows = 0;
}

// A operand (W tile rows [row0, row0+trows)) for k-block kb.  Full tiles use
// one 64x128 box, partial tiles 64x16 boxes (1024-B aligned 2-KB steps keep
// the SW128 pattern identical to the big box).  Returns bytes in flight.
__device__ __forceinline__ uint32_t load_w_tile(uint8_t* dst, const CUtensorMap* w128, const CUtensorMap* w16,
                                                uint64_t* bar, int kb, int row0, int trows, uint64_t pol) {
    if (trows == kTileV) {
        tma_load_2d(dst, w128, bar, kb * kBK, row0, pol);
        return kTileBytesA;
    }
    const int nl = (trows + 15) >> 4;
    for (int l = 0; l < nl; ++l) tma_load_2d(dst + l * 2048, w16, bar, kb * kBK, row0 + 16 * l, pol);
    return (uint32_t)nl * 2048u;
}
__device__ __forceinline__ uint32_t w_tile_bytes(int trows) {
    return trows == kTileV ? (uint32_t)kTileBytesA : (uint32_t)((trows + 15) >> 4) * 2048u;
}

__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------------------
// k_gemm_rows: persistent GEMM over a contiguous row buffer H[R, d].
//   WRITE   : logits[row, x] fp32 (pitch ld_out), x local vocab id
//   STATS   : per (row, CTA) online-softmax partial (m, s) -> part_m/part_s
//   CAPTURE : dl[row] = l_row(tok[row]) for the CTA owning that token
// Token rows are processed in chunks of box_rows (<= 256) with a double
// buffered TMEM accumulator (2 x 256 columns) so the epilogue of one
// (tile, chunk) item overlaps the MMAs of the next.
// ---------------------------------------------------------------------------
struct GemmRowsParams {
    int32_t R, box_rows, nchunks;
    int32_t V_local, U, num_kb, nstages, v_begin;
    float* logits;
    int64_t ld_out;
    float* part_m;
    float* part_s;
    int32_t part_ld;        // = grid
    const int32_t* tok;     // [R] global token ids (CAPTURE)
    double* dl;             // [R]
};

template <bool WRITE, bool STATS, bool CAPTURE>
__global__ void __launch_bounds__(kThreads, 1)
k_gemm_rows(const __grid_constant__ CUtensorMap tmW128, const __grid_constant__ CUtensorMap tmW16,
            const __grid_constant__ CUtensorMap tmH, const GemmRowsParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int S = p.nstages;
    const int bBytes = p.box_rows * 128;
    uint8_t* sA = smem;                                   // S x 16 KB
    uint8_t* sB = smem + (size_t)S * kTileBytesA;         // S x bBytes (1024-multiple)
    uint8_t* tail = sB + (size_t)S * bBytes;
    float2* scratch = reinterpret_cast<float2*>(tail);    // [4][256]
    float2* state = scratch + 4 * 256;                    // [R] (STATS)
    int32_t* stok = reinterpret_cast<int32_t*>(state + (STATS ? p.R : 0));   // [R] (CAPTURE)
    uint64_t* bars = reinterpret_cast<uint64_t*>(
        (reinterpret_cast<uintptr_t>(stok + (CAPTURE ? p.R : 0)) + 7) & ~uintptr_t(7));
    uint64_t* full = bars;
    uint64_t* empty = bars + S;
    uint64_t* tfull = bars + 2 * S;    // [2]
    uint64_t* tempty = bars + 2 * S + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 4);

    const int warp = (int)warp_id(), lane = (int)lane_id();
    const int grid = gridDim.x, cta = blockIdx.x;
    int r0, rows;
    vocab_range(p.U, grid, cta, p.V_local, r0, rows);
    const int ntiles = (rows + kTileV - 1) / kTileV;
    const int nitems = ntiles * p.nchunks;

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmW128);
        tma_prefetch_desc(&tmW16);
        tma_prefetch_desc(&tmH);
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4); }
        fence_barrier_init();
        fence_proxy_async();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    if (STATS)
        for (int i = threadIdx.x; i < p.R; i += kThreads) state[i] = make_float2(-INFINITY, 0.f);
    if (CAPTURE)
        for (int i = threadIdx.x; i < p.R; i += kThreads) stok[i] = p.tok[i] - p.v_begin;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // ------------------------------------------------ TMA producer
        const uint64_t pol_w = policy_evict_first();   // W streamed once
        const uint64_t pol_h = policy_evict_last();    // H re-read per tile
        int s = 0;
        uint32_t ph = 0;
        for (int it = 0; it < nitems; ++it) {
            const int t = it / p.nchunks, c = it % p.nchunks;
            const int trows = min(kTileV, rows - t * kTileV);
            const uint32_t bytes = w_tile_bytes(trows) + (uint32_t)bBytes;
            for (int kb = 0; kb < p.num_kb; ++kb) {
                mbar_wait(&empty[s], ph ^ 1);
                mbar_arrive_expect_tx(&full[s], bytes);
                load_w_tile(sA + (size_t)s * kTileBytesA, &tmW128, &tmW16, &full[s], kb, r0 + t * kTileV, trows,
                            pol_w);
                tma_load_2d(sB + (size_t)s * bBytes, &tmH, &full[s], kb * kBK, c * p.box_rows, pol_h);
                if (++s == S) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1 && lane == 0) {
        // ------------------------------------------------ MMA issuer
        int s = 0;
        uint32_t ph = 0;
        for (int it = 0; it < nitems; ++it) {
            const int c = it % p.nchunks;
            const int ncol = min(p.box_rows, p.R - c * p.box_rows);
            const uint32_t npad = (uint32_t)((ncol + 15) & ~15);
            const uint32_t idesc = idesc_bf16_f32(128, npad);
            const int buf = it & 1;
            mbar_wait(&tempty[buf], ((it >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t dt = tbase + (uint32_t)(buf * 256);
            for (int kb = 0; kb < p.num_kb; ++kb) {
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint64_t ad = sdesc_sw128(sA + (size_t)s * kTileBytesA);
                const uint64_t bd = sdesc_sw128(sB + (size_t)s * bBytes);
#pragma unroll
                for (int k = 0; k < kBK / 16; ++k)
                    mma_bf16(dt, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
                mma_commit(&empty[s]);
                if (++s == S) { s = 0; ph ^= 1; }
            }
            mma_commit(&tfull[buf]);
        }
    } else if (warp >= 4) {
        // ------------------------------------------------ epilogue
        const int q = warp & 3;
        const int et = threadIdx.x - 128;   // 0..127
        const uint32_t lane_base = tbase + ((uint32_t)(q * 32) << 16);
        for (int it = 0; it < nitems; ++it) {
            const int t = it / p.nchunks, c = it % p.nchunks;
            const int trows = min(kTileV, rows - t * kTileV);
            const int vr = q * 32 + lane;
            const bool valid = vr < trows;
            const int xl = r0 + t * kTileV + vr;
            const int c0 = c * p.box_rows;
            const int ncol = min(p.box_rows, p.R - c0);
            const int buf = it & 1;
            mbar_wait(&tfull[buf], (it >> 1) & 1);
            tc_fence_after();
            for (int g = 0; g * 16 < ncol; ++g) {
                float v[16];
                tmem_ld16(lane_base + (uint32_t)(buf * 256 + g * 16), v);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int col = g * 16 + i;
                    if (col < ncol) {
                        const int row = c0 + col;
                        if (WRITE && valid) p.logits[(int64_t)row * p.ld_out + xl] = v[i];
                        if (CAPTURE && valid && stok[row] == xl) p.dl[row] = (double)v[i];
                        if (STATS) {
                            const float vv = valid ? v[i] : -INFINITY;
                            const float m = warp_max(vv);
                            const float e = valid ? __expf(vv - m) : 0.f;
                            const float sm = warp_sum(e);
                            if (lane == 0) scratch[q * 256 + col] = make_float2(m, sm);
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
            if (STATS) {
                named_bar(1, 128);
                for (int col = et; col < ncol; col += 128) {
                    float2 st = state[c0 + col];
#pragma unroll
                    for (int w = 0; w < 4; ++w) {
                        const float2 o = scratch[w * 256 + col];
                        ms_merge(st.x, st.y, o.x, o.y);
                    }
                    state[c0 + col] = st;
                }
                named_bar(1, 128);
            }
        }
    }
    __syncthreads();
    if (STATS)
        for (int i = threadIdx.x; i < p.R; i += kThreads) {
            p.part_m[(int64_t)i * p.part_ld + cta] = state[i].x;
            p.part_s[(int64_t)i * p.part_ld + cta] = state[i].y;
        }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_dealloc(tbase, 512);
}

// ---------------------------------------------------------------------------
// k_fused_verify<NPAD>: the whole verification step in ONE persistent
// cooperative kernel for N <= 48 rows (memory-bound regime, BJ config 2).
//   phase 1  GEMM over every row; all of this CTA's logits stay resident in
//            TMEM (ntiles * NPAD <= 512 columns); per-thread online softmax
//            (1 exp / element) + draft-token logit capture.
//   barrier  ---- grid-wide
//   phase 2  lse of every row (fixed-order fp64 merge of the per-CTA
//            partials), acceptance tests, first rejection (every CTA
//            redundantly, bit-identical).
//   phase 3  residual / bonus weights of each request's sample row straight
//            from TMEM; per-tile masses via warp scans; per-CTA mass.
//   barrier  ---- grid-wide
//   phase 4  fp64 prefix of CTA masses (fixed order) locates the owning CTA,
//            which locates the tile, then the token, by inclusive scans that
//            reproduce phase 3's arithmetic bit for bit.
// W is streamed from HBM exactly once; nothing of size V*N is written.
// ---------------------------------------------------------------------------
struct FusedParams {
    int32_t B, N, G;
    int32_t V_local, v_begin, U, num_kb, nstages;
    int32_t nbuf, scratch_col;   // scratch accumulators: nbuf x NPAD columns at scratch_col
    int32_t kpd;                 // k-blocks per drained partial (accuracy: 1)
    int32_t sacc;                // grouped mode: 1 = one partial per ring stage (restart every GK k-blocks)
    int32_t kgroup;              // k-blocks per TMA ring stage
    int32_t ngroups;             // >0: drain handshake per ring stage with ngroups x kgroup scratch buffers
    unsigned long long* phase_ts; // debug: [grid][8] %globaltimer stamps at phase boundaries (NULL: off)
    int32_t rows_cap;            // max vocab rows per CTA (q-slice pitch in smem)
    int32_t q_bytes_cap;         // bytes reserved for q slices at the start of the ring
    int32_t q_prefetch;          // 1: every draft row's q slice is cp.async'ed before barrier 1
    int32_t q_vec16;             // q rows 16-byte aligned at CTA starts (16-B cp.async)
    const int32_t* draft_tokens;
    const float* q;
    int64_t ldq;
    const float* u;
    int32_t* accept_len;
    int32_t* next_token;
    float* part_m;      // [N][grid]
    float* part_s;
    double* dl;         // [G] fp64 draft logits
    double* wpart;      // [B][grid]
    uint32_t* bar;      // grid-barrier word
    int32_t* fb_count;  // certified-fallback work list
    int32_t* fb_list;
    int32_t* req_flags; // [B]
    float* dbg_lse;
    float* dbg_pdraft;
    double* dbg_mass;
    int32_t* dbg_flags;
    int32_t certify, force_fallback;
    float eps_acc;      // relative acceptance margin (certificate)
    float eps_draw;     // absolute CDF margin (certificate), probability units
    int32_t row_off[kMaxB + 1];
};

// request bookkeeping shared by phases 2-4 (smem)
struct ReqInfo {
    int32_t n, gam, srow, qrow, resid, flag;
    double lse_s;
};

__device__ __forceinline__ void push_fallback(int32_t* fb_count, int32_t* fb_list, int32_t* req_flags, int b,
                                              int32_t bits) {
    const int32_t old = atomicOr(&req_flags[b], bits | 0x100);
    if (!(old & 0x100)) fb_list[atomicAdd(fb_count, 1)] = b;
}

#include "nj_fused.cuh"
#include "nj_gemm_acc.cuh"
#include "nj_gemm_big.cuh"

}  // namespace nj
