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
constexpr int kMaxStatRows = 1536;              // rows per statistics GEMM launch (K-A)
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
    double inv_t;                // 1 / temperature: target logits l / T (include/nj.h nj_set_temperature)
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
#include "nj_gemm_big.cuh"
#include "nj_lmhead.cuh"

}  // namespace nj
