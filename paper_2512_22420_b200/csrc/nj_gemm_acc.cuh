// nj_gemm_acc.cuh — k_gemm_acc<WRITE,STATS,CAPTURE>: the LM-head GEMM of the
// two-pass path (N > 48) with the fused path's accuracy scheme at a larger
// token tile.  Included from nj_gemm.cuh (namespace nj).
//
// * token rows of H[R, d] in chunks of 128 (MMA N <= 128), vocab tiles of 128
//   rows (MMA M), the persistent tile-balanced vocab split of the fused kernel;
//   items = (tile, chunk), tile-major so one vocab tile's W is re-read from L2
//   (not HBM) across its chunks;
// * every k-block's 4 MMAs write a FRESH TMEM accumulator (tcgen05 truncates on
//   every fp32 accumulate: restarting per k-block cuts the bias 68x, DESIGN.md
//   "accuracy"); 2 k-blocks per TMA ring stage, 2 double-buffered groups of 2
//   partials = all 512 TMEM columns;
// * 8 epilogue warps (2 per TMEM lane quadrant, 64 columns each) add the
//   partials into fp32 round-to-nearest running sums in registers (unbiased),
//   then per item: WRITE fp32 logits (coalesced: lanes = consecutive vocab),
//   STATS online-softmax partials merged across tiles in smem via a warp
//   reduce-scatter, CAPTURE the draft-token logit.
#pragma once

constexpr int kAccThreads = 384;
constexpr int kAccT = 128;        // token chunk (MMA N)
constexpr int kAccGK = 2;         // k-blocks per ring stage
constexpr int kAccNC = 64;        // columns per epilogue warp
constexpr int kAccMaxRowG = 256;  // staged path: rows mapped to draft indices (by value)

struct GemmAccParams {
    int32_t R, nchunks;
    int32_t V_local, U, num_kb, nstages, v_begin;
    float* logits;
    int64_t ld_out;
    float* part_m;          // [R][part_ld]
    float* part_s;
    int32_t part_ld;
    const int32_t* tok;     // [R] global token ids (CAPTURE), or with row_g: draft_tokens
    double* dl;             // [R] (or [G] with row_g)
    int32_t w_evict_first;  // single chunk: W is streamed once, keep L2 for the staged logits
    int32_t use_row_g;      // staged path: row r is draft row_g[r] (-1: bonus row)
    int32_t row_g[kAccMaxRowG];
};

template <bool WRITE, bool STATS, bool CAPTURE>
__global__ void __launch_bounds__(kAccThreads, 1)
k_gemm_acc(const __grid_constant__ CUtensorMap tmW128, const __grid_constant__ CUtensorMap tmW16,
           const __grid_constant__ CUtensorMap tmH, const GemmAccParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr int kBBytes = kAccT * 128;                     // 16 KB of H per k-block
    const int S = p.nstages;
    uint8_t* sA = smem;                                      // S x GK x 16 KB
    uint8_t* sB = smem + (size_t)S * kAccGK * kTileBytesA;   // S x GK x 16 KB
    float2* scratch = reinterpret_cast<float2*>(sB + (size_t)S * kAccGK * kBBytes);  // [2 halves][4 q][64]
    float2* state = scratch + 2 * 4 * kAccNC;                                        // [R] (STATS)
    int32_t* stok = reinterpret_cast<int32_t*>(state + (STATS ? p.R : 0));         // [R] (CAPTURE)
    uint64_t* bars = reinterpret_cast<uint64_t*>(
        (reinterpret_cast<uintptr_t>(stok + (CAPTURE ? p.R : 0)) + 7) & ~uintptr_t(7));
    uint64_t* full = bars;
    uint64_t* empty = bars + S;
    uint64_t* pfull = bars + 2 * S;   // [2] groups
    uint64_t* pempty = pfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pempty + 2);

    const int warp = (int)warp_id(), lane = (int)lane_id();
    const int grid = gridDim.x, cta = blockIdx.x;
    int r0, rows;
    vocab_range(p.U, grid, cta, p.V_local, r0, rows);
    const int ntiles = (rows + kTileV - 1) / kTileV;
    const int nitems = ntiles * p.nchunks;
    const int nkg = (p.num_kb + kAccGK - 1) / kAccGK;

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmW128);
        tma_prefetch_desc(&tmW16);
        tma_prefetch_desc(&tmH);
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int g = 0; g < 2; ++g) { mbar_init(&pfull[g], 1); mbar_init(&pempty[g], 8); }
        fence_barrier_init();
        fence_proxy_async();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    if (STATS)
        for (int i = threadIdx.x; i < p.R; i += kAccThreads) state[i] = make_float2(-INFINITY, 0.f);
    if (CAPTURE)
        for (int i = threadIdx.x; i < p.R; i += kAccThreads) {
            if (p.use_row_g) stok[i] = p.row_g[i] >= 0 ? p.tok[p.row_g[i]] - p.v_begin : -1;
            else stok[i] = p.tok[i] - p.v_begin;
        }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // ------------------------------------------------ TMA producer
        // a W tile is re-read for every chunk (evict_last), unless there is one chunk
        const uint64_t pol_w = p.w_evict_first ? policy_evict_first() : policy_evict_last();
        const uint64_t pol_h = policy_evict_last();
        int s = 0;
        uint32_t ph = 0;
        for (int it = 0; it < nitems; ++it) {
            const int t = it / p.nchunks, c = it - t * p.nchunks;
            const int trows = min(kTileV, rows - t * kTileV);
            for (int kg = 0; kg < nkg; ++kg) {
                const int ng = min(kAccGK, p.num_kb - kg * kAccGK);
                mbar_wait(&empty[s], ph ^ 1);
                mbar_arrive_expect_tx(&full[s], (uint32_t)ng * (w_tile_bytes(trows) + (uint32_t)kBBytes));
                for (int g = 0; g < ng; ++g) {
                    const int kb = kg * kAccGK + g;
                    const size_t slot = (size_t)s * kAccGK + g;
                    load_w_tile(sA + slot * kTileBytesA, &tmW128, &tmW16, &full[s], kb, r0 + t * kTileV, trows,
                                pol_w);
                    tma_load_2d(sB + slot * kBBytes, &tmH, &full[s], kb * kBK, c * kAccT, pol_h);
                }
                if (++s == S) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1 && lane == 0) {
        // ------------------------------------------------ MMA issuer
        int s = 0, grp = 0;
        uint32_t ph = 0, gph = 0;
        for (int it = 0; it < nitems; ++it) {
            const int c = it % p.nchunks;
            const int ncol = min(kAccT, p.R - c * kAccT);
            const uint32_t idesc = idesc_bf16_f32(128, (uint32_t)((ncol + 15) & ~15));
            for (int kg = 0; kg < nkg; ++kg) {
                const int ng = min(kAccGK, p.num_kb - kg * kAccGK);
                mbar_wait(&pempty[grp], gph ^ 1);
                mbar_wait(&full[s], ph);
                tc_fence_after();
                for (int g = 0; g < ng; ++g) {
                    const uint32_t dt = tbase + (uint32_t)((grp * kAccGK + g) * kAccT);
                    const size_t slot = (size_t)s * kAccGK + g;
                    const uint64_t ad = sdesc_sw128(sA + slot * kTileBytesA);
                    const uint64_t bd = sdesc_sw128(sB + slot * kBBytes);
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k) mma_bf16(dt, ad + 2 * k, bd + 2 * k, idesc, k != 0);
                }
                mma_commit(&empty[s]);
                mma_commit(&pfull[grp]);
                if (++s == S) { s = 0; ph ^= 1; }
                if (++grp == 2) { grp = 0; gph ^= 1; }
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------ epilogue (8 warps)
        const int q = warp & 3;
        const int e = (warp - 4) >> 2;   // column half
        const uint32_t lane_base = tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(e * kAccNC);
        const int vr = q * 32 + lane;
        const uint64_t pol_keep = policy_evict_last();   // staged logits stay in L2 for the sampler
        int grp = 0;
        uint32_t gph = 0;
        for (int it = 0; it < nitems; ++it) {
            const int t = it / p.nchunks, c = it - t * p.nchunks;
            const int c0 = c * kAccT;
            const int ncol = min(kAccT, p.R - c0);
            float acc[kAccNC];
#pragma unroll
            for (int j = 0; j < kAccNC; ++j) acc[j] = 0.f;
            for (int kg = 0; kg < nkg; ++kg) {
                const int ng = min(kAccGK, p.num_kb - kg * kAccGK);
                mbar_wait(&pfull[grp], gph);
                tc_fence_after();
                for (int g = 0; g < ng; ++g) {
#pragma unroll
                    for (int h = 0; h < kAccNC / 16; ++h) {
                        float v[16];
                        tmem_ld16(lane_base + (uint32_t)((grp * kAccGK + g) * kAccT + h * 16), v);
#pragma unroll
                        for (int i = 0; i < 16; ++i) acc[h * 16 + i] += v[i];   // fp32 RN, unbiased
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&pempty[grp]);
                if (++grp == 2) { grp = 0; gph ^= 1; }
            }
            const bool valid = vr < min(kTileV, rows - t * kTileV);
            const int xl = r0 + t * kTileV + vr;
#pragma unroll
            for (int j = 0; j < kAccNC; ++j) {
                const int col = e * kAccNC + j;
                if (col < ncol) {
                    const int row = c0 + col;
                    if (WRITE && valid) st_evict_last(&p.logits[(int64_t)row * p.ld_out + xl], acc[j], pol_keep);
                    if (CAPTURE && valid && stok[row] == xl) p.dl[p.use_row_g ? p.row_g[row] : row] = (double)acc[j];
                }
            }
            if (STATS) {
                // two reduce-scatters of 32 columns: lane l then owns column
                // col_of_lane<32>(l) of each half -> scratch[e][q][col]; the 4
                // quadrant warps of half e merge them into the row state
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    float tm[32], ts[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int col = e * kAccNC + hh * 32 + j;
                        const bool ok = valid && col < ncol;
                        tm[j] = ok ? acc[hh * 32 + j] : -INFINITY;
                        ts[j] = ok ? 1.f : 0.f;
                    }
                    float wm, ws;
                    warp_scatter_ms<32>(tm, ts, wm, ws);
                    scratch[(e * 4 + q) * kAccNC + hh * 32 + col_of_lane<32>(lane)] = make_float2(wm, ws);
                }
                named_bar(1 + e, 128);
                const int ht = (warp - 4 - 4 * e) * 32 + lane;   // 0..127 within the half
                if (ht < kAccNC) {
                    const int col = e * kAccNC + ht;
                    if (col < ncol) {
                        float2 st = state[c0 + col];
#pragma unroll
                        for (int w = 0; w < 4; ++w) {
                            const float2 o = scratch[(e * 4 + w) * kAccNC + ht];
                            ms_merge(st.x, st.y, o.x, o.y);
                        }
                        state[c0 + col] = st;
                    }
                }
                named_bar(1 + e, 128);
            }
        }
    }
    __syncthreads();
    if (STATS)
        for (int i = threadIdx.x; i < p.R; i += kAccThreads) {
            p.part_m[(int64_t)i * p.part_ld + cta] = state[i].x;
            p.part_s[(int64_t)i * p.part_ld + cta] = state[i].y;
        }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_dealloc(tbase, 512);
}
