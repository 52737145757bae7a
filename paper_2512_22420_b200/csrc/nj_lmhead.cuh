// nj_lmhead.cuh — k_lmhead<MODE, CG>: the LM-head GEMM of the staged path
// (every N > 48), with tokens on the TMEM lanes and the vocabulary along the
// MMA N dimension.  Included from nj_gemm.cuh (namespace nj).
//
// BJ step (1) l_j(x) = sum_k W[x,k] h_j[k]
// with BJ step (2)'s online-softmax statistics (row a3), the draft-logit
// capture of step (3) and, for greedy verification, the row argmax fused into
// the epilogue.
//
// Why a second GEMM: k_gemm_big puts 128 vocab rows on the TMEM
// lanes and up to 256 tokens on N, so (i) each row's softmax statistics are
// column reductions across lanes (shuffles, shared scratch, CAS merges: ~8 us
// of exposed epilogue per item) and (ii) per SM and k-block it pulls 16 KB of
// W + 32 KB of H from L2, and the L2 -> SM operand stream (~15 TB/s measured
// chip-wide, ~50 B/cycle/SM) -- not the tensor pipe -- bounds it above the
// ridge.  Here
//   * MMA M = the token rows (128 per CTA; 256 over a CTA pair with
//     cta_group::2), N = a vocab tile of <= 256 ids: thread (quadrant q, lane)
//     of an epilogue warp owns token row 32q + lane, so row statistics, the
//     argmax and the draft-logit capture are per-thread register loops;
//   * a CTA pair loads its own 128 token rows of H (A) and HALF of the W tile
//     (B): 16 + 16 KB per SM and k-block for a 128 x 256 x 64 MMA step
//     (-33 % operand traffic);
//   * every pair (CTA) owns a contiguous vocabulary range split into tiles of
//     equal width (multiple of 16, <= 256): the load is balanced to 16 ids
//     whatever V (round-robin 128-row tiles leave 8-11 % idle at V = 152064),
//     and for each tile it runs all token chunks back to back, so a W tile is
//     read from HBM once and from L2 by the other chunks one item later;
//   * the accumulator restarts every `ks` k-blocks (accuracy);
//     16 epilogue warps add the partials into fp32 round-to-nearest running
//     sums in registers (4 warps per lane quadrant, interleaved 16-column
//     granules), with as many TMEM buffers as the tile width allows.
#pragma once

constexpr int kLmEpiWarps = 16;
constexpr int kLmThreads = (kLmEpiWarps + 2) * 32;   // warps 0..15 epilogue, 16 TMA, 17 MMA/TMEM
constexpr int kLmWarpTMA = kLmEpiWarps, kLmWarpMMA = kLmEpiWarps + 1;
constexpr int kLmTok = 128;                          // token rows per CTA and chunk (MMA M per CTA)
constexpr int kLmMaxNV = 256;                        // vocab tile width upper bound (MMA N)
constexpr int kLmNC = 64;                            // accumulator registers per thread (4 granules of 16)
constexpr int kLmMaxBuf = 8;
constexpr int kLmHBytes = kLmTok * kBK * 2;          // 16 KB H box per k-block

enum : int { LM_WRITE = 1, LM_STATS = 2, LM_CAPTURE = 4, LM_ARGMAX = 8 };

struct LmheadParams {
    float inv_t;                 // 1 / temperature applied to the logits (1: none)
    int32_t R;                   // token rows
    int32_t nchunks;             // token chunks of 128 * CG rows; unit u works on chunk u % nchunks over the
                                 // vocabulary range of group u / nchunks (nunits = groups x nchunks)
    int32_t V_local, U, num_kb;  // local vocabulary, its 16-id units, k-blocks
    int32_t nstages, gk, ks;     // ring stages, k-blocks per stage, k-blocks per accumulator restart
    int32_t mb;                  // ring stages the MMA warp consumes per operand wait (1, 2, ...)
    int32_t nstages_mem;         // probe only (no-load runs): ring stages backed by shared memory (0: all)
    int32_t sleep_ns;            // epilogue accumulator waits: test_wait + nanosleep backoff (0: try_wait)
    int32_t ks0;                 // k-blocks of the first accumulator group of every item (>= ks)
    int32_t arv1;                // 1: one accumulator-release arrival per CTA (named barrier first)
    int32_t fence_full;          // probe: tcgen05.fence::after_thread_sync after every operand wait
    int32_t mma4;                // 1: a k-block's four MMAs issued from one asm block under one elect
    int32_t* zero_ptr;           // staged step: CTA 0 zeroes zero_ptr[0, zero_n) (the fallback block the
    int32_t zero_n;              //    sampler kernels read after this grid; replaces a memset node)
    int32_t out_keep;            // 1: TMA logits stores with an L2 evict_last hint (small R: the sampler
                                 //    re-reads them right after; W streams evict_first)
    int32_t pdl;                 // 1: trigger the dependent grid's launch at the start (k_sample_small's
                                 //    CTAs take the SMs this grid's CTAs free; they wait for its writes)
    int32_t nbuf, bstride;       // TMEM accumulator buffers and their column stride
    int32_t tile_w;              // vocab tile width (multiple of 16, <= 256; the last tile of a range is ragged)
    int32_t wbox;                // W box rows per CTA (tile_w / CG)
    int32_t hbox;                // H box rows (128, or R rounded up to 8 for a single CTA chunk)
    int32_t w_evict_first;
    int32_t pf;                  // W L2 prefetch distance in k-blocks (0: off); issued 4 k-blocks at a time
    float* logits;               // WRITE: [R][ld_out] fp32 (local vocab ids)
    int64_t ld_out;
    int32_t ost_n;               // WRITE via TMA: staging boxes per epilogue warp (1 or 2)
    int32_t tma_out;             // WRITE: 1 = TMA tensor stores of 32 x 16 boxes staged in swizzled smem
                                 // (tmL, SWIZZLE_64B); 0 = direct 16-byte stores (ld_out % 4 != 0)
    float* part_m;               // STATS: [R][part_ld] per-group (max, sum e^{l - max});
    float* part_s;               // ARGMAX: (order-preserving uint32 of the max as float bits, id as int bits)
    int32_t part_ld;
    const int32_t* tok;          // CAPTURE: draft tokens (global ids)
    double* dl;                  // CAPTURE: fp64 draft logits
    int32_t cap_staged;          // 1: rows request-major (row_off); row r of request b is draft row r - b,
                                 //    its last row the bonus row (no capture); 0: row r is draft row r
    int32_t v_begin;
    int32_t dbg;                 // probe bits (results garbage): 1 no MMAs, 2 no TMEM drain, 8 no per-item output,
                                 // 16 no H loads, 32 no W loads, 64 every unit loads unit 0's addresses,
                                 // 128 no logits stores, 256 no statistics, 512 no ring handshakes (with 48)
    unsigned long long* ts;      // debug timeline of CTA 0 (NJ_PHASE_TS): [0, 4K) producer (wait start, wait
                                 // end) per stage, [4K, 8K) MMA (wait start, wait end, commit) per stage,
                                 // [8K, 12K) epilogue warp 0 (output start, output end) per item
    const float* qpf;            // optional: draft-probability rows prefetched into L2 by the producer
    int64_t qpf_ld;              //   warps (the staged sampler reads the rejected ones right after)
    int32_t qpf_rows, qpf_cols;
    int32_t B;
    int32_t row_off[kMaxB + 1];
};

// this unit's (pair's / CTA's) vocabulary range and its tiling
struct LmRange {
    int r0, rows, ntile, w;
};
__device__ __forceinline__ LmRange lm_range(const LmheadParams& p, int unit, int nunits) {
    LmRange g;
    vocab_range(p.U, nunits, unit, p.V_local, g.r0, g.rows);
    // tiles of tile_w ids (the host's balanced width for the largest range: a
    // multiple of 16, <= 256, the W box and TMEM buffers are sized for it), the
    // last one ragged (MMA N rounded up to 16)
    g.w = p.tile_w;
    g.ntile = (g.rows + g.w - 1) / g.w;
    return g;
}

__device__ __forceinline__ void st_f4_hint(float* p, float a, float b, float c, float d, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(a), "f"(b), "f"(c),
                 "f"(d), "l"(pol)
                 : "memory");
}

template <int MODE, int CG>
__global__ void __launch_bounds__(kLmThreads, 1)
k_lmhead(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmH,
         const __grid_constant__ CUtensorMap tmL, const __grid_constant__ LmheadParams p) {
    constexpr bool WRITE = MODE & LM_WRITE, STATS = MODE & LM_STATS, CAPTURE = MODE & LM_CAPTURE,
                   ARGMAX = MODE & LM_ARGMAX;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int S = p.nstages, GK = p.gk;
    const int SM_ = p.nstages_mem > 0 ? p.nstages_mem : S;   // ring stages backed by memory (probe: < S)
    const uint32_t wBytes = (uint32_t)p.wbox * 128u;                 // this CTA's W box per k-block
    // H box: 128 token rows, or fewer (a multiple of 8) when the launch has fewer rows
    // (single chunk): the MMA still reads 128 rows, the ones past the box are garbage
    // rows of unused TMEM lanes (never output)
    const uint32_t hBytes = (uint32_t)p.hbox * 128u;
    const size_t stageBytes = (size_t)GK * (hBytes + wBytes);
    const int nloc = kLmTok;                                          // this CTA's token rows (one chunk)
    uint8_t* ring = smem;
    // WRITE via TMA: per epilogue warp two 2-KB staging boxes (32 rows x 16 fp32, 64B-swizzled)
    uint8_t* ostage = ring + (size_t)SM_ * stageBytes;
    const size_t ostageBytes = (WRITE && p.tma_out) ? (size_t)kLmEpiWarps * p.ost_n * 2048 : 0;
    float2* state = reinterpret_cast<float2*>(ostage + ostageBytes);   // [4 slices][nloc]
    int32_t* stok = reinterpret_cast<int32_t*>(state + ((STATS || ARGMAX) ? 4 * nloc : 0));   // [nloc]
    int32_t* sdl = stok + (CAPTURE ? nloc : 0);                                                 // [nloc]
    uint64_t* bars = reinterpret_cast<uint64_t*>(
        (reinterpret_cast<uintptr_t>(sdl + (CAPTURE ? nloc : 0)) + 7) & ~uintptr_t(7));
    uint64_t* full = bars;
    uint64_t* empty = bars + S;
    uint64_t* afull = bars + 2 * S;
    uint64_t* aempty = afull + kLmMaxBuf;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + kLmMaxBuf);
    const int NBUF = p.nbuf;

    const int warp = (int)warp_id(), lane = (int)lane_id();
    const int crank = CG == 2 ? (int)cluster_ctarank() : 0;
    const bool leader = crank == 0;
    const int unit = CG == 2 ? (int)cluster_id_x() : (int)blockIdx.x;
    const int nunits = CG == 2 ? (int)nclusters_x() : (int)gridDim.x;
    // the nchunks units of a group share its vocabulary range, one token chunk each, so
    // they read every W tile at about the same time (one HBM read, L2 for the others)
    // and the live W set is ~grid / nchunks tiles
    const int group = unit / p.nchunks, cfix = unit - group * p.nchunks;
    const LmRange rg = lm_range(p, group, nunits / p.nchunks);
    const int nitems = rg.ntile;   // item it: tile it of the range, chunk cfix
    const int ngk = (p.num_kb + GK - 1) / GK;

    if (p.pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // every thread
    if (p.zero_ptr && blockIdx.x == 0)
        for (int i = threadIdx.x; i < p.zero_n; i += kLmThreads) p.zero_ptr[i] = 0;
    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmW);
        tma_prefetch_desc(&tmH);
        if (WRITE && p.tma_out) tma_prefetch_desc(&tmL);
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int g = 0; g < NBUF; ++g) { mbar_init(&afull[g], 1); mbar_init(&aempty[g], (p.arv1 ? 1 : kLmEpiWarps) * CG); }
        fence_barrier_init();
        fence_proxy_async();
    }
    if (warp == kLmWarpMMA) {
        if (CG == 2) tmem_alloc_cg2(tmem_slot, 512);
        else tmem_alloc(tmem_slot, 512);
    }
    if (STATS || ARGMAX)
        for (int i = threadIdx.x; i < 4 * nloc; i += kLmThreads)
            state[i] = ARGMAX ? make_float2(__uint_as_float(0u), __int_as_float(0x7fffffff)) : make_float2(-INFINITY, 0.f);
    if (CAPTURE)
        for (int i = threadIdx.x; i < nloc; i += kLmThreads) {
            const int row = cfix * kLmTok * CG + crank * kLmTok + i;
            int g = -1;
            if (row < p.R) {
                if (p.cap_staged) {
                    int lo = 0, hi = p.B;   // request b: row_off[b] <= row < row_off[b + 1]
                    while (hi - lo > 1) {
                        const int mid = (lo + hi) >> 1;
                        if (p.row_off[mid] <= row) lo = mid; else hi = mid;
                    }
                    g = row + 1 < p.row_off[lo + 1] ? row - lo : -1;
                } else {
                    g = row;
                }
            }
            sdl[i] = g;
            stok[i] = g >= 0 ? p.tok[g] - p.v_begin : -1;
        }
    tc_fence_before();
    if (CG == 2) cluster_sync_all();   // peer barriers initialised before any remote signal
    else __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;

    const bool noring = (p.dbg & 512) != 0;   // probe: no ring handshakes at all (no loads either)
    if (warp == kLmWarpTMA) {
      if (!noring) {
        // ------------------------------------------------ TMA producer (both CTAs)
        // whole warp in convergent control flow, one elected lane issues
        if (p.qpf && lane == 0) {
            // this CTA's share of the q rows, 32 KB segments, spread over the grid
            constexpr int kSeg = 8192;   // floats
            const int nseg = (p.qpf_cols + kSeg - 1) / kSeg;
            for (int i = (int)blockIdx.x; i < p.qpf_rows * nseg; i += (int)gridDim.x) {
                const int r = i / nseg, sg = i - r * nseg;
                const int c0 = sg * kSeg, n = min(kSeg, p.qpf_cols - c0) & ~3;
                if (n > 0) bulk_prefetch_l2(p.qpf + (int64_t)r * p.qpf_ld + c0, (uint32_t)n * 4u);
            }
        }
        const uint64_t pol_w = p.w_evict_first ? policy_evict_first() : policy_evict_last();
        const uint64_t pol_h = policy_evict_last();
        int s = 0;
        uint32_t ph = 0;
        for (int it = 0; it < nitems; ++it) {
            const int ti = it, c = cfix;
            const int v0 = rg.r0 + ti * rg.w;
            const int wn = min(rg.w, rg.r0 + rg.rows - v0);               // ids of this tile
            const int nmma = (wn + 15) & ~15;
            // this CTA's W rows: the first (CG = 1) or second (rank 1) half of the MMA's N rows;
            // a box past the local vocabulary is clamped (its rows are masked in the epilogue)
            int wrow = min(v0 + crank * (nmma / CG), p.V_local - 1);
            const int hrow = c * kLmTok * CG + crank * kLmTok;
            if (p.dbg & 64) wrow = ti * rg.w + crank * (nmma / CG);   // probe: unit 0's W rows
            for (int kg = 0; kg < ngk; ++kg) {
                const int ng = min(GK, p.num_kb - kg * GK);
                const int si = it * ngk + kg;
                const bool tsx = p.ts != nullptr && blockIdx.x == 0 && lane == 0 && si < 2000;
                if (tsx) p.ts[2 * si] = globaltimer();
                mbar_wait_w(&empty[s], ph ^ 1);
                if (tsx) p.ts[2 * si + 1] = globaltimer();
                uint8_t* st = ring + (size_t)(s % SM_) * stageBytes;
                const bool ldh = !(p.dbg & 16), ldw = !(p.dbg & 32);   // probes
                const uint32_t kbb = (ldh ? hBytes : 0u) + (ldw ? wBytes : 0u);
                if (CG == 1) {
                    if (kbb) mbar_arrive_expect_tx_w(&full[s], (uint32_t)ng * kbb);
                    else mbar_arrive_w(&full[s]);
                    for (int g = 0; g < ng; ++g) {
                        const int kb = kg * GK + g;
                        if (ldh) tma_load_2d_w(st + (size_t)g * hBytes, &tmH, &full[s], kb * kBK, hrow, pol_h);
                        if (ldw)
                            tma_load_2d_w(st + (size_t)GK * hBytes + (size_t)g * wBytes, &tmW, &full[s], kb * kBK,
                                          wrow, pol_w);
                    }
                } else {
                    // both CTAs' bytes complete on the LEADER's full[s]
                    if (leader) {
                        if (kbb) mbar_arrive_expect_tx_w(&full[s], (uint32_t)ng * 2u * kbb);
                        else mbar_arrive_w(&full[s]);
                    }
                    const uint32_t fbs = mapa_shared(&full[s], 0);
                    for (int g = 0; g < ng; ++g) {
                        const int kb = kg * GK + g;
                        if (ldh) tma_load_2d_cg2_w(st + (size_t)g * hBytes, &tmH, fbs, kb * kBK, hrow, pol_h);
                        if (ldw)
                            tma_load_2d_cg2_w(st + (size_t)GK * hBytes + (size_t)g * wBytes, &tmW, fbs, kb * kBK,
                                              wrow, pol_w);
                    }
                }
                if (p.pf > 0 && (kg * GK) % 4 == 0) {
                    // L2 prefetch of W k-blocks [kb + pf, kb + pf + 4) of this or a later tile:
                    // four boxes back to back = 512 contiguous bytes per W row (DRAM page locality)
                    const int tgt = it * p.num_kb + kg * GK + p.pf;
                    const int pit = tgt / p.num_kb, pkb = tgt - pit * p.num_kb;
                    if (pit < nitems) {
                        const int pv0 = rg.r0 + pit * rg.w;
                        const int pn = (min(rg.w, rg.r0 + rg.rows - pv0) + 15) & ~15;
                        const int prow = min(pv0 + crank * (pn / CG), p.V_local - 1);
                        for (int k = 0; k < 4 && pkb + k < p.num_kb; ++k)
                            tma_prefetch_l2_2d_w(&tmW, (pkb + k) * kBK, prow);
                    }
                }
                if (++s == S) { s = 0; ph ^= 1; }
            }
        }
      }
    } else if (warp == kLmWarpMMA) {
        if (leader) {
            // ------------------------------------------------ MMA issuer (leader CTA)
            // consumes p.mb ring stages per iteration (one operand wait + fence per mb x GK
            // k-blocks: the issuing warp is paced by the tensor pipe, so its per-iteration
            // overhead is exposed)
            int s = 0, abuf = 0, gall = 0;
            uint32_t ph = 0, aph = 0;
            const int MB = p.mb;
            for (int it = 0; it < nitems; ++it) {
                const int ti = it;
                const int wn = min(rg.w, rg.r0 + rg.rows - (rg.r0 + ti * rg.w));
                const uint32_t idesc = idesc_bf16_f32(kLmTok * CG, (uint32_t)((wn + 15) & ~15));
                int kin = 0;
                uint32_t dt = 0;
                for (int kg0 = 0; kg0 < ngk; kg0 += MB) {
                    const int nst = min(MB, ngk - kg0);
                    const int si = it * ngk + kg0;
                    const bool tsx = p.ts != nullptr && blockIdx.x == 0 && lane == 0 && si < 1300;
                    if (tsx) p.ts[4096 + 3 * si] = globaltimer();
                    {
                        int s2 = s;
                        uint32_t ph2 = ph;
                        for (int m = 0; m < nst && !noring; ++m) {
                            mbar_wait_w(&full[s2], ph2);
                            if (++s2 == S) { s2 = 0; ph2 ^= 1; }
                        }
                    }
                    if (tsx) p.ts[4096 + 3 * si + 1] = globaltimer();
                    // (no tcgen05 fence here: the operands are TMA-written shared memory that the
                    // MMAs read through the async proxy; the full barrier's completion orders them)
                    if (p.fence_full) tc_fence_after();
                    for (int m = 0; m < nst; ++m) {
                        const int kg = kg0 + m;
                        const int ng = min(GK, p.num_kb - kg * GK);
                        uint8_t* st = ring + (size_t)(s % SM_) * stageBytes;
                        for (int g = 0; g < ng; ++g) {
                            if (kin == 0) {
                                const int gw = gall++;   // accumulator groups issued so far (timeline index)
                                const bool tsa = p.ts != nullptr && blockIdx.x == 0 && lane == 0 && gw < 1000;
                                if (tsa) p.ts[16384 + 2 * gw] = globaltimer();
                                mbar_wait_w(&aempty[abuf], aph ^ 1);
                                if (tsa) p.ts[16384 + 2 * gw + 1] = globaltimer();
                                tc_fence_after();
                                dt = tbase + (uint32_t)(abuf * p.bstride);
                            }
                            const uint64_t ad = sdesc_sw128(st + (size_t)g * hBytes);
                            const uint64_t bd = sdesc_sw128(st + (size_t)GK * hBytes + (size_t)g * wBytes);
                            if (!(p.dbg & 1)) {
                                if (p.mma4) {
                                    mma_kblock_w<CG>(dt, ad, bd, idesc, kin != 0);
                                } else {
#pragma unroll
                                    for (int k = 0; k < kBK / 16; ++k) {
                                        if (CG == 2) mma_bf16_cg2_w(dt, ad + 2 * k, bd + 2 * k, idesc, (kin | k) != 0);
                                        else mma_bf16_w(dt, ad + 2 * k, bd + 2 * k, idesc, (kin | k) != 0);
                                    }
                                }
                            }
                            const int kb = kg * GK + g;
                            // group boundary: the first group of an item spans ks0 k-blocks, the
                            // rest ks (the longer first group covers the epilogue's per-item output)
                            if (++kin == (kb < p.ks0 ? p.ks0 : p.ks) || kb == p.num_kb - 1) {
                                if (CG == 2) mma_commit_mc2_w(&afull[abuf], 3);
                                else mma_commit_w(&afull[abuf]);
                                if (++abuf == NBUF) { abuf = 0; aph ^= 1u; }
                                kin = 0;
                            }
                        }
                        if (!noring) {
                            if (CG == 2) mma_commit_mc2_w(&empty[s], 3);
                            else mma_commit_w(&empty[s]);
                        }
                        if (++s == S) { s = 0; ph ^= 1; }
                    }
                    if (tsx) p.ts[4096 + 3 * si + 2] = globaltimer();
                }
            }
        }
    } else {
        // ------------------------------------------------ epilogue (16 warps per CTA)
        // warp (q = warp & 3, e = warp >> 2): TMEM lanes 32q..32q+31 (token rows), granules
        // e, e + 4, e + 8, e + 12 of 16 vocab columns (acc[16 j + i] = granule e + 4 j)
        const int q = warp & 3, e = warp >> 2;
        const uint32_t lane_base = tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(e * 16);
        // a lane quadrant whose 32 token rows are all past R drains nothing (it still releases)
        const bool quad_empty = cfix * kLmTok * CG + crank * kLmTok + q * 32 >= p.R;
        const int ngroups = p.num_kb <= p.ks0 ? 1 : 1 + (p.num_kb - p.ks0 + p.ks - 1) / p.ks;
        const uint64_t pol_out = policy_evict_first();   // logits: do not push W / H out of L2
        const uint64_t pol_keep = policy_evict_last();   // out_keep: small staged logits stay for the sampler
        const bool vec_ok = (p.ld_out & 3) == 0 && (reinterpret_cast<uintptr_t>(p.logits) & 15) == 0;
        uint8_t* my_ost = ostage + (size_t)warp * p.ost_n * 2048;   // this warp's staging boxes
        int osb = 0;                                          // next staging box
        int ebuf = 0;
        uint32_t eph = 0;
        for (int it = 0; it < nitems; ++it) {
            const int ti = it, c = cfix;
            const int v0t = rg.r0 + ti * rg.w;
            const int wn = min(rg.w, rg.r0 + rg.rows - v0t);
            const int ngr = (wn + 15) >> 4;   // granules of this tile
            const int myg = ngr > e ? (ngr - e + 3) >> 2 : 0;   // granules of this warp (0..4)
            float acc[kLmNC];
#pragma unroll
            for (int j = 0; j < kLmNC; ++j) acc[j] = 0.f;
            for (int g = 0; g < ngroups; ++g) {
                const int buf = ebuf;
                const int gi = it * ngroups + g;
                const bool tsg = p.ts != nullptr && blockIdx.x == 0 && warp == 0 && lane == 0 && gi < 1000;
                if (tsg) p.ts[12288 + 2 * gi] = globaltimer();
                if (p.sleep_ns > 0) mbar_wait_sleep(&afull[buf], eph, (uint32_t)p.sleep_ns);
                else mbar_wait(&afull[buf], eph);
                if (tsg) p.ts[12288 + 2 * gi + 1] = globaltimer();
                if (++ebuf == NBUF) { ebuf = 0; eph ^= 1; }
                tc_fence_after();
                const uint32_t ta = lane_base + (uint32_t)(buf * p.bstride);
                if (!(p.dbg & 2) && !quad_empty) {
                    if (myg >= 2) {
                        float v[32];
                        tmem_ld16x2(ta, ta + 64u, v);
#pragma unroll
                        for (int i = 0; i < 32; ++i) acc[i] += v[i];   // fp32 RN, unbiased
                        if (myg >= 4) {
                            tmem_ld16x2(ta + 128u, ta + 192u, v);
#pragma unroll
                            for (int i = 0; i < 32; ++i) acc[32 + i] += v[i];
                        } else if (myg == 3) {
                            float w[16];
                            tmem_ld16(ta + 128u, w);
#pragma unroll
                            for (int i = 0; i < 16; ++i) acc[32 + i] += w[i];
                        }
                    } else if (myg == 1) {
                        float v[16];
                        tmem_ld16(ta, v);
#pragma unroll
                        for (int i = 0; i < 16; ++i) acc[i] += v[i];
                    }
                }
                tc_fence_before();
                if (p.arv1) {
                    // one arrival per CTA: the 16 epilogue warps meet at a named barrier first
                    named_bar(1, kLmEpiWarps * 32);
                    if (warp == 0 && lane == 0) {
                        if (CG == 2) mbar_arrive_cluster(mapa_shared(&aempty[buf], 0));
                        else mbar_arrive(&aempty[buf]);
                    }
                } else {
                    __syncwarp();
                    if (lane == 0) {
                        if (CG == 2) mbar_arrive_cluster(mapa_shared(&aempty[buf], 0));
                        else mbar_arrive(&aempty[buf]);
                    }
                }
                if (tsg) p.ts[14336 + gi] = globaltimer();
            }
            const bool tso = p.ts != nullptr && blockIdx.x == 0 && warp == 0 && lane == 0 && it < 2000;
            if (tso) p.ts[8192 + 2 * it] = globaltimer();
            if (p.dbg & 8) continue;   // probe: no per-item output
            const int lr = q * 32 + lane;                                  // index into this CTA's rows
            const int row = c * kLmTok * CG + crank * kLmTok + q * 32 + lane;
            if (myg == 0 || row - lane >= p.R) continue;   // warp-uniform: nothing of this warp's box exists
            if (p.inv_t != 1.f) {
#pragma unroll
                for (int j = 0; j < kLmNC; ++j) acc[j] *= p.inv_t;
            }
            // valid columns of granule j: [0, nv_j); the tile's last granule may be ragged
            int nvj[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) nvj[j] = j < myg ? min(16, wn - (e + 4 * j) * 16) : 0;
            // row statistics: the item max first (one pass), then the exponentials granule by
            // granule, interleaved with the granule's TMA store (its smem read overlaps them)
            float2 stt = make_float2(-INFINITY, 0.f);
            float s4[4] = {0.f, 0.f, 0.f, 0.f};   // four chains (latency)
            const bool do_stats = STATS && !(p.dbg & 256) && row < p.R;
            if (do_stats) {
                float mx = -INFINITY;
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        if (i < nvj[j]) mx = fmaxf(mx, acc[16 * j + i]);
                stt = state[e * nloc + lr];
                if (mx > stt.x) {
                    stt.y *= __expf(stt.x - mx);   // stt.x = -inf: stt.y = 0
                    stt.x = mx;
                }
            }
            const bool tma_w = WRITE && p.tma_out && !(p.dbg & 128);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (j >= myg) break;
                if (tma_w) {
                    // granule j -> staging box (row = lane, 16-byte chunk i at i ^ ((lane >> 1) & 3): the
                    // SWIZZLE_64B pattern, conflict-free) -> one TMA store of rows [row - lane, +32) x 16
                    // ids (rows past R / ids past V_local are clipped by the tensor map)
                    if (p.ost_n == 1) bulk_wait_read<0>();   // the previous box has been read
                    else bulk_wait_read<1>();                // the box before it
                    __syncwarp();
                    uint8_t* box = my_ost + osb * 2048;
                    const int sw = (lane >> 1) & 3;
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        *reinterpret_cast<float4*>(box + lane * 64 + ((i ^ sw) << 4)) =
                            make_float4(acc[16 * j + 4 * i], acc[16 * j + 4 * i + 1], acc[16 * j + 4 * i + 2],
                                        acc[16 * j + 4 * i + 3]);
                    fence_proxy_async();   // generic-proxy smem writes -> visible to the TMA (async proxy)
                    __syncwarp();
                    if (lane == 0) {
                        if (p.out_keep) tma_store_2d_hint(&tmL, box, v0t + (e + 4 * j) * 16, row - lane, pol_keep);
                        else tma_store_2d(&tmL, box, v0t + (e + 4 * j) * 16, row - lane);
                        bulk_commit();
                    }
                    if (p.ost_n == 2) osb ^= 1;
                }
                if (do_stats) {
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        if (i < nvj[j]) s4[i & 3] += __expf(acc[16 * j + i] - stt.x);
                }
            }
            if (do_stats) {
                stt.y += (s4[0] + s4[1]) + (s4[2] + s4[3]);
                state[e * nloc + lr] = stt;
            }
            if (WRITE && !p.tma_out && !(p.dbg & 128) && row < p.R) {
                float* pr = p.logits + (int64_t)row * p.ld_out + v0t + e * 16;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (nvj[j] == 16 && vec_ok) {
#pragma unroll
                        for (int i = 0; i < 16; i += 4)
                            st_f4_hint(pr + 64 * j + i, acc[16 * j + i], acc[16 * j + i + 1], acc[16 * j + i + 2],
                                       acc[16 * j + i + 3], pol_out);
                    } else {
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            if (i < nvj[j]) pr[64 * j + i] = acc[16 * j + i];
                    }
                }
            }
            if (row >= p.R) continue;   // rows past R (the TMA stores above clipped them)
            if (CAPTURE) {
                const int tk = stok[lr] - v0t;   // tile column of this row's draft token
                const int gj = tk >> 4;          // its granule
                if (tk >= 0 && tk < wn && (gj & 3) == e) {
                    const int idx = (gj >> 2) * 16 + (tk & 15);
                    float val = 0.f;
#pragma unroll
                    for (int jj = 0; jj < kLmNC; ++jj)
                        if (jj == idx) val = acc[jj];
                    p.dl[sdl[lr]] = (double)val;
                }
            }
            if (ARGMAX) {
                // highest logit, lowest id among equals: values compared as order-preserving
                // uint32 (the key of k_argmax_rows / the oracle's argmax, -0 < +0), ascending
                // scan with strict > inside the item, (ord, -id) merge into the row state
                uint32_t bo = 0u;
                int bi = -1;
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        if (i < nvj[j]) {
                            const uint32_t u = __float_as_uint(acc[16 * j + i]);
                            const uint32_t o = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
                            if (bi < 0 || o > bo) { bo = o; bi = v0t + (e + 4 * j) * 16 + i; }
                        }
                if (bi >= 0) {
                    const float2 st = state[e * nloc + lr];
                    const uint32_t so = __float_as_uint(st.x);
                    const int sid = __float_as_int(st.y);
                    if (bo > so || (bo == so && bi < sid))
                        state[e * nloc + lr] = make_float2(__uint_as_float(bo), __int_as_float(bi));
                }
            }
            if (tso) p.ts[8192 + 2 * it + 1] = globaltimer();
        }
    }
    if (WRITE && p.tma_out && warp < kLmEpiWarps && lane == 0) bulk_wait<0>();   // stores complete before exit
    __syncthreads();
    if (p.ts != nullptr && threadIdx.x == 0 && blockIdx.x < 512) p.ts[20480 + blockIdx.x] = globaltimer();
    if (STATS || ARGMAX) {
        // merge the 4 column slices of every row of this CTA into its group's partial
        for (int i = threadIdx.x; i < nloc; i += kLmThreads) {
            const int row = cfix * kLmTok * CG + crank * kLmTok + i;
            if (row >= p.R) continue;
            float2 a = state[i];
            for (int e = 1; e < 4; ++e) {
                const float2 b = state[e * nloc + i];
                if (ARGMAX) {
                    const uint32_t ao = __float_as_uint(a.x), bo = __float_as_uint(b.x);
                    if (bo > ao || (bo == ao && __float_as_int(b.y) < __float_as_int(a.y))) a = b;
                } else {
                    ms_merge(a.x, a.y, b.x, b.y);
                }
            }
            p.part_m[(int64_t)row * p.part_ld + group] = a.x;
            p.part_s[(int64_t)row * p.part_ld + group] = a.y;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (CG == 2) {
        cluster_sync_all();   // neither CTA of the pair frees TMEM while the other may still signal it
        if (warp == kLmWarpMMA) tmem_dealloc_cg2(tbase, 512);
    } else if (warp == kLmWarpMMA) {
        tmem_dealloc(tbase, 512);
    }
}
