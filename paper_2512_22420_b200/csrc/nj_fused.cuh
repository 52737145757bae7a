// nj_fused.cuh — k_fused_verify<NPAD>: the whole verification step (BJ steps
// 1-3) in ONE persistent cooperative kernel for N <= 48 rows (memory-bound
// regime, BJ config 2).  Included from nj_gemm.cuh (namespace nj).
//
//   phase 1  GEMM over every row.  Accuracy: the MMA
//            accumulator is restarted every ring stage (GK = 4 k-blocks, 16
//            MMAs; NJ_SACC=0: every k-block) in a scratch TMEM buffer and the
//            epilogue sums the partials in fp64 — tcgen05 truncates (RZ) on
//            every fp32 accumulate, which over K = 3584 biases logits by
//            -3.3e-6*l; restarting cuts that ~14x (acceptance certificate
//            eps_acc_fused x the stage span, nj_api.cu).
//            The fp64 logits are captured for draft tokens and stored back to
//            TMEM as fp32 (this CTA's logits stay resident: ntiles*NPAD +
//            nbuf*NPAD <= 512 columns); softmax statistics follow from them.
//   barrier  ---- grid-wide
//   phase 2  lse of every row (fixed-order fp64 merge of the per-CTA
//            partials), Leviathan acceptance tests, first rejection
//            (every CTA redundantly and bit-identically).
//   phase 3  residual max(0, p_n - q_n) / bonus p_gamma weights of each
//            request's sample row straight from TMEM; per-warp inclusive scans
//            give per-tile masses; per-CTA mass = fixed-order fp64 sum.
//   barrier  ---- grid-wide
//   phase 4  fixed-order fp64 prefix of CTA masses locates the owning CTA,
//            which locates the tile from its stored prefixes and the token
//            with boundaries E(x) = I(x-1) built from the same fp32 scans, so
//            the intervals [E, I) tile [0, W) exactly (no gaps, no overlaps).
// W is streamed from HBM exactly once; nothing of size V x N is written.
// Every acceptance test whose margin is inside the certificate, and every
// zero-mass draw (R6), is queued for the fp64 fallback (nj_sampler.cuh); the
// draws themselves are not certified (R16, include/nj.h accuracy contract).

// NC consecutive TMEM columns, one wait (NC in {8, 16, 24, 32, 48})
template <int NC>
__device__ __forceinline__ void ld_cols(uint32_t taddr, float (&v)[NC]) {
    if constexpr (NC == 48) tmem_ld48(taddr, v);
    else if constexpr (NC == 32) tmem_ld32(taddr, v);
    else if constexpr (NC == 24) tmem_ld24(taddr, v);
    else if constexpr (NC == 16) tmem_ld16(taddr, v);
    else tmem_ld8(taddr, v);
}
template <int NC>
__device__ __forceinline__ void st_cols(uint32_t taddr, const float (&v)[NC]) {
#pragma unroll
    for (int g = 0; g < NC / 8; ++g) {
        float tmp[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) tmp[i] = v[g * 8 + i];
        tmem_st8(taddr + (uint32_t)(g * 8), tmp);
    }
}

// Warp reduce-scatter of online-softmax pairs over 32 lanes for NCP columns
// (NCP = 8/16/32): at every step each lane keeps half of its columns and merges
// the other half received from lane ^ o.  NCP merges per lane instead of
// 5 * NCP for per-column butterflies.  On return lane l holds the warp-wide
// (m, s) of column col_of_lane<NCP>(l) (every column is held by 32/NCP lanes).
template <int NCP>
__device__ __forceinline__ int col_of_lane(int l) {
    // bits consumed in order 16, 8, 4, ... while columns remain; bit set = upper half
    int col = 0, width = NCP;
#pragma unroll
    for (int o = 16; o >= 1 && width > 1; o >>= 1) {
        width >>= 1;
        if (l & o) col += width;
    }
    return col;
}
template <int NCP>
__device__ __forceinline__ void warp_scatter_ms(float (&m)[NCP], float (&s)[NCP], float& mo, float& so) {
    const int l = (int)lane_id();
    int width = NCP;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        if (width > 1) {
            const int h = width >> 1;
            const bool up = (l & o) != 0;
#pragma unroll
            for (int j = 0; j < NCP / 2; ++j) {
                if (j < h) {
                    // keep half [up ? h : 0, +h), send the other half
                    const float sm_m = up ? m[j] : m[h + j];
                    const float sm_s = up ? s[j] : s[h + j];
                    const float rm = __shfl_xor_sync(0xffffffffu, sm_m, o);
                    const float rs = __shfl_xor_sync(0xffffffffu, sm_s, o);
                    float km = up ? m[h + j] : m[j];
                    float ks = up ? s[h + j] : s[j];
                    ms_merge(km, ks, rm, rs);
                    m[j] = km;
                    s[j] = ks;
                }
            }
            width = h;
        } else {
            const float rm = __shfl_xor_sync(0xffffffffu, m[0], o);
            const float rs = __shfl_xor_sync(0xffffffffu, s[0], o);
            ms_merge(m[0], s[0], rm, rs);
        }
    }
    mo = m[0];
    so = s[0];
}

// 16 columns over 32 lanes: lanes l and l ^ 1 both end with column l >> 1.
template <int H>
__device__ __forceinline__ void scatter_ms16_level(float (&m)[16], float (&s)[16], bool up) {
#pragma unroll
    for (int j = 0; j < H / 2; ++j) {
        const float sm_m = up ? m[j] : m[H / 2 + j];
        const float sm_s = up ? s[j] : s[H / 2 + j];
        float km = up ? m[H / 2 + j] : m[j];
        float ks = up ? s[H / 2 + j] : s[j];
        const float rm = __shfl_xor_sync(0xffffffffu, sm_m, H);
        const float rs = __shfl_xor_sync(0xffffffffu, sm_s, H);
        ms_merge(km, ks, rm, rs);
        m[j] = km;
        s[j] = ks;
    }
}
__device__ __forceinline__ void warp_scatter_ms16(float (&m)[16], float (&s)[16], float& mo, float& so) {
    const int l = (int)lane_id();
    scatter_ms16_level<16>(m, s, (l & 16) != 0);
    scatter_ms16_level<8>(m, s, (l & 8) != 0);
    scatter_ms16_level<4>(m, s, (l & 4) != 0);
    scatter_ms16_level<2>(m, s, (l & 2) != 0);
    const float rm = __shfl_xor_sync(0xffffffffu, m[0], 1);
    const float rs = __shfl_xor_sync(0xffffffffu, s[0], 1);
    ms_merge(m[0], s[0], rm, rs);
    mo = m[0];
    so = s[0];
}
// Plain-op version of scatter_ms16_level / warp_scatter_ms16 (lanes l, l ^ 1 end
// with op over column l >> 1).
template <int H, typename Op>
__device__ __forceinline__ void scatter16_level(float (&v)[16], bool up, Op op) {
#pragma unroll
    for (int j = 0; j < H / 2; ++j) {
        const float send = up ? v[j] : v[H / 2 + j];
        const float keep = up ? v[H / 2 + j] : v[j];
        v[j] = op(keep, __shfl_xor_sync(0xffffffffu, send, H));
    }
}
template <typename Op>
__device__ __forceinline__ float warp_scatter16(float (&v)[16], Op op) {
    const int l = (int)lane_id();
    scatter16_level<16>(v, (l & 16) != 0, op);
    scatter16_level<8>(v, (l & 8) != 0, op);
    scatter16_level<4>(v, (l & 4) != 0, op);
    scatter16_level<2>(v, (l & 2) != 0, op);
    return op(v[0], __shfl_xor_sync(0xffffffffu, v[0], 1));
}
// Column (max, sum e^{x - max}) of 16 columns with ONE exponential per element:
// max reduce-scatter, the 16 column maxima broadcast back (lane 2j holds column
// j), e^{x - max_j} summed by a second reduce-scatter.  x: -inf = invalid;
// lanes l, l ^ 1 end with column l >> 1.
__device__ __forceinline__ void warp_colstats16(const float (&x)[16], float& mo, float& so) {
    float t[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) t[j] = x[j];
    const float cm = warp_scatter16(t, [](float a, float b) { return fmaxf(a, b); });
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const float mj = __shfl_sync(0xffffffffu, cm, 2 * j);
        t[j] = x[j] == -INFINITY ? 0.f : __expf(x[j] - mj);
    }
    mo = cm;
    so = warp_scatter16(t, [](float a, float b) { return a + b; });
}
constexpr int kFusedThreads = 384;   // warps 0-3 control, 4-11 epilogue (2 per TMEM lane quadrant)

// residual / bonus weight of one vocab entry (BJ step 3); the lse shift is
// taken in fp64 so no common-mode fp32 rounding of lse scales p against q.
// qrow: this CTA's slice of the q row in smem (x relative to the CTA start).
// p = exp(l - c) * corr with c = fp32(lse), corr = exp(c - lse) computed once in
// fp64 per request: no common-mode fp32 rounding of lse scales p against q, and
// no fp64 work per vocab entry.
__device__ __forceinline__ float sample_weight(float l, float c, float corr, bool resid, const float* qrow, int xr,
                                               bool valid) {
    if (!valid) return 0.f;
    const float pe = __expf(l - c) * corr;
    return resid ? fmaxf(pe - qrow[xr], 0.f) : pe;
}

// Debug phase stamps (NJ_PHASE_TS=1): the extra barrier plus a dependent shared
// load make the stamp wait for the whole CTA (BAR.SYNC itself is defer-blocking).
#define NJ_STAMP(k)                                                                   \
    do {                                                                              \
        if (p.phase_ts) {                                                             \
            __syncthreads();                                                          \
            const int dep_ = *reinterpret_cast<volatile int*>(&spick[0]);             \
            if (threadIdx.x == 0 && dep_ != 0x7fffffff) p.phase_ts[cta * 16 + (k)] = globaltimer(); \
        }                                                                             \
    } while (0)

template <int NPAD>
__global__ void __launch_bounds__(kFusedThreads, 1)
k_fused_verify(const __grid_constant__ CUtensorMap tmW128, const __grid_constant__ CUtensorMap tmW16,
               const __grid_constant__ CUtensorMap tmH, const FusedParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr int kBBytes = NPAD * 128;
    constexpr int kMaxT = 16;
    constexpr int kMaxBufs = 8;
    const int S = p.nstages;
    const int GK = p.kgroup;                 // k-blocks per ring stage (one barrier round trip)
    const int NB = p.nbuf;
    const uint32_t scol = (uint32_t)p.scratch_col;
    const int nkg = (p.num_kb + GK - 1) / GK;  // stages per tile
    uint8_t* sA = smem;                                       // S x GK x 16 KB
    uint8_t* sB = smem + (size_t)S * GK * kTileBytesA;        // S x GK x NPAD*128
    uint8_t* tail = sB + (size_t)S * GK * kBBytes;
    float2* red = reinterpret_cast<float2*>(tail);                        // [4][NPAD]
    double* lse_s = reinterpret_cast<double*>(red + 4 * NPAD);            // [NPAD]
    ReqInfo* req = reinterpret_cast<ReqInfo*>(lse_s + NPAD);              // [NPAD]
    float* wtile = reinterpret_cast<float*>(req + NPAD);                  // [NPAD][kMaxT][4]
    double* cprefix = reinterpret_cast<double*>(wtile + NPAD * kMaxT * 4);// [NPAD][kMaxT+1]
    double* tprime = cprefix + NPAD * (kMaxT + 1);                        // [NPAD]
    int32_t* ctok = reinterpret_cast<int32_t*>(tprime + NPAD);            // [NPAD]
    int32_t* cg = ctok + NPAD;                                            // [NPAD]
    int32_t* owner = cg + NPAD;                                           // [NPAD]
    int32_t* spick = owner + NPAD;                                        // [4]
    int32_t* dpass = spick + 4;                                           // [NPAD] per-draft test result
    int32_t* qslot = dpass + NPAD;                                        // [NPAD] q-slice slot of request b
    float* qx_sm = reinterpret_cast<float*>(qslot + NPAD);                // [NPAD] q_i(x_i) of draft rows
    float* u_sm = qx_sm + NPAD;                                           // [NPAD] uniforms
    uint64_t* bars = reinterpret_cast<uint64_t*>(
        (reinterpret_cast<uintptr_t>(u_sm + NPAD) + 7) & ~uintptr_t(7));
    uint64_t* full = bars;
    uint64_t* empty = bars + S;
    uint64_t* pfull = bars + 2 * S;   // [kMaxBufs] scratch accumulator ready
    uint64_t* pempty = pfull + kMaxBufs;  // [kMaxBufs] scratch accumulator drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pempty + kMaxBufs);

    const int warp = (int)warp_id(), lane = (int)lane_id();
    const int grid = gridDim.x, cta = blockIdx.x;
    int r0, rows;
    vocab_range(p.U, grid, cta, p.V_local, r0, rows);
    const int ntiles = (rows + kTileV - 1) / kTileV;   // host guarantees ntiles <= kMaxT, ntiles*NPAD <= 512
    const int B = p.B, N = p.N;

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmW128);
        tma_prefetch_desc(&tmW16);
        tma_prefetch_desc(&tmH);
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int b = 0; b < kMaxBufs; ++b) { mbar_init(&pfull[b], 1); mbar_init(&pempty[b], 8); }
        fence_barrier_init();
        fence_proxy_async();
        if (cta == 0) *p.fb_count = 0;   // every append happens after grid barrier 1
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    for (int j = threadIdx.x; j < NPAD; j += kFusedThreads) {   // row -> (draft index, local token)
        int tok = -1, g = -1;
        if (j < N) {
            int lo = 0, hi = B - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (p.row_off[mid] <= j) lo = mid; else hi = mid - 1;
            }
            const int pos = j - p.row_off[lo];
            const int gam = p.row_off[lo + 1] - p.row_off[lo] - 1;
            if (pos < gam) {
                g = p.row_off[lo] - lo + pos;
                tok = p.draft_tokens[g] - p.v_begin;
            }
        }
        ctok[j] = tok;
        cg[j] = g;
        // inputs of the acceptance tests, fetched now so they never sit on the
        // critical path after the grid barrier
        u_sm[j] = j < N ? __ldg(&p.u[j]) : 0.f;
        qx_sm[j] = g >= 0 ? __ldg(&p.q[(int64_t)g * p.ldq + tok + p.v_begin]) : 0.f;
    }
    if (cta == 0)
        for (int b = threadIdx.x; b < B; b += kFusedThreads) p.req_flags[b] = 0;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;
    NJ_STAMP(0);

    // =============================================================== phase 1
    if (warp == 0 && lane == 0) {
        const uint64_t pol_w = policy_evict_first();
        const uint64_t pol_h = policy_evict_last();
        int s = 0;
        uint32_t ph = 0;
        for (int t = 0; t < ntiles; ++t) {
            const int trows = min(kTileV, rows - t * kTileV);
            for (int kg = 0; kg < nkg; ++kg) {
                const int ng = min(GK, p.num_kb - kg * GK);
                mbar_wait(&empty[s], ph ^ 1);
                mbar_arrive_expect_tx(&full[s], (uint32_t)ng * (w_tile_bytes(trows) + (uint32_t)kBBytes));
                for (int g = 0; g < ng; ++g) {
                    const int kb = kg * GK + g;
                    const size_t slot = (size_t)s * GK + g;
                    load_w_tile(sA + slot * kTileBytesA, &tmW128, &tmW16, &full[s], kb, r0 + t * kTileV, trows,
                                pol_w);
                    tma_load_2d(sB + slot * kBBytes, &tmH, &full[s], kb * kBK, 0, pol_h);
                }
                if (++s == S) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1 && lane == 0) {
        // k-block partials go to scratch buffer `buf`; a partial spans kpd
        // k-blocks (accumulator restarted at its first MMA).
        constexpr uint32_t idesc = idesc_bf16_f32(128, NPAD);
        const int kpd = p.kpd;
        int s = 0, buf = 0, kin = 0;
        uint32_t ph = 0, bph = 0;
        const int NGRP = p.ngroups;   // > 0: one handshake per ring stage (GK partials)
        int grp = 0;
        uint32_t gph = 0;
        for (int t = 0; t < ntiles; ++t) {
            for (int kg = 0; kg < nkg; ++kg) {
                const int ng = min(GK, p.num_kb - kg * GK);
                if (NGRP > 0) mbar_wait(&pempty[grp], gph ^ 1);   // group buffers drained
                mbar_wait(&full[s], ph);
                tc_fence_after();
                for (int g = 0; g < ng; ++g) {
                    const int kb = kg * GK + g;
                    uint32_t dt;
                    if (NGRP > 0) {
                        // sacc: the stage's GK k-blocks accumulate into ONE partial
                        // (restart every GK k-blocks); else one partial per k-block
                        dt = tbase + scol + (uint32_t)((p.sacc ? grp : grp * GK + g) * NPAD);
                    } else {
                        if (kin == 0) { mbar_wait(&pempty[buf], bph ^ 1); tc_fence_after(); }
                        dt = tbase + scol + (uint32_t)(buf * NPAD);
                    }
                    const size_t slot = (size_t)s * GK + g;
                    const uint64_t ad = sdesc_sw128(sA + slot * kTileBytesA);
                    const uint64_t bd = sdesc_sw128(sB + slot * kBBytes);
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k)
                        mma_bf16(dt, ad + 2 * k, bd + 2 * k, idesc, ((NGRP > 0 && p.sacc ? g : kin) | k) != 0);
                    if (NGRP == 0 && (++kin == kpd || kb + 1 == p.num_kb)) {
                        mma_commit(&pfull[buf]);
                        kin = 0;
                        if (++buf == NB) { buf = 0; bph ^= 1; }
                    }
                }
                mma_commit(&empty[s]);
                if (NGRP > 0) {
                    mma_commit(&pfull[grp]);
                    if (++grp == NGRP) { grp = 0; gph ^= 1; }
                }
                if (++s == S) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp >= 4) {
        // 8 epilogue warps: quadrant q = warp % 4 (TMEM lanes 32q..32q+31),
        // column slice e = (warp - 4) / 4 of NC = NPAD/2 columns.
        constexpr int NC = NPAD / 2;
        const int q = warp & 3;
        const int e = (warp - 4) >> 2;
        const uint32_t lane_base = tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(e * NC);
        const int vr = q * 32 + lane;
        int buf = 0;
        uint32_t bph = 0;
        const int ndrain = (p.num_kb + p.kpd - 1) / p.kpd;
        const int NGRP = p.ngroups;
        int grp = 0;
        uint32_t gph = 0;
        // softmax statistics: at every tile end a warp reduce-scatter turns this
        // warp's (tile x NC columns) values into one (m, s) per column, merged into
        // a running pair held by the lanes owning that column (2 registers).
        constexpr int NCP = NC <= 8 ? 8 : (NC <= 16 ? 16 : 32);
        float run_m = -INFINITY, run_s = 0.f;
        for (int t = 0; t < ntiles; ++t) {
            double acc[NC];
#pragma unroll
            for (int j = 0; j < NC; ++j) acc[j] = 0.0;
            if (NGRP > 0) {
                for (int kg = 0; kg < nkg; ++kg) {   // one group = the GK partials of a ring stage
                    const int ng = min(GK, p.num_kb - kg * GK);
                    mbar_wait(&pfull[grp], gph);
                    tc_fence_after();
                    // the stage's k-block partials (each restarted: no RZ bias) are summed
                    // in fp32 round-to-nearest (unbiased, ~1e-8 |l|), then once in fp64
                    float ssum[NC];
#pragma unroll
                    for (int j = 0; j < NC; ++j) ssum[j] = 0.f;
                    for (int g = 0; g < (p.sacc ? 1 : ng); ++g) {
                        float v[NC];
                        ld_cols<NC>(lane_base + scol + (uint32_t)((p.sacc ? grp : grp * GK + g) * NPAD), v);
#pragma unroll
                        for (int j = 0; j < NC; ++j) ssum[j] += v[j];
                    }
#pragma unroll
                    for (int j = 0; j < NC; ++j) acc[j] += (double)ssum[j];
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&pempty[grp]);
                    if (++grp == NGRP) { grp = 0; gph ^= 1; }
                }
            } else {
                for (int dk = 0; dk < ndrain; ++dk) {   // drain one partial
                    mbar_wait(&pfull[buf], bph);
                    tc_fence_after();
                    float v[NC];
                    ld_cols<NC>(lane_base + scol + (uint32_t)(buf * NPAD), v);
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&pempty[buf]);
                    if (++buf == NB) { buf = 0; bph ^= 1; }
#pragma unroll
                    for (int j = 0; j < NC; ++j) acc[j] += (double)v[j];
                }
            }
            const bool valid = vr < min(kTileV, rows - t * kTileV);
            const int xl = r0 + t * kTileV + vr;
            if (p.inv_t != 1.0) {   // temperature: the target distribution is softmax(l / T)
#pragma unroll
                for (int j = 0; j < NC; ++j) acc[j] *= p.inv_t;
            }
            float f[NC];
#pragma unroll
            for (int j = 0; j < NC; ++j) f[j] = (float)acc[j];
            if (valid) {
#pragma unroll
                for (int j = 0; j < NC; ++j) {
                    const int col = e * NC + j;
                    if (col < N && ctok[col] == xl) p.dl[cg[col]] = acc[j];   // fp64 draft logit
                }
            }
            st_cols<NC>(lane_base + (uint32_t)(t * NPAD), f);
            float tm[NCP], ts[NCP];
#pragma unroll
            for (int j = 0; j < NCP; ++j) {
                const bool ok = valid && j < NC;
                tm[j] = ok ? f[j < NC ? j : 0] : -INFINITY;
                ts[j] = ok ? 1.f : 0.f;
            }
            float wm, ws;
            warp_scatter_ms<NCP>(tm, ts, wm, ws);
            ms_merge(run_m, run_s, wm, ws);
        }
        {
            const int c = col_of_lane<NCP>(lane);
            // the lowest lane holding column c writes it
            if (c < NC && lane == (lane & ~((32 / NCP) - 1)) && ((lane & ((32 / NCP) - 1)) == 0 || NCP == 32))
                red[q * NPAD + e * NC + c] = make_float2(run_m, run_s);
        }
        named_bar(2, 256);
        const int et = threadIdx.x - 128;
        if (et < N) {
            float mj = -INFINITY, sj = 0.f;
#pragma unroll
            for (int w = 0; w < 4; ++w) ms_merge(mj, sj, red[w * NPAD + et].x, red[w * NPAD + et].y);
            p.part_m[(int64_t)et * grid + cta] = mj;
            p.part_s[(int64_t)et * grid + cta] = sj;
        }
    }
    __syncthreads();   // phase 1 done: the TMA ring is idle from here on
    NJ_STAMP(1);
    // The idle ring becomes scratch for the latency-bound phases (every global
    // read below is one cooperative sweep, so each phase pays ~one memory
    // latency instead of one per request).
    const int rows_cap = p.rows_cap;                                      // max rows per CTA
    float* qsl = reinterpret_cast<float*>(smem);                          // [G or nq][rows_cap] (3-4)
    grid_barrier(p.bar, grid);
    tc_fence_after();
    NJ_STAMP(2);

    // =============================================================== phase 2
    // (a) lse_j = M + log(sum_c s_c e^{m_c - M}): 8 lanes per row, all rows at
    //     once, partials read straight from L2 (L1 was invalidated by the barrier)
    // the acceptance test's fp64 draft logit rides on the same memory round trip
    const double dlv = ((int)threadIdx.x < N && cg[threadIdx.x] >= 0) ? p.dl[cg[threadIdx.x]] : 0.0;
    {   // N <= 48 = kFusedThreads / 8 row groups: one pass
        const int j = warp * 4 + (lane >> 3);
        const int sub = lane & 7;
        const bool act = j < N;
        constexpr int kPer = 20;   // grid <= 160: every lane's partials in registers, loads issued together
        float mv[kPer], sv[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int c = sub + 8 * k;
            const bool ok = act && c < grid;
            mv[k] = ok ? p.part_m[(int64_t)j * grid + c] : -INFINITY;
            sv[k] = ok ? p.part_s[(int64_t)j * grid + c] : 0.f;
        }
    if (p.q_prefetch) {
        // every draft row's q slice [r0, r0+rows) -> smem, fire-and-forget; it lands
        // while this CTA runs phase 2 (issued after the barrier: its fence would wait on it).
        // Issued by the warps the lse merge leaves idle (rows j = 4 warp + lane / 8 >= N),
        // in parallel with the merge; by every thread when all warps merge (N > 44).
        const int G = p.G;
        const int w0 = (N + 3) / 4;                       // first warp without lse rows
        const int nw = kFusedThreads / 32 - w0;
        const bool split = nw > 0;
        const int t0 = split ? (int)threadIdx.x - w0 * 32 : (int)threadIdx.x;
        const int nt = split ? nw * 32 : kFusedThreads;
        if (t0 >= 0) {
            if (p.q_vec16) {
                const int n4 = (rows + 3) >> 2;
                for (int i = t0; i < G * n4; i += nt) {
                    const int g = i / n4, x = (i - g * n4) * 4;
                    cp_async16(qsl + (size_t)g * rows_cap + x, p.q + (int64_t)g * p.ldq + p.v_begin + r0 + x);
                }
            } else {
                for (int i = t0; i < G * rows; i += nt) {
                    const int g = i / rows, x = i - g * rows;
                    cp_async4(qsl + (size_t)g * rows_cap + x, p.q + (int64_t)g * p.ldq + p.v_begin + r0 + x);
                }
            }
        }
        cp_async_commit();
    }
        NJ_STAMP(3);
        float mx = -INFINITY;
#pragma unroll
        for (int k = 0; k < kPer; ++k) mx = fmaxf(mx, mv[k]);
#pragma unroll
        for (int o = 4; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        double sacc = 0.0;
#pragma unroll
        for (int k = 0; k < kPer; ++k)
            if (mv[k] != -INFINITY) sacc += (double)sv[k] * (double)__expf(mv[k] - mx);
#pragma unroll
        for (int o = 4; o; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
        if (act && sub == 0) {
            lse_s[j] = (double)mx + log(sacc);
            if (cta == 0 && p.dbg_lse) p.dbg_lse[j] = (float)lse_s[j];
        }
    }
    __syncthreads();
    NJ_STAMP(4);
    // (b) every drafted token tested in parallel (Leviathan, R2: accept iff u*q < p)
    for (int j = threadIdx.x; j < N; j += kFusedThreads) {   // N <= 48 < threads: j == jd
        int res = 1;   // 1 accept, 0 reject, | 2 near-tie (certificate)
        const int g = cg[j];
        if (g >= 0) {
            const double pd = exp(dlv - lse_s[j]);
            const double uq = (double)u_sm[j] * (double)qx_sm[j];
            res = (uq < pd) ? 1 : 0;
            if (fabs(uq - pd) <= (double)p.eps_acc * pd) res |= 2;
            if (cta == 0 && p.dbg_pdraft) p.dbg_pdraft[g] = (float)pd;
        }
        dpass[j] = res;
    }
    __syncthreads();
    // (c) first rejection per request; q-slice slots for rejected requests
    if (threadIdx.x < 32) {
        int base = 0;
        for (int b0 = 0; b0 < B; b0 += 32) {
            const int b = b0 + lane;
            int is_rej = 0;
            ReqInfo r;
            if (b < B) {
                const int ro = p.row_off[b];
                const int gam = p.row_off[b + 1] - ro - 1;
                int n = gam, flag = 0;
                for (int i = 0; i < gam; ++i) {
                    const int res = dpass[ro + i];
                    if (res & 2) flag = 1;
                    if (!(res & 1)) { n = i; break; }
                }
                r.n = n; r.gam = gam; r.srow = ro + n; r.qrow = ro - b + n; r.resid = n < gam;
                r.flag = flag; r.lse_s = lse_s[ro + n];
                req[b] = r;
                is_rej = r.resid;
                if (cta == 0 && p.certify && (flag || p.force_fallback))
                    push_fallback(p.fb_count, p.fb_list, p.req_flags, b, 0);
            }
            const unsigned m = __ballot_sync(0xffffffffu, is_rej);
            if (b < B) qslot[b] = is_rej ? base + __popc(m & ((1u << lane) - 1u)) : -1;
            base += __popc(m);
        }
    }
    __syncthreads();
    NJ_STAMP(5);
    // (d) the rejected requests' q slices [r0, r0+rows) -> smem (unless prefetched):
    //     every slice's async copies in flight at once (q may be host memory read
    //     in place, where a load-store loop would pay one link latency per request)
    if (!p.q_prefetch) {
        for (int b = 0; b < B; ++b) {
            const int s = qslot[b];
            if (s < 0) continue;
            const float* src = p.q + (int64_t)req[b].qrow * p.ldq + p.v_begin + r0;
            float* dst = qsl + (size_t)s * rows_cap;
            if (p.q_vec16) {
                const int n4 = (rows + 3) >> 2;
                for (int i = threadIdx.x; i < n4; i += kFusedThreads) cp_async16(dst + 4 * i, src + 4 * i);
            } else {
                for (int x = threadIdx.x; x < rows; x += kFusedThreads) cp_async4(dst + x, src + x);
            }
        }
        cp_async_commit();
    }
    cp_async_wait_all();
    __syncthreads();
    NJ_STAMP(6);

    // =============================================================== phase 3
    // this CTA's residual max(0, p_n - q_n) / bonus p_gamma mass of every
    // request, straight from TMEM: all 12 warps (3 sets x 4 lane quadrants) split
    // the requests; per lane a sequential sum over its tiles, then one warp sum.
    {
        const int q = warp & 3;
        const int set = warp >> 2;
        const uint32_t lane_base = tbase + ((uint32_t)(q * 32) << 16);
        const int vr = q * 32 + lane;
        for (int b = set; b < B; b += kFusedThreads / 128) {
            const ReqInfo r = req[b];
            const float* qrow = !r.resid ? nullptr
                                : qsl + (size_t)(p.q_prefetch ? r.qrow : qslot[b]) * rows_cap;
            const float c = (float)r.lse_s;
            const float corr = (float)exp((double)c - r.lse_s);
            uint32_t a[kMaxT];
#pragma unroll
            for (int t = 0; t < kMaxT; ++t)
                a[t] = lane_base + (uint32_t)((t < ntiles ? t : 0) * NPAD + r.srow);
            float lv[kMaxT];
            tmem_ld1x16(a, lv);
            float s = 0.f;
#pragma unroll
            for (int t = 0; t < kMaxT; ++t) {
                const bool valid = t < ntiles && vr < min(kTileV, rows - t * kTileV);
                s += sample_weight(lv[t], c, corr, r.resid, qrow, t * kTileV + vr, valid);
            }
            s = warp_sum(s);
            if (lane == 0) wtile[b * 4 + q] = s;
        }
    }
    __syncthreads();
    NJ_STAMP(7);
    for (int b = threadIdx.x; b < B; b += kFusedThreads) {   // CTA mass, fixed fp64 order
        const float* wq = &wtile[b * 4];
        p.wpart[(int64_t)b * grid + cta] = (((double)wq[0] + (double)wq[1]) + (double)wq[2]) + (double)wq[3];
    }
    NJ_STAMP(8);
    grid_barrier(p.bar, grid);
    tc_fence_after();
    NJ_STAMP(9);

    // =============================================================== phase 4
    if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // warp per request: each lane sums a contiguous run of CTA masses, an inclusive
    // warp scan of the run totals gives every CTA's interval [E_c, I_c) with
    // E_c = I_{c-1} taken from the same values, so the intervals tile [0, W)
    // exactly and every CTA computes bit-identical bounds.
    for (int b = warp; b < B; b += kFusedThreads / 32) {
        const ReqInfo r = req[b];
        const int per = (grid + 31) / 32;
        const int c0 = lane * per, c1 = min(grid, c0 + per);
        double wv[8];
        double run = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            wv[k] = (k < per && c0 + k < c1) ? p.wpart[(int64_t)b * grid + c0 + k] : 0.0;
            if (k < per && c0 + k < c1) run = run + wv[k];
        }
        const double incl = warp_incl_scan_d(run);
        const double W = __shfl_sync(0xffffffffu, incl, 31);
        double base = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) base = 0.0;
        double Ec = 0.0, Ic = 0.0;
        int last_pos = -1;
        {
            double acc = base;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int c = c0 + k;
                if (k < per && c < c1) {
                    const double nx = (c == c1 - 1) ? incl : acc + wv[k];   // run end = scan value
                    if (c == cta) { Ec = acc; Ic = nx; }
                    if (wv[k] > 0.0) last_pos = c;
                    acc = nx;
                }
            }
        }
        int lp = last_pos;
#pragma unroll
        for (int o = 16; o; o >>= 1) lp = max(lp, __shfl_xor_sync(0xffffffffu, lp, o));
        const int src = min(cta / max(per, 1), 31);
        Ec = __shfl_sync(0xffffffffu, Ec, src);
        Ic = __shfl_sync(0xffffffffu, Ic, src);
        if (lane == 0) {
            const double T = (double)u_sm[p.row_off[b] + r.gam] * W;   // final-draw slot (R3)
            int own = 0;
            double tp = T - Ec;
            if (W > 0.0) {
                if (T >= W) own = (cta == lp) ? 2 : 0;   // rounding overshoot (R5): clamp
                else if (Ec <= T && T < Ic) own = 1;
            } else if (cta == 0) {   // zero residual mass (R6): the fp64 fallback (always
                p.accept_len[b] = r.n;   // launched) draws from p_n, certified or not
                p.next_token[b] = 0;
                if (p.dbg_mass) p.dbg_mass[b] = 0.0;
                if (p.dbg_flags) p.dbg_flags[b] = 2;
                push_fallback(p.fb_count, p.fb_list, p.req_flags, b, 2);
            }
            owner[b] = own;
            tprime[b] = tp;
            if (own && p.dbg_mass) p.dbg_mass[b] = W;
        }
    }
    __syncthreads();
    NJ_STAMP(11);
    // owner CTA: per-tile inclusive scans of its weights (tile-major = vocab
    // order), fixed-order tile prefix, then the token whose interval [E, I)
    // holds tp; E(x) = I(x-1) from the same scan values.  If rounding puts tp
    // past this CTA's recomputed total the draw is clamped and certified.
    if (warp >= 4 && warp < 8) {
        const int q = warp & 3;
        const int et = threadIdx.x - 128;
        const uint32_t lane_base = tbase + ((uint32_t)(q * 32) << 16);
        const int vr = q * 32 + lane;
        for (int b = 0; b < B; ++b) {
            const int own = owner[b];
            if (!own) continue;
            const ReqInfo r = req[b];
            const double tp = tprime[b];
            const float* qrow = !r.resid ? nullptr
                                : qsl + (size_t)(p.q_prefetch ? r.qrow : qslot[b]) * rows_cap;
            const float c = (float)r.lse_s;
            const float corr = (float)exp((double)c - r.lse_s);
            uint32_t a[kMaxT];
#pragma unroll
            for (int t = 0; t < kMaxT; ++t)
                a[t] = lane_base + (uint32_t)((t < ntiles ? t : 0) * NPAD + r.srow);
            float lv[kMaxT], w[kMaxT], inc[kMaxT];
            tmem_ld1x16(a, lv);
#pragma unroll
            for (int t = 0; t < kMaxT; ++t) {
                const bool valid = t < ntiles && vr < min(kTileV, rows - t * kTileV);
                w[t] = sample_weight(lv[t], c, corr, r.resid, qrow, t * kTileV + vr, valid);
                inc[t] = w[t];
            }
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
                for (int t = 0; t < kMaxT; ++t) {
                    const float y = __shfl_up_sync(0xffffffffu, inc[t], o);
                    if (lane >= o) inc[t] += y;
                }
            }
            float* wt = &wtile[B * 4];   // [kMaxT][4] quadrant totals (after the phase-3 area)
            if (lane == 31) {
#pragma unroll
                for (int t = 0; t < kMaxT; ++t)
                    if (t < ntiles) wt[t * 4 + q] = inc[t];
            }
            named_bar(1, 128);
            double* cp = &cprefix[0];
            if (et == 0) {
                double acc = 0.0;
                for (int t = 0; t < ntiles; ++t) {
                    cp[t] = acc;
                    acc = acc + ((((double)wt[t * 4] + (double)wt[t * 4 + 1]) + (double)wt[t * 4 + 2]) +
                                 (double)wt[t * 4 + 3]);
                }
                cp[ntiles] = acc;
            }
            named_bar(1, 128);
            int tsel = -1;
            bool clamp = (own == 2);
            if (!clamp)
                for (int t = 0; t < ntiles; ++t)
                    if (cp[t + 1] > tp) { tsel = t; break; }
            if (tsel < 0) {                // clamp: last tile with positive mass
                clamp = true;
                for (int t = ntiles - 1; t >= 0; --t)
                    if (cp[t + 1] > cp[t]) { tsel = t; break; }
            }
            float wsel = 0.f, isel = 0.f;
#pragma unroll
            for (int t = 0; t < kMaxT; ++t)
                if (t == tsel) { wsel = w[t]; isel = inc[t]; }
            float exc = __shfl_up_sync(0xffffffffu, isel, 1);
            if (lane == 0) exc = 0.f;
            double Sq = 0.0;
            for (int w2 = 0; w2 < q; ++w2) Sq = Sq + (double)wt[tsel * 4 + w2];
            const double lo = cp[tsel] + (Sq + (double)exc);   // E(x) = I(x-1)
            const double hi = cp[tsel] + (Sq + (double)isel);  // I(x)
            const int xl = r0 + tsel * kTileV + vr;
            if (clamp) {
                const unsigned mpos = __ballot_sync(0xffffffffu, wsel > 0.f);
                if (lane == 0) spick[q] = mpos ? (31 - __clz((int)mpos)) : -1;
                named_bar(1, 128);
                if (et == 0) {
                    int pick = -1;
                    for (int w2 = 3; w2 >= 0 && pick < 0; --w2)
                        if (spick[w2] >= 0) pick = w2 * 32 + spick[w2];
                    p.accept_len[b] = r.n;
                    p.next_token[b] = r0 + tsel * kTileV + (pick < 0 ? 0 : pick) + p.v_begin;
                    if (p.dbg_flags) p.dbg_flags[b] = 4;
                    if (p.certify) push_fallback(p.fb_count, p.fb_list, p.req_flags, b, 4);
                }
                named_bar(1, 128);
                continue;
            }
            if (wsel > 0.f && lo <= tp && tp < hi) {   // exactly one lane of the CTA
                p.accept_len[b] = r.n;
                p.next_token[b] = xl + p.v_begin;
                if (p.dbg_flags) p.dbg_flags[b] = 0;
                const double margin = fmin(tp - lo, hi - tp);
                if (p.certify && (margin <= (double)p.eps_draw || r.flag || p.force_fallback))
                    push_fallback(p.fb_count, p.fb_list, p.req_flags, b, 0);
            }
            named_bar(1, 128);   // wt / cp reused by the next owned request
        }
    }
    tc_fence_before();
    __syncthreads();
    NJ_STAMP(12);
    if (warp == 2) tmem_dealloc(tbase, 512);
}
