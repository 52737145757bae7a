// nj_fused.cuh — k_fused_verify<NPAD>: the whole verification step (BJ steps
// 1-3) in ONE persistent cooperative kernel for N <= 48 rows (memory-bound
// regime, BJ config 2).  Included from nj_gemm.cuh (namespace nj).
//
//   phase 1  GEMM over every row.  Accuracy: the MMA
//            accumulator is restarted every k-block (4 MMAs, K = 64) in a
//            scratch TMEM buffer and the epilogue sums the partials in fp64 —
//            tcgen05 truncates (RZ) on every fp32 accumulate, which over
//            K = 3584 biases logits by -3.3e-6*l; restarting cuts that 68x.
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
// Every decision whose margin is inside the certificate is queued for the fp64
// fallback (nj_sampler.cuh), which makes the output equal the fp64 definition.

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

constexpr int kFusedThreads = 384;   // warps 0-3 control, 4-11 epilogue (2 per TMEM lane quadrant)

// residual / bonus weight of one vocab entry (BJ step 3); the lse shift is
// taken in fp64 so no common-mode fp32 rounding of lse scales p against q.
__device__ __forceinline__ float sample_weight(float l, double lse, bool resid, const float* qrow, int xl,
                                               bool valid) {
    if (!valid) return 0.f;
    const float pe = __expf((float)((double)l - lse));
    return resid ? fmaxf(pe - __ldg(&qrow[xl]), 0.f) : pe;
}

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
    uint64_t* bars = reinterpret_cast<uint64_t*>(
        (reinterpret_cast<uintptr_t>(spick + 4) + 7) & ~uintptr_t(7));
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
    }
    if (cta == 0)
        for (int b = threadIdx.x; b < B; b += kFusedThreads) p.req_flags[b] = 0;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;

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
        for (int t = 0; t < ntiles; ++t) {
            for (int kg = 0; kg < nkg; ++kg) {
                const int ng = min(GK, p.num_kb - kg * GK);
                mbar_wait(&full[s], ph);
                for (int g = 0; g < ng; ++g) {
                    const int kb = kg * GK + g;
                    if (kin == 0) mbar_wait(&pempty[buf], bph ^ 1);
                    tc_fence_after();
                    const uint32_t dt = tbase + scol + (uint32_t)(buf * NPAD);
                    const size_t slot = (size_t)s * GK + g;
                    const uint64_t ad = sdesc_sw128(sA + slot * kTileBytesA);
                    const uint64_t bd = sdesc_sw128(sB + slot * kBBytes);
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k)
                        mma_bf16(dt, ad + 2 * k, bd + 2 * k, idesc, (kin | k) != 0);
                    if (++kin == kpd || kb + 1 == p.num_kb) {
                        mma_commit(&pfull[buf]);
                        kin = 0;
                        if (++buf == NB) { buf = 0; bph ^= 1; }
                    }
                }
                mma_commit(&empty[s]);
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
        for (int t = 0; t < ntiles; ++t) {
            double acc[NC];
#pragma unroll
            for (int j = 0; j < NC; ++j) acc[j] = 0.0;
            float accf[NC];
#pragma unroll
            for (int j = 0; j < NC; ++j) accf[j] = 0.f;
            for (int dk = 0; dk < ndrain; ++dk) {   // drain one partial
                mbar_wait(&pfull[buf], bph);
                tc_fence_after();
                float v[NC];
                ld_cols<NC>(lane_base + scol + (uint32_t)(buf * NPAD), v);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&pempty[buf]);
                if (++buf == NB) { buf = 0; bph ^= 1; }
                if (p.f32drain) {
#pragma unroll
                    for (int j = 0; j < NC; ++j) accf[j] += v[j];
                } else {
#pragma unroll
                    for (int j = 0; j < NC; ++j) acc[j] += (double)v[j];
                }
            }
            if (p.f32drain) {
#pragma unroll
                for (int j = 0; j < NC; ++j) acc[j] = (double)accf[j];
            }
            const bool valid = vr < min(kTileV, rows - t * kTileV);
            const int xl = r0 + t * kTileV + vr;
            if (valid) {
#pragma unroll
                for (int j = 0; j < NC; ++j) {
                    const int col = e * NC + j;
                    if (col < N && ctok[col] == xl) p.dl[cg[col]] = acc[j];   // fp64 draft logit
                }
            }
            float f[NC];
#pragma unroll
            for (int j = 0; j < NC; ++j) f[j] = (float)acc[j];
            st_cols<NC>(lane_base + (uint32_t)(t * NPAD), f);
        }
        // softmax statistics of this thread's vocab lanes from the stored logits
        // (tcgen05.ld is warp-collective: every lane loads, invalid lanes are masked after)
        float m[NC], sm[NC];
#pragma unroll
        for (int j = 0; j < NC; ++j) { m[j] = -INFINITY; sm[j] = 0.f; }
        for (int t = 0; t < ntiles; ++t) {
            float v[NC];
            ld_cols<NC>(lane_base + (uint32_t)(t * NPAD), v);
            if (vr < min(kTileV, rows - t * kTileV)) {
#pragma unroll
                for (int j = 0; j < NC; ++j) m[j] = fmaxf(m[j], v[j]);
            }
        }
        for (int t = 0; t < ntiles; ++t) {
            float v[NC];
            ld_cols<NC>(lane_base + (uint32_t)(t * NPAD), v);
            if (vr < min(kTileV, rows - t * kTileV)) {
#pragma unroll
                for (int j = 0; j < NC; ++j) sm[j] += __expf(v[j] - m[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < NC; ++j) {
            float mj = m[j], sj = sm[j];
            warp_ms_merge(mj, sj);
            if (lane == 0) red[q * NPAD + e * NC + j] = make_float2(mj, sj);
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
    grid_barrier(p.bar_count, p.bar_gen, grid);
    tc_fence_after();

    // =============================================================== phase 2
    for (int j = warp; j < N; j += kFusedThreads / 32) {   // lse_j, warp per row
        float mx = -INFINITY;
        for (int c = lane; c < grid; c += 32) mx = fmaxf(mx, __ldcg(&p.part_m[(int64_t)j * grid + c]));
        mx = warp_max(mx);
        double sacc = 0.0;
        for (int c = lane; c < grid; c += 32) {
            const float mc = __ldcg(&p.part_m[(int64_t)j * grid + c]);
            const float sc = __ldcg(&p.part_s[(int64_t)j * grid + c]);
            if (mc != -INFINITY) sacc += (double)sc * (double)__expf(mc - mx);
        }
        sacc = warp_sum_d(sacc);
        if (lane == 0) {
            lse_s[j] = (double)mx + log(sacc);
            if (cta == 0 && p.dbg_lse) p.dbg_lse[j] = (float)lse_s[j];
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < B; b += kFusedThreads) {   // Leviathan acceptance (R2: u*q < p)
        const int ro = p.row_off[b];
        const int gam = p.row_off[b + 1] - ro - 1;
        const int g0 = ro - b;
        int n = gam, flag = 0;
        for (int i = 0; i < gam; ++i) {
            const int g = g0 + i;
            const double pd = exp(__ldcg(&p.dl[g]) - lse_s[ro + i]);
            const double qx = (double)p.q[(int64_t)g * p.ldq + p.draft_tokens[g]];
            const double uq = (double)p.u[ro + i] * qx;
            if (cta == 0 && p.dbg_pdraft) p.dbg_pdraft[g] = (float)pd;
            if (fabs(uq - pd) <= (double)p.eps_acc * pd) flag = 1;
            if (!(uq < pd)) { n = i; break; }
        }
        if (cta == 0 && p.dbg_pdraft)   // untested drafts still report p_i(x_i)
            for (int i = n + 1; i < gam; ++i)
                p.dbg_pdraft[g0 + i] = (float)exp(__ldcg(&p.dl[g0 + i]) - lse_s[ro + i]);
        ReqInfo r;
        r.n = n; r.gam = gam; r.srow = ro + n; r.qrow = g0 + n; r.resid = n < gam;
        r.flag = flag; r.lse_s = lse_s[ro + n];
        req[b] = r;
        if (cta == 0 && p.certify && (flag || p.force_fallback))
            push_fallback(p.fb_count, p.fb_list, p.req_flags, b, 0);
    }
    __syncthreads();

    // =============================================================== phase 3
    if (warp >= 4 && warp < 8) {
        const int q = warp & 3;
        const uint32_t lane_base = tbase + ((uint32_t)(q * 32) << 16);
        const int vr = q * 32 + lane;
        for (int b = 0; b < B; ++b) {
            const ReqInfo r = req[b];
            const float* qrow = p.q + (int64_t)r.qrow * p.ldq + p.v_begin;
            uint32_t a[kMaxT];
#pragma unroll
            for (int t = 0; t < kMaxT; ++t)
                a[t] = lane_base + (uint32_t)((t < ntiles ? t : 0) * NPAD + r.srow);
            float lv[kMaxT];
            tmem_ld1x16(a, lv);
#pragma unroll
            for (int t = 0; t < kMaxT; ++t) {
                if (t < ntiles) {
                    const bool valid = vr < min(kTileV, rows - t * kTileV);
                    const float w = sample_weight(lv[t], r.lse_s, r.resid, qrow, r0 + t * kTileV + vr, valid);
                    const float inc = warp_incl_scan(w);
                    if (lane == 31) wtile[(b * kMaxT + t) * 4 + q] = inc;
                }
            }
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < B; b += kFusedThreads) {   // CTA mass, fixed fp64 order
        double acc = 0.0;
        for (int t = 0; t < ntiles; ++t) {
            cprefix[b * (kMaxT + 1) + t] = acc;
            const float* wt = &wtile[(b * kMaxT + t) * 4];
            acc = acc + ((((double)wt[0] + (double)wt[1]) + (double)wt[2]) + (double)wt[3]);
        }
        cprefix[b * (kMaxT + 1) + ntiles] = acc;
        p.wpart[(int64_t)b * grid + cta] = acc;
    }
    grid_barrier(p.bar_count, p.bar_gen, grid);
    tc_fence_after();

    // =============================================================== phase 4
    for (int b = threadIdx.x; b < B; b += kFusedThreads) {
        const ReqInfo r = req[b];
        double P = 0.0, Pc = 0.0, mine = 0.0;
        int last_pos = -1;
        for (int c = 0; c < grid; ++c) {   // P_{c+1} = P_c + wpart_c, c ascending
            const double wc = __ldcg(&p.wpart[(int64_t)b * grid + c]);
            if (c == cta) { Pc = P; mine = wc; }
            if (wc > 0.0) last_pos = c;
            P = P + wc;
        }
        const double W = P;
        const double T = (double)p.u[p.row_off[b] + r.gam] * W;   // final-draw slot (R3)
        int own = 0;
        double tp = T - Pc;
        if (W > 0.0) {
            if (T >= W) {                  // rounding overshoot (R5): clamp in the last positive CTA
                own = (cta == last_pos) ? 2 : 0;
            } else if (Pc <= T && T < Pc + mine) {
                own = 1;
            }
        } else if (cta == 0) {             // zero residual mass (R6): the fp64 fallback draws from p_n
            p.accept_len[b] = r.n;
            p.next_token[b] = 0;
            if (p.dbg_mass) p.dbg_mass[b] = 0.0;
            if (p.dbg_flags) p.dbg_flags[b] = 2;
            if (p.certify) push_fallback(p.fb_count, p.fb_list, p.req_flags, b, 2);
        }
        owner[b] = own;
        tprime[b] = tp;
        if (own && p.dbg_mass) p.dbg_mass[b] = W;
    }
    __syncthreads();
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
            const double* cp = &cprefix[b * (kMaxT + 1)];
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
            const float l = tmem_ld1(lane_base + (uint32_t)(tsel * NPAD + r.srow));
            const bool valid = vr < min(kTileV, rows - tsel * kTileV);
            const int xl = r0 + tsel * kTileV + vr;
            const float w = sample_weight(l, r.lse_s, r.resid,
                                          p.q + (int64_t)r.qrow * p.ldq + p.v_begin, xl, valid);
            const float inc = warp_incl_scan(w);
            float exc = __shfl_up_sync(0xffffffffu, inc, 1);
            if (lane == 0) exc = 0.f;
            const float* wt = &wtile[(b * kMaxT + tsel) * 4];
            double Sq = 0.0;
            for (int w2 = 0; w2 < q; ++w2) Sq = Sq + (double)wt[w2];
            const double lo = cp[tsel] + (Sq + (double)exc);   // E(x) = I(x-1)
            const double hi = cp[tsel] + (Sq + (double)inc);   // I(x)
            if (clamp) {
                const unsigned mpos = __ballot_sync(0xffffffffu, w > 0.f);
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
            if (w > 0.f && lo <= tp && tp < hi) {   // exactly one lane of the CTA
                p.accept_len[b] = r.n;
                p.next_token[b] = xl + p.v_begin;
                if (p.dbg_flags) p.dbg_flags[b] = 0;
                const double margin = fmin(tp - lo, hi - tp);
                if (p.certify && (margin <= (double)p.eps_draw || r.flag || p.force_fallback))
                    push_fallback(p.fb_count, p.fb_list, p.req_flags, b, 0);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_dealloc(tbase, 512);
}
