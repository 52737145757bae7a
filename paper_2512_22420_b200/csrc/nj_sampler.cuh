// nj_sampler.cuh — acceptance / residual-resampling kernels of the two-pass
// path, and the fp64 certified fallback shared by both paths.
//
// BJ step (3) (Leviathan): accept draft i iff u_i q_i(x_i) <
// p_i(x_i) (R2), first rejection n, resample from norm(max(0, p_n - q_n)),
// bonus from p_gamma on full acceptance, inverse CDF in ascending token id (R5).
//
// Sampler arithmetic is bandwidth-bound: rows are streamed with coalesced
// loads (consecutive threads = consecutive vocab ids), masses are built from
// warp inclusive scans with fp64 cross-warp / cross-chunk prefixes, and the
// located token's interval boundaries are taken from the SAME fp32 scan values
// (E(x) = I(x-1)) so the intervals tile [0, W) exactly.
#pragma once
#include "nj_gemm.cuh"

namespace nj {

struct ReqMeta {
    int32_t B;
    int32_t row_off[kMaxB + 1];
};

__device__ __forceinline__ int req_of_row(const ReqMeta& m, int j) {
    int lo = 0, hi = m.B - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (m.row_off[mid] <= j) lo = mid; else hi = mid - 1;
    }
    return lo;
}
__device__ __forceinline__ int req_of_draft(const ReqMeta& m, int g) {   // draft_off[b] = row_off[b] - b
    int lo = 0, hi = m.B - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (m.row_off[mid] - mid <= g) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// copy one bf16 row of d elements (d % 8 == 0) with 16-B vector loads
__device__ __forceinline__ void copy_row(uint16_t* dst, const uint16_t* src, int d, int t, int nt) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (int i = t; i < d / 8; i += nt) d4[i] = __ldg(&s4[i]);
}

// gather the draft rows of hidden into a contiguous [G, d] buffer (block per row)
// Programmatic dependent launch: every sampler kernel first waits for its
// predecessor grid (a no-op unless launched with the PDL attribute), then lets
// its own successor be scheduled, which waits in turn -- so each launch's ramp
// overlaps the previous kernel instead of following its drain.  The wait comes
// before any global access in EVERY CTA, so a grid never completes before its
// predecessor (the chain stays transitive).
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__global__ void k_gather_drafts(const uint16_t* __restrict__ hidden, int d, const ReqMeta m,
                                uint16_t* __restrict__ out) {
    const int g = blockIdx.x;
    const int b = req_of_draft(m, g);
    const int row = m.row_off[b] + (g - (m.row_off[b] - b));
    copy_row(out + (int64_t)g * d, hidden + (int64_t)row * d, d, threadIdx.x, blockDim.x);
}

// gather rows by a device row list (test-only GEMM probe)
__global__ void k_gather_rows(const uint16_t* __restrict__ hidden, int d, const int32_t* __restrict__ rows,
                              uint16_t* __restrict__ out) {
    copy_row(out + (int64_t)blockIdx.x * d, hidden + (int64_t)rows[blockIdx.x] * d, d, threadIdx.x, blockDim.x);
}

__global__ void k_iota(int32_t* out, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = i;
}

// lse of row j from per-CTA partials (warp-cooperative, fixed order)
__device__ __forceinline__ double warp_lse(const float* pm, const float* ps, int ld, int j, int grid) {
    const int lane = (int)lane_id();
    float mx = -INFINITY;
    for (int c = lane; c < grid; c += 32) mx = fmaxf(mx, __ldcg(&pm[(int64_t)j * ld + c]));
    mx = warp_max(mx);
    double sacc = 0.0;
    for (int c = lane; c < grid; c += 32) {
        const float mc = __ldcg(&pm[(int64_t)j * ld + c]);
        const float sc = __ldcg(&ps[(int64_t)j * ld + c]);
        if (mc != -INFINITY) sacc += (double)sc * (double)__expf(mc - mx);
    }
    sacc = warp_sum_d(sacc);
    return (double)mx + log(sacc);
}

struct AcceptParams {
    const float* part_m;   // [G][grid] stats of draft rows (K-A)
    const float* part_s;
    int32_t grid;          // CTAs that wrote partials
    int32_t pld;           // partial row stride (>= grid)
    const double* dl;      // [G] draft logits
    const int32_t* draft_tokens;
    const float* q;
    int64_t ldq;
    const float* u;
    const uint16_t* hidden;
    int32_t d;
    uint16_t* hs;          // [B, d] gathered sample rows
    int32_t* accept_len;
    int32_t* s_resid;      // [B]
    int32_t* s_qrow;       // [B]
    double* s_lse;         // [B] lse of the sample row if residual (else NaN)
    int32_t* fb_count;
    int32_t* fb_list;
    int32_t* req_flags;
    float* dbg_lse;
    float* dbg_pdraft;
    int32_t certify, force_fallback;
    float eps_acc;
    // staged path: stats are per ROW (part index = row, not draft index), every
    // row's logits are staged, so no hidden-row copy; s_row[b] = sample row
    int32_t staged;
    int32_t* s_row;
    // vocab-sharded mode (nj_shard.cuh): merged X1 entries [nranks][xld][2]
    const double* xr1;
    int32_t nranks, xld;
    // lse of every partial row, precomputed by k_lse_rows (NULL: merge here)
    const double* pre_lse;
    int32_t lse_sample_from_c;
};

// lse of partial rows [0, n) from the per-CTA partials, one warp per row (all
// rows in parallel; k_accept then only reads them)
__global__ void k_lse_rows(const float* __restrict__ pm, const float* __restrict__ ps, int pld, int grid, int n,
                           double* __restrict__ out);

__device__ __forceinline__ double xmerge_lse(const double* xr, int nranks, int ld, int g, double& dl);

// K-B: warp per request — lse of its draft rows, acceptance tests, first
// rejection, sample-row bookkeeping, and the copy of the sample hidden row.
__global__ void k_accept(const AcceptParams p, const ReqMeta m) {
    pdl_enter();
    const int b = blockIdx.x * (blockDim.x / 32) + (int)warp_id();
    if (b >= m.B) return;
    const int lane = (int)lane_id();
    const int ro = m.row_off[b], gam = m.row_off[b + 1] - ro - 1, g0 = ro - b;
    int n = gam, flag = 0;
    double lse_n = __longlong_as_double(0x7ff8000000000000ll);
    for (int i = 0; i < gam; ++i) {
        const int g = g0 + i;
        double lse, dlv;
        if (p.xr1) lse = xmerge_lse(p.xr1, p.nranks, p.xld, g, dlv);
        else {
            const int pr = p.staged ? ro + i : g;
            lse = p.pre_lse ? __ldcg(&p.pre_lse[pr]) : warp_lse(p.part_m, p.part_s, p.pld, pr, p.grid);
            dlv = __ldcg(&p.dl[g]);
        }
        const double pd = exp(dlv - lse);
        const double qx = (double)p.q[(int64_t)g * p.ldq + p.draft_tokens[g]];
        const double uq = (double)p.u[ro + i] * qx;
        if (lane == 0) {
            if (p.dbg_lse) p.dbg_lse[ro + i] = (float)lse;
            if (p.dbg_pdraft) p.dbg_pdraft[g] = (float)pd;
        }
        if (fabs(uq - pd) <= (double)p.eps_acc * pd) flag = 1;
        if (!(uq < pd)) { n = i; lse_n = lse; break; }
    }
    // remaining drafts (untested) still get debug values
    for (int i = n + 1; i < gam && p.dbg_pdraft; ++i) {
        const int g = g0 + i;
        double lse, dlv;
        if (p.xr1) lse = xmerge_lse(p.xr1, p.nranks, p.xld, g, dlv);
        else {
            const int pr = p.staged ? ro + i : g;
            lse = p.pre_lse ? __ldcg(&p.pre_lse[pr]) : warp_lse(p.part_m, p.part_s, p.pld, pr, p.grid);
            dlv = __ldcg(&p.dl[g]);
        }
        if (lane == 0) {
            if (p.dbg_lse) p.dbg_lse[ro + i] = (float)lse;
            p.dbg_pdraft[g] = (float)exp(dlv - lse);
        }
    }
    if (p.staged) {
        if (n == gam)   // bonus row
            lse_n = p.pre_lse ? __ldcg(&p.pre_lse[ro + gam]) : warp_lse(p.part_m, p.part_s, p.pld, ro + gam, p.grid);
    } else {
        copy_row(p.hs + (int64_t)b * p.d, p.hidden + (int64_t)(ro + n) * p.d, p.d, lane, 32);
    }
    if (lane == 0) {
        if (p.staged) p.s_row[b] = ro + n;
        p.accept_len[b] = n;
        p.s_resid[b] = n < gam;
        p.s_qrow[b] = g0 + n;
        // lse_sample_from_c: the sample row's lse comes from K-C's own statistics
        // (the two-pass path's accurate sample-row GEMM), not from K-A's
        p.s_lse[b] = p.lse_sample_from_c ? __longlong_as_double(0x7ff8000000000000ll) : lse_n;
        if (p.certify && (flag || p.force_fallback)) push_fallback(p.fb_count, p.fb_list, p.req_flags, b, 0);
    }
}

__global__ void k_lse_rows(const float* __restrict__ pm, const float* __restrict__ ps, int pld, int grid, int n,
                           double* __restrict__ out) {
    pdl_enter();
    const int r = blockIdx.x * (blockDim.x / 32) + (int)warp_id();
    if (r >= n) return;
    const double l = warp_lse(pm, ps, pld, r, grid);
    if (lane_id() == 0) out[r] = l;
}

// lse of each request's logits row [B, ld] (stage-isolated sampler), fp64 merge
__global__ void k_row_lse(const float* __restrict__ logits, int64_t ld, int V, double* __restrict__ lse) {
    const int b = blockIdx.x;
    const float* row = logits + (int64_t)b * ld;
    float m = -INFINITY, s = 0.f;
    for (int x = threadIdx.x; x < V; x += blockDim.x) {
        const float v = row[x];
        const float d = v - m;
        const float e = __expf(-fabsf(d));
        if (d <= 0.f) s += e; else { s = s * e + 1.f; m = v; }
    }
    warp_ms_merge(m, s);
    __shared__ float2 red[32];
    if (lane_id() == 0) red[warp_id()] = make_float2(m, s);
    __syncthreads();
    if (threadIdx.x == 0) {
        float M = -INFINITY;
        for (int w = 0; w < (int)(blockDim.x / 32); ++w) M = fmaxf(M, red[w].x);
        double S = 0.0;
        for (int w = 0; w < (int)(blockDim.x / 32); ++w)
            if (red[w].x != -INFINITY) S += (double)red[w].y * (double)__expf(red[w].x - M);
        lse[b] = (double)M + log(S);
    }
}

constexpr int kSampThreads = 256;
constexpr int kSubTiles = 16;                         // chunk = 16 sub-tiles of 256
constexpr int kChunk = kSampThreads * kSubTiles;      // 4096 vocab ids per chunk

struct MassParams {
    const float* logits;   // [B][ld] local vocab (or [N][ld] with s_row)
    int64_t ld;
    const int32_t* s_row;  // staged path: logits row of request b (NULL: row b)
    int32_t V_local, v_begin, nchunks;
    const int32_t* s_resid;
    const int32_t* s_qrow;
    const double* s_lse;   // residual rows: lse from K-B; NaN -> merge part2 (bonus rows)
    const float* part2_m;  // [B][grid2] (K-C stats)
    const float* part2_s;
    int32_t grid2;
    int32_t pld2;          // part2 row stride (>= grid2)
    int32_t part2_by_row;  // 1: part2 row of request b is s_row[b] (vocab-sharded staged step)
    int32_t pf_rows;       // k_sample_small: L2-prefetch the candidate rows while testing
    int32_t small_pb;      // k_sample_small: chunks per staged batch
    int32_t pdl_trigger;   // k_sample_small: trigger the fallback kernel's launch at the start
    int32_t small_reuse;   // k_sample_small: the owner CTA reads the located chunk from its staging buffer
    // nj_verify_host with host-resident q: draft rows g with bit g set were staged into
    // q_loc (same pitch ldq) while the GEMM ran; the others are read in place (q)
    const float* q_loc;
    uint64_t q_loc_mask[4];
    // k_sample_small<FLAT = true>: CTAs per request (no cluster); chunk masses go through
    // global memory (cm_glob[b][nchunks]) and a per-request arrival barrier (cm_cnt[b],
    // zeroed before every call)
    int32_t flat_cpr;
    double* cm_glob;
    int32_t* cm_cnt;
    const float* q;
    int64_t ldq;
    const float* u;        // final-draw uniform of request b at u[row_off[b]+gamma_b] (or u[b] in stage mode)
    int32_t stage_mode;    // 1: u indexed by b
    double* cmass;         // [B][nchunks]
    int32_t* accept_len;
    int32_t* next_token;
    int32_t* fb_count;
    int32_t* fb_list;
    int32_t* req_flags;
    double* dbg_mass;
    int32_t* dbg_flags;
    float* dbg_lse;
    int32_t certify;
    float eps_draw;
    // vocab-sharded mode: X2 entries [nranks][B][2] (lse used, local mass);
    // next_token then points at the X3 buffer (-1 on non-owner ranks) and
    // flags go to xflags[b] (reduced by MAX, queued by k_xfinish)
    const double* xr2;
    int64_t xstride;       // doubles per rank in xr2 (entries of 3 per request)
    int32_t nranks, rank;
    int32_t* xflags;
    // nj_propose: k_mass writes each bonus row's weights exp(l - lse) over its
    // logits in place (the q rows), and k_locate then reads them as weights
    int32_t w_inplace;
    unsigned long long* ts;   // debug (NJ_PHASE_TS): k_sample_small phase stamps at [18432 + 16 CTA + k], CTA < 128
    int32_t probe;         // k_mass timing probes (NJ_MASS_PROBE; 0 in normal runs): 1 no copies, 2 no scans, 4 no totals
};

// Queue a draw for the fp64 fallback: certificate hits (certify on) and, always,
// zero residual mass (R6: the draw must come from p_n, which the fallback does;
// the fallback kernel is launched on every call).
__device__ __forceinline__ void flag_draw(const MassParams& p, int b, int32_t bits) {
    // sharded mode: informational flags only (exchanged in X3); the draw itself is
    // final -- the fp64 fallback there takes acceptance near-ties, decided before X2
    if (p.xflags) atomicOr(&p.xflags[b], bits);
    else if (p.certify || (bits & 2)) push_fallback(p.fb_count, p.fb_list, p.req_flags, b, bits);
}

__device__ __forceinline__ int part2_row(const MassParams& p, int b) { return p.part2_by_row ? p.s_row[b] : b; }
__device__ __forceinline__ double sample_lse(const MassParams& p, int b) {
    __shared__ double s_l;
    double l = p.s_lse[b];
    if (isnan(l)) {
        if (warp_id() == 0) {
            const double v = warp_lse(p.part2_m, p.part2_s, p.pld2, part2_row(p, b), p.grid2);
            if (lane_id() == 0) s_l = v;
        }
        __syncthreads();
        l = s_l;
    }
    return l;
}

// weights of sub-tile s of chunk c for this thread (one element per thread)
__device__ __forceinline__ const float* logits_row(const MassParams& p, int b) {
    return p.logits + (int64_t)(p.s_row ? p.s_row[b] : b) * p.ld;
}
// p(x) = exp(l(x) - lse) as exp(l - c) * corr with c = fp32(lse) and corr =
// exp(c - lse) formed once per request in fp64: the fp32 rounding of lse (up to
// ~1e-6 relative for |lse| ~ 15-25) would otherwise scale every p of the row
// against q in the residual max(0, p - q) (the fused kernel's sample_weight
// does the same).  __fmul_rn / __fsub_rn keep k_mass and k_locate bit-identical
// (no contraction into an FMA in one of them only).
__device__ __forceinline__ float p_weight(float l, float c, float corr) { return __fmul_rn(__expf(l - c), corr); }
__device__ __forceinline__ float resid_weight(float pe, float qv) { return fmaxf(__fsub_rn(pe, qv), 0.f); }
__device__ __forceinline__ float lse_corr(double lse) {
    const float c = (float)lse;
    return (float)exp((double)c - lse);
}

__device__ __forceinline__ float chunk_weight(const MassParams& p, const float* lrow, int c, int s, float lsef,
                                              float corr, bool resid, const float* qrow) {
    const int x = c * kChunk + s * kSampThreads + (int)threadIdx.x;
    if (x >= p.V_local) return 0.f;
    const float pe = p.w_inplace ? __ldcg(&lrow[x]) : p_weight(__ldcg(&lrow[x]), lsef, corr);
    return resid ? resid_weight(pe, __ldg(&qrow[x])) : pe;
}


// Sample-row lse of every request whose s_lse is NaN (bonus rows / the
// two-pass path's K-C statistics), merged once per request so that k_mass's
// items and k_locate read one value.  Warp per request.
__global__ void k_sample_lse(const MassParams p, int B, double* s_lse) {   // s_lse == p.s_lse
    pdl_enter();
    const int b = blockIdx.x * (blockDim.x / 32) + (int)warp_id();
    if (b >= B) return;
    if (!isnan(__ldcg(&p.s_lse[b]))) return;
    const double v = warp_lse(p.part2_m, p.part2_s, p.pld2, part2_row(p, b), p.grid2);
    if (lane_id() == 0) s_lse[b] = v;
}

// The 16 sub-tile warp totals of a thread's v[0..15] (destroyed) by a
// reduce-scatter over lane bits 0, 1, 2, 3 (each step halves the set a lane
// keeps) and a final xor-16 step: every total is the aligned binary tree over
// lanes 0..31, which is exactly the lane-31 value of warp_incl_scan (fp32
// addition is commutative; tests/test_reduction_order.py), in 16 shuffles
// instead of 16 scans' 80.  wt[s][warp] gets sub-tile s's total.
__device__ __forceinline__ void warp_totals16(float (&v)[kSubTiles], float (*wt)[8]) {
    const uint32_t lane = lane_id();
#pragma unroll
    for (int m = 1, n = kSubTiles / 2; m <= 8; m <<= 1, n >>= 1) {
        const bool hi = (lane & (uint32_t)m) != 0;
#pragma unroll
        for (int k = 0; k < n; ++k) {
            const float keep = hi ? v[k + n] : v[k];
            const float send = hi ? v[k] : v[k + n];
            v[k] = keep + __shfl_xor_sync(0xffffffffu, send, m);
        }
    }
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], 16);
    // lane bits (0, 1, 2, 3) chose halves (8, 4, 2, 1) of the sub-tile index
    const int s = ((lane & 1) << 3) | ((lane & 2) << 1) | ((lane & 4) >> 1) | ((lane & 8) >> 3);
    if (lane < 16) wt[s][warp_id()] = v[0];
}

// K-D1: chunk masses.  Items (request b, chunk c), request-major, are taken
// round-robin by a grid of num_sms x resident CTAs (every CTA sees a mix of
// residual items, which read logits + q, and bonus items, which read logits
// only).  Each CTA streams its items through a ring of NST shared-memory
// stages with cp.async (16-byte copies where the rows are 16-byte aligned),
// NST - 1 items in flight while it scans the current one, so the bytes in
// flight per SM do not depend on the register budget.  Needs s_lse non-NaN
// (k_sample_lse).  The per-item arithmetic (and so cmass) is the same
// expression and order as k_locate's recomputation.
__device__ __forceinline__ void mass_copy_chunk(float* dst, const float* src, int n) {
    if (n == kChunk && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
#pragma unroll
        for (int k = 0; k < kChunk / 4 / kSampThreads; ++k) {
            const int f = k * kSampThreads + (int)threadIdx.x;
            cp_async16(dst + 4 * f, src + 4 * f);
        }
    } else if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
        for (int f = threadIdx.x; 4 * f < n; f += kSampThreads) {
            if (4 * f + 4 <= n) cp_async16(dst + 4 * f, src + 4 * f);
            else
                for (int e = 4 * f; e < n; ++e) cp_async4(dst + e, src + e);
        }
    } else {
        for (int x = threadIdx.x; x < n; x += kSampThreads) cp_async4(dst + x, src + x);
    }
}

template <int NST>
__global__ void __launch_bounds__(kSampThreads) k_mass(const MassParams p, int B) {
    pdl_enter();
    extern __shared__ __align__(16) float ring[];   // NST x {logits[kChunk], q[kChunk]}, then the request table
    __shared__ float wt[kSubTiles][8];
    __shared__ double sst[kSubTiles];
    // per-request scalars staged once per CTA: the item loop then has no
    // dependent global load (each would cost a DRAM latency per item)
    int* t_qrow = reinterpret_cast<int*>(ring + (size_t)NST * 2 * kChunk);   // -1: bonus row (no q)
    float* t_lsef = reinterpret_cast<float*>(t_qrow + B);
    float* t_corr = t_lsef + B;
    for (int b = threadIdx.x; b < B; b += kSampThreads) {
        t_qrow[b] = p.s_resid[b] ? p.s_qrow[b] : -1;
        const double l = __ldcg(&p.s_lse[b]);
        t_lsef[b] = (float)l;
        t_corr[b] = lse_corr(l);
    }
    __syncthreads();
    const int total = B * p.nchunks;
    const int G = gridDim.x;
    auto issue = [&](int it, int slot) {
        if (it < total && !(p.probe & 1)) {
            const int b = it / p.nchunks, c = it - b * p.nchunks;
            const int x0 = c * kChunk, n = min(kChunk, p.V_local - x0);
            float* d = ring + (size_t)slot * 2 * kChunk;
            mass_copy_chunk(d, logits_row(p, b) + x0, n);
            const int qr = t_qrow[b];
            if (qr >= 0) mass_copy_chunk(d + kChunk, p.q + (int64_t)qr * p.ldq + p.v_begin + x0, n);
        }
        cp_async_commit();
    };
#pragma unroll
    for (int s = 0; s < NST - 1; ++s) issue(blockIdx.x + s * G, s);
    int j = 0;
    for (int it = blockIdx.x; it < total; it += G, ++j) {
        cp_async_wait<NST - 2>();
        __syncthreads();   // item j's stage is visible; stage (j - 1) % NST is free
        issue(it + (NST - 1) * G, (j + NST - 1) % NST);
        const int b = it / p.nchunks, c = it - b * p.nchunks;
        const int slot = j % NST;
        const bool resid = t_qrow[b] >= 0;
        const float lsef = t_lsef[b], corr = t_corr[b];
        const float* sl = ring + (size_t)slot * 2 * kChunk;
        const float* sq = sl + kChunk;
        const int x0 = c * kChunk + (int)threadIdx.x;
        float v[kSubTiles];
        if (x0 - (int)threadIdx.x + kChunk <= p.V_local) {   // whole chunk in range
#pragma unroll
            for (int s = 0; s < kSubTiles; ++s) {
                const int o = s * kSampThreads + (int)threadIdx.x;
                const float e = p_weight(sl[o], lsef, corr);
                v[s] = resid ? resid_weight(e, sq[o]) : e;
            }
        } else {
#pragma unroll
            for (int s = 0; s < kSubTiles; ++s) {
                const int o = s * kSampThreads + (int)threadIdx.x;
                const bool in = x0 + s * kSampThreads < p.V_local;
                const float e = in ? p_weight(sl[o], lsef, corr) : 0.f;
                v[s] = resid ? resid_weight(e, in ? sq[o] : 0.f) : e;
            }
        }
        if (p.w_inplace && !resid) {   // nj_propose: q = the draw's weights, over the logits
            float* wrow = const_cast<float*>(logits_row(p, b)) + c * kChunk;
#pragma unroll
            for (int s = 0; s < kSubTiles; ++s) {
                const int o = s * kSampThreads + (int)threadIdx.x;
                if (x0 + s * kSampThreads < p.V_local) wrow[o] = v[s];
            }
        }
        if (!(p.probe & 2)) {
            warp_totals16(v, wt);
        } else if (v[0] == 1234.5f) {
            wt[0][0] = v[1];
        }
        if (p.probe & 4) continue;
        __syncthreads();
        // sub-tile totals in parallel (same left-to-right fp64 order as k_locate),
        // then the chunk total over the 16 sub-tiles
        if (threadIdx.x < kSubTiles) {
            double st = 0.0;
#pragma unroll
            for (int k = 0; k < 8; ++k) st = st + (double)wt[threadIdx.x][k];
            sst[threadIdx.x] = st;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double acc = 0.0;
#pragma unroll
            for (int s = 0; s < kSubTiles; ++s) acc = acc + sst[s];
            p.cmass[(int64_t)b * p.nchunks + c] = acc;
        }
    }
    cp_async_wait_all();
}
// Small-batch staged sampler (unsharded staged path, B * CTAs per request <= SMs):
// the acceptance tests (K-B), the chunk masses (K-D1) and the draw (K-D2) of
// request b in ONE launch by CL CTAs -- the request's chunks dealt over them.
// FLAT (default): num_sms / B CTAs per request, no cluster, chunk masses through
// global memory and a per-request arrival barrier; launched as a programmatic
// dependent of k_lmhead, so its CTAs take the SMs the GEMM's CTAs free during the
// GEMM's tail and read the inputs the GEMM does not produce (q_i(x_i), u_i) before
// griddepcontrol.wait (C2 208.3-209.3 -> 204.4-205.1 us/step).
// !FLAT: a cluster of 16 / 12 / 8 / ... CTAs per request, chunk masses exchanged
// through distributed shared memory.  The arithmetic and its order are k_accept's,
// k_mass's and k_locate's (bit-identical decisions, masses and draws in both modes).
constexpr int kSmallCl = 8;         // CTAs per request (16 when B <= 8: one cluster per GPC)
constexpr int kSmallMaxPerCta = 4;  // chunks per staged batch (two batch buffers of <= 3 x 32 KB)
constexpr int kSmallMaxChunks = 64;
constexpr int kSmallMaxRows = 16;   // gamma_max <= 15
__device__ __forceinline__ const float* small_q_row(const MassParams& p, int g) {
    return (p.q_loc && ((p.q_loc_mask[g >> 6] >> (g & 63)) & 1ull)) ? p.q_loc + (int64_t)g * p.ldq
                                                                      : p.q + (int64_t)g * p.ldq;
}
template <bool FLAT>
__global__ void __launch_bounds__(kSampThreads) k_sample_small(const AcceptParams ap, const MassParams p,
                                                               const ReqMeta m) {
    // launched with programmatic dependent launch: the CTAs start on SMs the GEMM's
    // finished CTAs free, then wait here for the whole GEMM grid and its writes
    if (p.ts && threadIdx.x == 0 && blockIdx.x < 128) p.ts[18432 + blockIdx.x * 16 + 0] = globaltimer();
    // FLAT: flat_cpr CTAs per request without a cluster (a PDL dependent can then be
    // scheduled on the SMs the GEMM's CTAs free during its tail)
    const int b = FLAT ? (int)blockIdx.x / p.flat_cpr : (int)cluster_id_x();
    const int rank = FLAT ? (int)blockIdx.x - b * p.flat_cpr : (int)cluster_ctarank();
    const int CL = FLAT ? p.flat_cpr : (int)cluster_nctarank();   // CTAs per request
    const int ro = m.row_off[b], gam = m.row_off[b + 1] - ro - 1, g0 = ro - b;
    // inputs of the acceptance tests that the GEMM does not produce (q_i(x_i), u_i) are
    // read before the wait, while the GEMM's tail still runs
    double qx_pre = 0.0, u_pre = 0.0;
    if (warp_id() == 0 && (int)lane_id() < gam) {
        const int g = g0 + (int)lane_id();
        qx_pre = (double)small_q_row(p, g)[ap.draft_tokens[g]];
        u_pre = (double)ap.u[ro + (int)lane_id()];
    }
    // optional: this CTA's chunks of every candidate q row into L2 before the wait
    if (FLAT && p.pf_rows == 2 && threadIdx.x < 32) {
        const int c = rank + (int)(threadIdx.x >> 2) * CL;
        if (c < p.nchunks) {
            const int x0 = c * kChunk, nn = min(kChunk, p.V_local - x0) & ~3;
            for (int i = (int)(threadIdx.x & 3); i < gam; i += 4)
                bulk_prefetch_l2(small_q_row(p, g0 + i) + p.v_begin + x0, (uint32_t)nn * 4u);
        }
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (p.ts && threadIdx.x == 0 && blockIdx.x < 128) p.ts[18432 + blockIdx.x * 16 + 1] = globaltimer();

    // let the fp64 fallback kernel (launched next with programmatic serialization) be
    // scheduled now: it waits in its own griddepcontrol.wait for this grid to finish
    if (p.pdl_trigger && threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    __shared__ double s_lrow[kSmallMaxRows];
    __shared__ int s_n;
    // every candidate sample row's (and its q row's) chunks of this CTA into L2 while
    // the acceptance tests run; the staging after them then hits L2
    if (p.pf_rows == 1 && threadIdx.x < 32) {
        const int c = rank + (int)(threadIdx.x >> 2) * CL;   // lanes: (chunk slot, 4 rows each)
        if (c < p.nchunks) {
            const int x0 = c * kChunk, nn = min(kChunk, p.V_local - x0) & ~3;
            for (int i = (int)(threadIdx.x & 3); i <= gam; i += 4) {
                bulk_prefetch_l2(p.logits + (int64_t)(ro + i) * p.ld + x0, (uint32_t)nn * 4u);
                if (i < gam) bulk_prefetch_l2(p.q + (int64_t)(g0 + i) * p.ldq + p.v_begin + x0, (uint32_t)nn * 4u);
            }
        }
    }
    __shared__ double cml[kSmallMaxChunks];   // this CTA's chunk masses (slot = chunk)
    __shared__ double cm[kSmallMaxChunks];    // every chunk mass of the request
    __shared__ float wt[kSubTiles][8];
    __shared__ double sst[kSubTiles];
    __shared__ double spre[kSubTiles + 1];
    __shared__ double sh_tp, sh_W;
    __shared__ int sh_c, sh_clamp, ssel;
    __shared__ int wpick[8];
    // (1) lse of every row of the request from its per-row partials, one warp per row
    for (int i = (int)warp_id(); i <= gam; i += kSampThreads / 32) {
        const double l = warp_lse(ap.part_m, ap.part_s, ap.pld, ro + i, ap.grid);
        if (lane_id() == 0) s_lrow[i] = l;
    }
    __syncthreads();
    if (p.ts && threadIdx.x == 0 && blockIdx.x < 128) p.ts[18432 + blockIdx.x * 16 + 2] = globaltimer();
    // (2) acceptance and first rejection: lane i of warp 0 tests draft i (k_accept's
    //     expressions), the first failing lane is the rejection; a near-tie flag counts
    //     only for tests up to it (k_accept stops there).  Every CTA of the cluster
    //     decides identically, rank 0 writes.
    if (warp_id() == 0) {
        const int lane = (int)lane_id();
        bool fail = false, near = false;
        double pd = 0.0;
        if (lane < gam) {
            const int g = g0 + lane;
            const double lse = s_lrow[lane], dlv = __ldcg(&ap.dl[g]);
            pd = exp(dlv - lse);
            const double uq = u_pre * qx_pre;   // u_i * q_i(x_i), read before the wait
            near = fabs(uq - pd) <= (double)ap.eps_acc * pd;
            fail = !(uq < pd);
        }
        const unsigned fm = __ballot_sync(0xffffffffu, fail);
        const int n = fm ? __ffs(fm) - 1 : gam;
        const bool flag = __ballot_sync(0xffffffffu, near && lane <= n) != 0u;
        if (rank == 0) {
            if (lane < gam) {
                if (ap.dbg_lse) ap.dbg_lse[ro + lane] = (float)s_lrow[lane];
                if (ap.dbg_pdraft) ap.dbg_pdraft[g0 + lane] = (float)pd;
            }
            if (lane == 0) {
                ap.accept_len[b] = n;
                if (ap.certify && (flag || ap.force_fallback))
                    push_fallback(ap.fb_count, ap.fb_list, ap.req_flags, b, 0);
            }
        }
        if (lane == 0) s_n = n;
    }
    __syncthreads();
    if (p.ts && threadIdx.x == 0 && blockIdx.x < 128) p.ts[18432 + blockIdx.x * 16 + 3] = globaltimer();
    const int n = s_n;
    const bool resid = n < gam;
    const float* lrow = p.logits + (int64_t)(ro + n) * p.ld;
    const float* qrow = resid ? small_q_row(p, g0 + n) + p.v_begin : nullptr;
    const double lse = s_lrow[n];
    const float lsef = (float)lse, corr = lse_corr(lse);
    // (3) this CTA's chunk masses (k_mass's weights and reduction order): its chunks
    //     c = rank, rank + CL, ... (logits, and q for a residual row) staged with cp.async
    //     in batches of PB chunks, double-buffered; per batch every chunk's 16 sub-tile
    //     warp totals first, then the sub-tile sums in parallel and each chunk total
    extern __shared__ __align__(16) float stage[];   // [2 buffers][PB][2][kChunk]
    __shared__ float wtc[kSmallMaxPerCta][kSubTiles][8];
    __shared__ double sstc[kSmallMaxPerCta][kSubTiles];
    const int PB = p.small_pb;
    const int nmine = rank < p.nchunks ? (p.nchunks - rank + CL - 1) / CL : 0;
    const int nbat = (nmine + PB - 1) / PB;
    auto stage_batch = [&](int bi) {
        float* buf = stage + (size_t)(bi & 1) * PB * 2 * kChunk;
        for (int k = 0; k < PB; ++k) {
            const int j = bi * PB + k;
            if (j >= nmine) break;
            const int x0 = (rank + j * CL) * kChunk, nn = min(kChunk, p.V_local - x0);
            mass_copy_chunk(buf + (size_t)k * 2 * kChunk, lrow + x0, nn);
            if (resid) mass_copy_chunk(buf + (size_t)k * 2 * kChunk + kChunk, qrow + x0, nn);
        }
        cp_async_commit();
    };
    if (nbat > 0) stage_batch(0);
    for (int bi = 0; bi < nbat; ++bi) {
        if (bi + 1 < nbat) {
            stage_batch(bi + 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const float* buf = stage + (size_t)(bi & 1) * PB * 2 * kChunk;
        const int nk = min(PB, nmine - bi * PB);
        for (int k = 0; k < nk; ++k) {
            const int c = rank + (bi * PB + k) * CL;
            const float* sl = buf + (size_t)k * 2 * kChunk;
            const float* sq = sl + kChunk;
            const int x0 = c * kChunk + (int)threadIdx.x;
            float v[kSubTiles];
#pragma unroll
            for (int s2 = 0; s2 < kSubTiles; ++s2) {
                const int o = s2 * kSampThreads + (int)threadIdx.x;
                const bool in = x0 + s2 * kSampThreads < p.V_local;
                const float e = in ? p_weight(sl[o], lsef, corr) : 0.f;
                v[s2] = resid ? resid_weight(e, in ? sq[o] : 0.f) : e;
            }
            warp_totals16(v, wtc[k]);
        }
        __syncthreads();
        for (int t = threadIdx.x; t < nk * kSubTiles; t += kSampThreads) {
            const int k2 = t / kSubTiles, s2 = t - k2 * kSubTiles;
            double st = 0.0;
#pragma unroll
            for (int k = 0; k < 8; ++k) st = st + (double)wtc[k2][s2][k];
            sstc[k2][s2] = st;
        }
        __syncthreads();
        for (int k2 = threadIdx.x; k2 < nk; k2 += kSampThreads) {
            double acc = 0.0;
#pragma unroll
            for (int s2 = 0; s2 < kSubTiles; ++s2) acc = acc + sstc[k2][s2];
            cml[rank + (bi * PB + k2) * CL] = acc;
        }
        __syncthreads();   // wtc / sstc / this buffer are reused two batches on
    }
    // (4) every chunk mass from the CTA that owns it (distributed shared memory); the
    //     second cluster barrier keeps each CTA's cml alive until all have read it
    if (p.ts && threadIdx.x == 0 && blockIdx.x < 128) p.ts[18432 + blockIdx.x * 16 + 4] = globaltimer();
    if constexpr (FLAT) {
        // this CTA's chunk masses to global memory, then a barrier over the request's
        // CTAs (arrival counter, zeroed by the call's fb_block memset; all B x CL CTAs are
        // co-resident once the GEMM's CTAs have exited, B x CL <= SMs), then every CTA
        // reads all masses, so the owner of the located chunk draws from its staging buffer
        for (int j = threadIdx.x; j < nmine; j += kSampThreads) {
            const int c = rank + j * CL;
            p.cm_glob[(int64_t)b * p.nchunks + c] = cml[c];
        }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) {
            atomicAdd(&p.cm_cnt[b], 1);
            const long long t0 = clock64();
            while ((int)ld_acquire_gpu(reinterpret_cast<const uint32_t*>(&p.cm_cnt[b])) < CL) {
                __nanosleep(20);
                watchdog(t0);
            }
        }
        __syncthreads();
        if (p.ts && threadIdx.x == 0 && blockIdx.x < 128) p.ts[18432 + blockIdx.x * 16 + 5] = globaltimer();
        for (int c = threadIdx.x; c < p.nchunks; c += kSampThreads) cm[c] = __ldcg(&p.cm_glob[(int64_t)b * p.nchunks + c]);
        __syncthreads();
    } else {
        cluster_sync_all();
        if (p.ts && threadIdx.x == 0 && blockIdx.x < 128) p.ts[18432 + blockIdx.x * 16 + 5] = globaltimer();
        for (int c = threadIdx.x; c < p.nchunks; c += kSampThreads)
            cm[c] = ld_shared_cluster_f64(mapa_shared(&cml[c], (uint32_t)(c % CL)));
        __syncthreads();
        cluster_sync_all();
    }
    if (p.ts && threadIdx.x == 0 && blockIdx.x < 128) p.ts[18432 + blockIdx.x * 16 + 6] = globaltimer();
    // (5) the draw: k_locate's unsharded arithmetic; the CTA owning the located chunk finishes
    if (threadIdx.x == 0) {
        double W = 0.0;
        for (int c = 0; c < p.nchunks; ++c) W = W + cm[c];
        const double T = (double)p.u[ro + gam] * W;
        double P = 0.0, Pc = 0.0;
        int csel = -1, lastpos = -1;
        for (int c = 0; c < p.nchunks; ++c) {
            const double wc = cm[c];
            if (wc > 0.0) lastpos = c;
            if (csel < 0 && T < P + wc) { csel = c; Pc = P; }
            P = P + wc;
        }
        int clamp = 0;
        if (!(W > 0.0)) clamp = 2;               // zero mass (R6) -> fp64 fallback
        else if (csel < 0) { clamp = 1; csel = lastpos; Pc = 0.0; }
        sh_tp = T - Pc;
        sh_c = csel;
        sh_clamp = clamp;
        sh_W = W;
        if (rank == 0 && p.dbg_lse && !resid) p.dbg_lse[ro + gam] = (float)lse;
    }
    __syncthreads();
    const int clamp = sh_clamp;
    if (clamp == 2) {
        if (rank == 0 && threadIdx.x == 0) {
            p.next_token[b] = 0;
            if (p.dbg_mass) p.dbg_mass[b] = 0.0;
            if (p.dbg_flags) p.dbg_flags[b] = 2;
            flag_draw(p, b, 2);
        }
        return;
    }
    const int c = sh_c;
    if (p.ts && threadIdx.x == 0 && blockIdx.x < 128) p.ts[18432 + blockIdx.x * 16 + 7] = globaltimer();
    if (c % CL != rank) return;
    const double tp = sh_tp;
    float w[kSubTiles], v[kSubTiles];
    // the located chunk's weights again (k_locate's chunk_weight: same expression), from
    // this CTA's staging buffer when no later batch reused it (<= 2 batches), else global
    if (p.small_reuse && nbat <= 2) {
        const int j = (c - rank) / CL;
        const float* sl = stage + (size_t)((j / PB) & 1) * PB * 2 * kChunk + (size_t)(j % PB) * 2 * kChunk;
        const float* sq = sl + kChunk;
        const int x0 = c * kChunk + (int)threadIdx.x;
#pragma unroll
        for (int s2 = 0; s2 < kSubTiles; ++s2) {
            const int o = s2 * kSampThreads + (int)threadIdx.x;
            const bool in = x0 + s2 * kSampThreads < p.V_local;
            const float e = in ? p_weight(sl[o], lsef, corr) : 0.f;
            v[s2] = w[s2] = resid ? resid_weight(e, in ? sq[o] : 0.f) : e;
        }
    } else {
#pragma unroll
        for (int s2 = 0; s2 < kSubTiles; ++s2) v[s2] = w[s2] = chunk_weight(p, lrow, c, s2, lsef, corr, resid, qrow);
    }
    warp_totals16(v, wt);
    __syncthreads();
    if (threadIdx.x < kSubTiles) {
        double st = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) st = st + (double)wt[threadIdx.x][k];
        sst[threadIdx.x] = st;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double acc = 0.0;
        int sel = -1, lastpos = -1;
        for (int s2 = 0; s2 < kSubTiles; ++s2) {
            spre[s2] = acc;
            const double st = sst[s2];
            if (st > 0.0) lastpos = s2;
            acc = acc + st;
            if (sel < 0 && tp < acc) sel = s2;
        }
        spre[kSubTiles] = acc;
        if (clamp || sel < 0) sel = -1 - lastpos;
        ssel = sel;
    }
    __syncthreads();
    int s = ssel;
    const bool clamped = s < 0;
    if (clamped) s = -1 - s;
    float ws = 0.f;
#pragma unroll
    for (int k = 0; k < kSubTiles; ++k)
        if (k == s) ws = w[k];
    const float is = warp_incl_scan(ws);
    float ex = __shfl_up_sync(0xffffffffu, is, 1);
    if (lane_id() == 0) ex = 0.f;
    double Sq = 0.0;
    for (int k = 0; k < (int)warp_id(); ++k) Sq = Sq + (double)wt[s][k];
    const double lo = spre[s] + (Sq + (double)ex);
    const double hi = spre[s] + (Sq + (double)is);
    const int x = c * kChunk + s * kSampThreads + (int)threadIdx.x;
    if (clamped) {
        const unsigned mpos = __ballot_sync(0xffffffffu, ws > 0.f);
        if (lane_id() == 0) wpick[warp_id()] = mpos ? (31 - __clz((int)mpos)) : -1;
        __syncthreads();
        if (threadIdx.x == 0) {
            int pick = -1;
            for (int k = 7; k >= 0 && pick < 0; --k)
                if (wpick[k] >= 0) pick = k * 32 + wpick[k];
            p.next_token[b] = c * kChunk + s * kSampThreads + (pick < 0 ? 0 : pick) + p.v_begin;
            if (p.dbg_mass) p.dbg_mass[b] = sh_W;
            if (p.dbg_flags) p.dbg_flags[b] = 4;
            flag_draw(p, b, 4);
        }
        return;
    }
    if (ws > 0.f && lo <= tp && tp < hi) {
        p.next_token[b] = x + p.v_begin;
        if (p.dbg_mass) p.dbg_mass[b] = sh_W;
        if (p.dbg_flags) p.dbg_flags[b] = 0;
        const double margin = fmin(tp - lo, hi - tp);
        if (margin <= (double)p.eps_draw) flag_draw(p, b, 0);
        if (p.ts && blockIdx.x < 128) p.ts[18432 + blockIdx.x * 16 + 8] = globaltimer();
    }
}

constexpr size_t mass_smem(int nst, int B) { return (size_t)nst * 2 * kChunk * sizeof(float) + (size_t)B * 12; }

// nj_verify_greedy: argmax over the vocabulary of
// each fp32 logits row (ties -> lowest id).  Grid (nsplit, rows): a CTA scans
// one contiguous segment of a row with 8 loads in flight per thread and folds
// its (max, id) into the row's 64-bit key by atomicMax: key = order-preserving
// float bits << 32 | (0xffffffff - id), so the largest key is the largest
// logit with the lowest id.  keys must be zero on entry.
__device__ __forceinline__ unsigned long long argmax_key(float v, int x) {
    const uint32_t u = __float_as_uint(v);
    const uint32_t o = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    return ((unsigned long long)o << 32) | (unsigned long long)(0xffffffffu - (uint32_t)x);
}
__global__ void __launch_bounds__(256) k_argmax_rows(const float* __restrict__ logits, int64_t ld, int V,
                                                      unsigned long long* __restrict__ keys) {
    const float* row = logits + (int64_t)blockIdx.y * ld;
    const int seg = (V + gridDim.x - 1) / gridDim.x;
    const int x0 = blockIdx.x * seg, x1 = min(V, x0 + seg);
    unsigned long long best = 0ull;
    constexpr int U = 8;
    for (int base = x0 + (int)threadIdx.x; base < x1; base += U * 256) {
        float v[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int x = base + k * 256;
            v[k] = x < x1 ? __ldcs(&row[x]) : -INFINITY;
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int x = base + k * 256;
            if (x < x1) {
                const unsigned long long key = argmax_key(v[k], x);
                best = key > best ? key : best;
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long k2 = __shfl_xor_sync(0xffffffffu, best, o);
        best = k2 > best ? k2 : best;
    }
    __shared__ unsigned long long sk[8];
    if (lane_id() == 0) sk[warp_id()] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x / 32); ++w) best = sk[w] > best ? sk[w] : best;
        if (best) atomicMax(&keys[blockIdx.y], best);
    }
}

// Greedy target (p_i = one-hot at a_i = argmax l_i): Leviathan's test
// u q(x) < p(x) accepts x_i iff x_i == a_i; the residual max(0, p - q) of the
// first rejected row n is one-hot at a_n, and the bonus row gives a_gamma, so
// next_token = a_n in every case.  Thread per request.
// k_lmhead ARGMAX partials (per row, one per unit group: ordered value bits, id) -> the
// row's 64-bit argmax key (same ordering as argmax_key); warp per row
__global__ void k_argmax_merge(const float* __restrict__ pm, const float* __restrict__ ps, int pld, int nparts,
                               int n, unsigned long long* __restrict__ keys) {
    const int r = blockIdx.x * (blockDim.x / 32) + (int)(threadIdx.x >> 5);
    if (r >= n) return;
    unsigned long long best = 0ull;
    for (int c = (int)(threadIdx.x & 31); c < nparts; c += 32) {
        const uint32_t o = __float_as_uint(pm[(int64_t)r * pld + c]);
        const int id = __float_as_int(ps[(int64_t)r * pld + c]);
        if (o == 0u) continue;   // a group without ids of this row
        const unsigned long long k = ((unsigned long long)o << 32) | (unsigned long long)(0xffffffffu - (uint32_t)id);
        best = k > best ? k : best;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long k2 = __shfl_xor_sync(0xffffffffu, best, o);
        best = k2 > best ? k2 : best;
    }
    if ((threadIdx.x & 31) == 0) keys[r] = best;
}
__device__ __forceinline__ int argmax_of_key(unsigned long long k) {
    return (int)(0xffffffffu - (uint32_t)(k & 0xffffffffull));
}
__global__ void k_greedy_decide(const ReqMeta m, const int32_t* __restrict__ draft_tokens,
                                const unsigned long long* __restrict__ keys, int32_t* accept_len,
                                int32_t* next_token) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= m.B) return;
    const int ro = m.row_off[b], gam = m.row_off[b + 1] - ro - 1, g0 = ro - b;
    int n = gam;
    for (int i = 0; i < gam; ++i)
        if (draft_tokens[g0 + i] != argmax_of_key(keys[ro + i])) { n = i; break; }
    accept_len[b] = n;
    next_token[b] = argmax_of_key(keys[ro + n]);
}

// K-D2: block per request.  Locate chunk -> sub-tile -> token.
// Vocab-sharded mode (xr2: X2 entries (lse used, local mass W_r, rank-local lse
// of the sample row) per rank, `xstride` doubles apart): the rank whose
// exclusive prefix of the rescaled masses holds u * total locates the token,
// the others write -1.  If the residual mass is zero on every rank (R6), all
// ranks see it identically after X2 and draw from p_n instead: the masses are
// exp(lse_r(n) - M), and the owner recomputes its p_n chunk masses here.
__global__ void __launch_bounds__(kSampThreads) k_locate(const MassParams p, const ReqMeta m) {
    pdl_enter();
    const int b = blockIdx.x;
    const double lse = sample_lse(p, b);
    const bool resid0 = p.s_resid[b] != 0;
    const float* qrow = resid0 ? p.q + (int64_t)p.s_qrow[b] * p.ldq + p.v_begin : nullptr;
    const float* lrow = logits_row(p, b);
    __shared__ double sh[4];
    __shared__ int shi[4];
    __shared__ float wt[kSubTiles][8];
    const int gam = p.stage_mode ? 0 : m.row_off[b + 1] - m.row_off[b] - 1;
    const float uf = p.stage_mode ? p.u[b] : p.u[m.row_off[b] + gam];
    __shared__ int s_own, s_zero;
    __shared__ double s_scale, s_T, s_lse;
    // the request's chunk masses -> smem with one parallel load (thread 0's
    // fixed-order scans below then run on smem, not on dependent global loads)
    constexpr int kMaxSmemChunks = 64;
    __shared__ double scm[kMaxSmemChunks];
    const bool cm_smem = p.nchunks <= kMaxSmemChunks;
    if (cm_smem)
        for (int c = threadIdx.x; c < p.nchunks; c += blockDim.x) scm[c] = __ldcg(&p.cmass[(int64_t)b * p.nchunks + c]);
    __syncthreads();
    double* cm = cm_smem ? scm : p.cmass + (int64_t)b * p.nchunks;
    if (threadIdx.x == 0) {
        double W = 0.0;
        for (int c = 0; c < p.nchunks; ++c) W = W + cm[c];
        double T = (double)uf * W;
        int own = 1, zero_g = 0;
        double scale = 1.0;   // local mass units -> natural (p) units
        double lse_use = lse;
        if (p.xr2) {
            // global inverse CDF over the ranks' masses in rank order (nj_shard.cuh, X2)
            const int64_t xs = p.xstride;
            auto X = [&](int r, int k) { return p.xr2[(int64_t)r * xs + (int64_t)b * 3 + k]; };
            double M = -INFINITY;
            for (int r = 0; r < p.nranks; ++r)
                if (X(r, 1) > 0.0) M = fmax(M, X(r, 0));
            double Tot = 0.0;
            for (int r = 0; r < p.nranks; ++r)
                if (X(r, 1) > 0.0) Tot += X(r, 1) * exp(X(r, 0) - M);
            const bool pn = !(Tot > 0.0);   // zero residual mass on every rank (R6): p_n
            int col = 0;
            double nrm = resid0 ? 1.0 : 1.0 / Tot;   // bonus rows: natural mass = A / Tot
            if (pn) {
                zero_g = 1;
                M = -INFINITY;
                for (int r = 0; r < p.nranks; ++r) M = fmax(M, X(r, 2));
                Tot = 0.0;
                for (int r = 0; r < p.nranks; ++r) Tot += exp(X(r, 2) - M);
                col = 2;
                nrm = 1.0 / Tot;
            }
            const double Tg = (double)uf * Tot;
            double Pg = 0.0, Po = 0.0, Ao = 0.0;
            int o = -1, lastr = -1;
            for (int r = 0; r < p.nranks; ++r) {
                const double A = pn ? exp(X(r, 2) - M) : (X(r, 1) > 0.0 ? X(r, 1) * exp(X(r, 0) - M) : 0.0);
                if (A > 0.0) {
                    lastr = r;
                    if (o < 0 && Tg < Pg + A) { o = r; Po = Pg; Ao = A; }
                }
                Pg += A;
            }
            int clamp_g = 0;
            if (o < 0) { o = lastr; clamp_g = 1; }
            own = (o == p.rank);
            if (own) {
                const double e = exp(X(p.rank, col) - M);   // this rank's units -> the global ones
                scale = e * nrm;
                if (pn) {
                    lse_use = X(p.rank, 2);   // local weights exp(l - lse_r(n)) sum to 1
                    T = clamp_g ? 1.0 : (Tg - Po) / e;   // fraction of the local mass (rescaled below)
                } else {
                    T = clamp_g ? W : (Tg - Po) / e;
                    if (!clamp_g && fmin(Tg - Po, Po + Ao - Tg) * nrm <= (double)p.eps_draw) flag_draw(p, b, 0);
                }
                if (clamp_g) flag_draw(p, b, 4);
            }
            if (pn) flag_draw(p, b, 2);
            if (p.dbg_mass) p.dbg_mass[b] = pn ? 0.0 : (resid0 ? Tot : 1.0);
        }
        s_own = own;
        s_zero = zero_g;
        s_scale = scale;
        s_T = T;
        s_lse = lse_use;
        sh[1] = W;
    }
    __syncthreads();
    if (p.xr2 && !s_own) {   // another rank owns this draw
        if (threadIdx.x == 0) p.next_token[b] = -1;
        return;
    }
    const bool resid = resid0 && !s_zero;
    const float lsef = (float)s_lse, corr = lse_corr(s_lse);
    if (s_zero) {
        // R6 on the owner rank: this request's p_n chunk masses with the rank-local
        // lse (k_mass summed the residual), same reduction order as k_mass
        for (int c = 0; c < p.nchunks; ++c) {
            float v[kSubTiles];
#pragma unroll
            for (int s2 = 0; s2 < kSubTiles; ++s2) v[s2] = chunk_weight(p, lrow, c, s2, lsef, corr, false, qrow);
            warp_totals16(v, wt);
            __syncthreads();
            __shared__ double sst0[kSubTiles];
            if (threadIdx.x < kSubTiles) {
                double st = 0.0;
#pragma unroll
                for (int k = 0; k < 8; ++k) st = st + (double)wt[threadIdx.x][k];
                sst0[threadIdx.x] = st;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                double acc = 0.0;
#pragma unroll
                for (int k = 0; k < kSubTiles; ++k) acc = acc + sst0[k];
                cm[c] = acc;
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            double W = 0.0;
            for (int c = 0; c < p.nchunks; ++c) W = W + cm[c];
            sh[1] = W;
            s_T = s_T * W;   // fraction of the local mass -> local units
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double W = sh[1];
        const double T = s_T;
        double P = 0.0, Pc = 0.0;
        int csel = -1, lastpos = -1;
        for (int c = 0; c < p.nchunks; ++c) {
            const double wc = cm[c];
            if (wc > 0.0) lastpos = c;
            if (csel < 0 && T < P + wc) { csel = c; Pc = P; }
            P = P + wc;
        }
        int clamp = 0;
        if (!(W > 0.0)) clamp = 2;               // zero mass (R6, unsharded) -> fp64 fallback
        else if (csel < 0) { clamp = 1; csel = lastpos; Pc = 0.0; }
        sh[0] = T - Pc;
        shi[0] = csel;
        shi[1] = clamp;
        if (!p.stage_mode && p.dbg_lse && !resid0) p.dbg_lse[m.row_off[b] + gam] = (float)lse;
    }
    __syncthreads();
    const int clamp = shi[1];
    if (clamp == 2) {
        if (threadIdx.x == 0) {
            p.next_token[b] = p.xr2 ? -1 : 0;
            if (p.dbg_mass) p.dbg_mass[b] = 0.0;
            if (p.dbg_flags) p.dbg_flags[b] = 2;
            flag_draw(p, b, 2);
        }
        return;
    }
    const int c = shi[0];
    const double tp = sh[0];
    float w[kSubTiles], v[kSubTiles];
#pragma unroll
    for (int s = 0; s < kSubTiles; ++s) v[s] = w[s] = chunk_weight(p, lrow, c, s, lsef, corr, resid, qrow);
    warp_totals16(v, wt);   // k_mass's totals, bit for bit
    __syncthreads();
    __shared__ double spre[kSubTiles + 1];
    __shared__ double sst[kSubTiles];
    __shared__ int ssel;
    if (threadIdx.x < kSubTiles) {   // sub-tile totals in parallel (k_mass's order)
        double st = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) st = st + (double)wt[threadIdx.x][k];
        sst[threadIdx.x] = st;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double acc = 0.0;
        int sel = -1, lastpos = -1;
        for (int s = 0; s < kSubTiles; ++s) {
            spre[s] = acc;
            const double st = sst[s];
            if (st > 0.0) lastpos = s;
            acc = acc + st;
            if (sel < 0 && tp < acc) sel = s;
        }
        spre[kSubTiles] = acc;
        if (clamp || sel < 0) sel = -1 - lastpos;          // clamp marker
        ssel = sel;
    }
    __syncthreads();
    int s = ssel;
    const bool clamped = s < 0;
    if (clamped) s = -1 - s;
    float ws = 0.f;
#pragma unroll
    for (int k = 0; k < kSubTiles; ++k)
        if (k == s) ws = w[k];
    const float is = warp_incl_scan(ws);   // the located sub-tile's prefix only
    float ex = __shfl_up_sync(0xffffffffu, is, 1);
    if (lane_id() == 0) ex = 0.f;
    double Sq = 0.0;
    for (int k = 0; k < (int)warp_id(); ++k) Sq = Sq + (double)wt[s][k];
    const double lo = spre[s] + (Sq + (double)ex);
    const double hi = spre[s] + (Sq + (double)is);
    const int x = c * kChunk + s * kSampThreads + (int)threadIdx.x;
    if (clamped) {
        const unsigned mpos = __ballot_sync(0xffffffffu, ws > 0.f);
        __shared__ int wpick[8];
        if (lane_id() == 0) wpick[warp_id()] = mpos ? (31 - __clz((int)mpos)) : -1;
        __syncthreads();
        if (threadIdx.x == 0) {
            int pick = -1;
            for (int k = 7; k >= 0 && pick < 0; --k)
                if (wpick[k] >= 0) pick = k * 32 + wpick[k];
            p.next_token[b] = c * kChunk + s * kSampThreads + (pick < 0 ? 0 : pick) + p.v_begin;
            if (p.dbg_mass && !p.xr2) p.dbg_mass[b] = sh[1];
            if (p.dbg_flags) p.dbg_flags[b] = 4;
            flag_draw(p, b, 4);
        }
        return;
    }
    if (ws > 0.f && lo <= tp && tp < hi) {
        p.next_token[b] = x + p.v_begin;
        if (p.dbg_mass && !p.xr2) p.dbg_mass[b] = sh[1];
        if (p.dbg_flags) p.dbg_flags[b] = 0;
        const double margin = fmin(tp - lo, hi - tp) * s_scale;
        if (margin <= (double)p.eps_draw) flag_draw(p, b, 0);
    }
}

// ---------------------------------------------------------------------------
// Certified fallback (fp64 on CUDA cores): every queued request is recomputed
// from the bf16 inputs with fp64 accumulation -- the plain definition of
// include/nj.h -- and its outputs overwritten.  Launched unconditionally; an
// empty queue costs one tiny launch each.
// ---------------------------------------------------------------------------
struct FbParams {
    double inv_t;          // 1 / temperature (fp64 logits l / T); 0 taken as 1
    const uint16_t* hidden;
    const uint16_t* W;
    int32_t d, V_local, v_begin;
    const int32_t* fb_count;
    const int32_t* fb_list;
    int32_t* req_flags;
    double* fb_logits;     // [N][V_local] (row index = packed row of the request)
    int32_t* fb_done;      // k_fb completion counter (0 between calls)
    const int32_t* draft_tokens;
    const float* q;
    int64_t ldq;
    const float* u;
    int32_t* accept_len;
    int32_t* next_token;
    double* dbg_mass;
    int32_t* dbg_flags;
    // stage mode (nj_sample_from_logits): one fp32 logits row per request
    const float* st_logits;
    int64_t st_ld;
    const int32_t* st_resid;
    int32_t stage_mode;
};

__device__ __forceinline__ float bf16f(uint16_t h) { return __uint_as_float(((uint32_t)h) << 16); }

// FB-A: fp64 logits of every row of every queued request (warp per vocab id).
// Both fallback kernels are launched with programmatic dependent launch: they
// are scheduled while the producer kernel still runs and block here until its
// writes are visible, so an empty queue costs almost no launch latency.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void fb_logits_body(const FbParams& p, const ReqMeta& m, int nfb) {
    const int lane = (int)lane_id();
    const int gw = blockIdx.x * (blockDim.x / 32) + (int)warp_id();
    const int nw = gridDim.x * (blockDim.x / 32);
    const int nvec = p.d / 8;
    for (int x = gw; x < p.V_local; x += nw) {
        const uint4* wr = reinterpret_cast<const uint4*>(p.W + (int64_t)x * p.d);
        for (int k = 0; k < nfb; ++k) {
            const int b = __ldcg(&p.fb_list[k]);
            for (int j = m.row_off[b]; j < m.row_off[b + 1]; ++j) {
                const uint4* hr = reinterpret_cast<const uint4*>(p.hidden + (int64_t)j * p.d);
                double acc = 0.0;
                for (int i = lane; i < nvec; i += 32) {
                    const uint4 wv = __ldg(&wr[i]);
                    const uint4 hv = __ldg(&hr[i]);
                    const uint16_t* w16 = reinterpret_cast<const uint16_t*>(&wv);
                    const uint16_t* h16 = reinterpret_cast<const uint16_t*>(&hv);
#pragma unroll
                    for (int e = 0; e < 8; ++e) acc = fma((double)bf16f(w16[e]), (double)bf16f(h16[e]), acc);
                }
                acc = warp_sum_d(acc);
                if (p.inv_t != 0.0 && p.inv_t != 1.0) acc *= p.inv_t;
                if (lane == 0) p.fb_logits[(int64_t)j * p.V_local + x] = acc;
            }
        }
    }
}

__global__ void __launch_bounds__(256) k_fb_logits(const FbParams p, const ReqMeta m) {
    pdl_wait();
    const int nfb = __ldcg(p.fb_count);
    if (nfb == 0) return;
    fb_logits_body(p, m, nfb);
}

template <typename T>
__device__ double block_max_d(T v, double* sh) {
    double x = (double)v;
#pragma unroll
    for (int o = 16; o; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
    if (lane_id() == 0) sh[warp_id()] = x;
    __syncthreads();
    double r = -INFINITY;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) r = fmax(r, sh[w]);
    __syncthreads();
    return r;
}
__device__ double block_sum_d(double v, double* sh) {
    v = warp_sum_d(v);
    if (lane_id() == 0) sh[warp_id()] = v;
    __syncthreads();
    double r = 0.0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) r = r + sh[w];
    __syncthreads();
    return r;
}

template <typename LT>
__device__ double row_lse_d(const LT* row, int V, double* sh) {
    double mx = -INFINITY;
    for (int x = threadIdx.x; x < V; x += blockDim.x) mx = fmax(mx, (double)row[x]);
    mx = block_max_d(mx, sh);
    double s = 0.0;
    for (int x = threadIdx.x; x < V; x += blockDim.x) s += exp((double)row[x] - mx);
    s = block_sum_d(s, sh);
    return mx + log(s);
}

// FB-B: block per queued request.  fp64 lse, acceptance, residual / bonus,
// inverse CDF (block scan, ascending id) -- the plain definition.
__device__ __forceinline__ void fb_decide_body(const FbParams& p, const ReqMeta& m, int nfb, int k0, int kstep) {
    __shared__ double sh[32];
    __shared__ double lse[32];
    __shared__ int sn, st;
    __shared__ double sbase;
    const int V = p.V_local;
    for (int k = k0; k < nfb; k += kstep) {
        const int b = __ldcg(&p.fb_list[k]);
        int gam, ro;
        const double* L = nullptr;
        const float* Ls = nullptr;
        if (p.stage_mode) {
            gam = 0; ro = b;
            Ls = p.st_logits + (int64_t)b * p.st_ld;
            const double l = row_lse_d(Ls, V, sh);
            if (threadIdx.x == 0) { lse[0] = l; sn = p.st_resid[b] ? -1 : 0; }
        } else {
            ro = m.row_off[b];
            gam = m.row_off[b + 1] - ro - 1;
            L = p.fb_logits + (int64_t)ro * V;
            for (int j = 0; j <= gam; ++j) {
                const double l = row_lse_d(L + (int64_t)j * V, V, sh);
                if (threadIdx.x == 0) lse[j] = l;
            }
            if (threadIdx.x == 0) {
                const int g0 = ro - b;
                int n = gam;
                for (int i = 0; i < gam; ++i) {
                    const int x = p.draft_tokens[g0 + i] - p.v_begin;
                    const double pd = exp(L[(int64_t)i * V + x] - lse[i]);
                    const double qx = (double)p.q[(int64_t)(g0 + i) * p.ldq + p.draft_tokens[g0 + i]];
                    if (!((double)p.u[ro + i] * qx < pd)) { n = i; break; }
                }
                sn = n;
            }
        }
        __syncthreads();
        int n = sn;
        bool resid;
        const float* qrow;
        if (p.stage_mode) {
            resid = (n < 0);
            n = 0;
            qrow = p.q + (int64_t)b * p.ldq + p.v_begin;
        } else {
            resid = n < gam;
            qrow = p.q + (int64_t)(ro - b + n) * p.ldq + p.v_begin;
        }
        const double ln = lse[n];
        auto logit = [&](int x) -> double {
            return p.stage_mode ? (double)Ls[x] : L[(int64_t)n * V + x];
        };
        auto weight = [&](int x, bool res) -> double {
            const double pe = exp(logit(x) - ln);
            if (!res) return pe;
            const double d = pe - (double)qrow[x];
            return d > 0.0 ? d : 0.0;
        };
        double Wl = 0.0;
        for (int x = threadIdx.x; x < V; x += blockDim.x) Wl += weight(x, resid);
        double W = block_sum_d(Wl, sh);
        int zero = 0;
        if (W == 0.0) {   // R6
            zero = 2;
            resid = false;
            Wl = 0.0;
            for (int x = threadIdx.x; x < V; x += blockDim.x) Wl += weight(x, false);
            W = block_sum_d(Wl, sh);
        }
        const float uf = p.stage_mode ? p.u[b] : p.u[ro + gam];
        const double T = (double)uf * W;
        if (threadIdx.x == 0) { sbase = 0.0; st = 0x7fffffff; }
        __syncthreads();
        for (int x0 = 0; x0 < V; x0 += blockDim.x) {
            const int x = x0 + threadIdx.x;
            const double w = x < V ? weight(x, resid) : 0.0;
            const double inc = warp_incl_scan_d(w);
            double exc = __shfl_up_sync(0xffffffffu, inc, 1);
            if (lane_id() == 0) exc = 0.0;
            if (lane_id() == 31) sh[warp_id()] = inc;
            __syncthreads();
            double off = sbase;
            for (int k2 = 0; k2 < (int)warp_id(); ++k2) off += sh[k2];
            const double hi = off + inc;
            const double lo = off + exc;
            double tot = sbase;
            for (int k2 = 0; k2 < (int)(blockDim.x / 32); ++k2) tot += sh[k2];
            __syncthreads();
            if (w > 0.0 && lo <= T && T < hi) atomicMin(&st, x);   // first crossing (ties: smallest id)
            if (threadIdx.x == 0) sbase = tot;
            __syncthreads();
            if (st != 0x7fffffff) break;
        }
        int clampf = 0;
        if (st == 0x7fffffff) {   // overshoot (R5): last positive weight
            clampf = 4;
            if (threadIdx.x == 0) {
                int last = 0;
                for (int x = V - 1; x >= 0; --x)
                    if (weight(x, resid) > 0.0) { last = x; break; }
                st = last;
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            if (!p.stage_mode) p.accept_len[b] = n;
            p.next_token[b] = st + p.v_begin;
            if (p.dbg_mass) p.dbg_mass[b] = W;
            if (p.dbg_flags) p.dbg_flags[b] = 1 | zero | clampf;
            p.req_flags[b] = 0;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) k_fb_decide(const FbParams p, const ReqMeta m) {
    pdl_wait();
    fb_decide_body(p, m, __ldcg(p.fb_count), blockIdx.x, gridDim.x);
}

// FB (one launch): fp64 logits of the queued requests by every block, then the
// last block to finish decides them all.  An empty queue costs one PDL launch
// whose blocks exit at once (the common case).
__global__ void __launch_bounds__(256) k_fb(const FbParams p, const ReqMeta m) {
    pdl_wait();
    const int nfb = __ldcg(p.fb_count);
    if (nfb == 0) return;
    fb_logits_body(p, m, nfb);
    __threadfence();
    __syncthreads();
    __shared__ int last;
    if (threadIdx.x == 0) last = atomicAdd(p.fb_done, 1) == (int)gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    fb_decide_body(p, m, nfb, 0, 1);
    if (threadIdx.x == 0) *p.fb_done = 0;
}

}  // namespace nj
