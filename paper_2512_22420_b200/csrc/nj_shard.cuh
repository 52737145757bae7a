// nj_shard.cuh — device side of the vocab-sharded mode (BJ config 5; SURVEY
// §8a row a7, §8e "vocab-sharded").  Rank r of G owns the contiguous vocab
// shard [v_begin, v_end) of W_lm (rank order = ascending token id, R5).  The
// kernels here pack / merge the small per-rank summaries that the host
// exchanges between the phases of nj_verify -- FOUR collectives per step
// (NCCL allgather x3 + allreduce-MAX, or device copies inside an nj_group):
//
//   X1 (allgather)  per draft row g: (lse_r(g), l_g(x_g) if x_g is in this
//       shard else NaN) -> every rank merges lse(g) = logsumexp_r lse_r(g) in
//       rank order and takes the owner's draft logit: identical acceptance
//       decisions everywhere (k_accept with xr1).  Acceptance near-ties are
//       therefore known identically on every rank right after X1, and the
//       certified fp64 fallback's first stage (fp64 logits + per-row local
//       lse / owned draft logit of the queued requests) runs before X2.
//   X2 (allgather)  per request b: (lse used for the sample row, local mass
//       W_r, rank-local lse of the sample row) ++ the fallback's per-row
//       (lse_r, owned draft logit).  Residual rows use the global lse from X1
//       (so W_r are natural masses); bonus rows use the rank-local lse and are
//       rescaled by exp(lse_r - M).  The inverse CDF (R5) over the global
//       ascending order: T = u * sum_r A_r, owner = the rank whose exclusive
//       prefix interval holds T, local target (T - P_owner) / exp(lse_owner - M)
//       (k_locate with xr2).  Zero residual mass on every rank (R6) switches
//       every rank, identically, to p_n with masses exp(lse_r(n) - M).
//   X3 (allgather)  [next_token (-1 on non-owners) | flags] ++ the fallback's
//       fp64 local masses; every rank takes the MAX over ranks locally.
//   X4 (allreduce-MAX) the fallback's tokens (owner rank, -1 elsewhere).
#pragma once
#pragma once
#include "nj_sampler.cuh"

namespace nj {

// Merge of the X1 entries of draft row g: lse = M + log sum_r exp(lse_r - M)
// (rank order), dl = the owner's draft logit (exactly one rank is not NaN).
// (rank stride `rs` doubles between the ranks' blocks of entries)
__device__ __forceinline__ double xmerge_lse_s(const double* xr, int nranks, int64_t rs, int g, double& dl) {
    double M = -INFINITY;
    dl = __longlong_as_double(0x7ff8000000000000ll);
    for (int r = 0; r < nranks; ++r) {
        const double* e = xr + (int64_t)r * rs + (int64_t)g * 2;
        M = fmax(M, __ldcg(&e[0]));
        const double d = __ldcg(&e[1]);
        if (!isnan(d)) dl = d;
    }
    double S = 0.0;
    for (int r = 0; r < nranks; ++r) S += exp(__ldcg(&xr[(int64_t)r * rs + (int64_t)g * 2]) - M);
    return M + log(S);
}
__device__ __forceinline__ double xmerge_lse(const double* xr, int nranks, int ld, int g, double& dl) {
    return xmerge_lse_s(xr, nranks, (int64_t)ld * 2, g, dl);
}

// X1 pack: warp per draft row.
__global__ void k_xpack1(const float* part_m, const float* part_s, int pld, int grid, const double* dl, int G,
                         double* xs1, const int32_t* g2row) {
    const int g = blockIdx.x * (blockDim.x / 32) + (int)warp_id();
    if (g >= G) return;
    const double l = warp_lse(part_m, part_s, pld, g2row ? g2row[g] : g, grid);
    if (lane_id() == 0) {
        xs1[2 * g] = l;
        xs1[2 * g + 1] = __ldcg(&dl[g]);
    }
}

// X2 pack: warp per request: lse of the sample row as used by k_mass, the
// rank's mass sum_c cmass (fixed order, as k_locate sums it), and the
// rank-local lse of the sample row from K-C's statistics (R6 across shards).
// staged sharded step: the packed-row index of every draft row (row of draft g of
// request b is g + b), for k_xpack1 over per-row statistics
__global__ void k_draft_rows(const ReqMeta m, int32_t* g2row) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= m.B) return;
    for (int r = m.row_off[b]; r + 1 < m.row_off[b + 1]; ++r) g2row[r - b] = r;
}
__global__ void k_xpack2(const MassParams p, int B, double* xs2) {
    const int b = blockIdx.x * (blockDim.x / 32) + (int)warp_id();
    if (b >= B) return;
    const double lloc = warp_lse(p.part2_m, p.part2_s, p.pld2, part2_row(p, b), p.grid2);
    double l = __ldcg(&p.s_lse[b]);
    if (isnan(l)) l = lloc;
    if (lane_id() == 0) {
        double W = 0.0;
        for (int c = 0; c < p.nchunks; ++c) W = W + __ldcg(&p.cmass[(int64_t)b * p.nchunks + c]);
        xs2[3 * b] = l;
        xs2[3 * b + 1] = W;
        xs2[3 * b + 2] = lloc;
    }
}

// The fallback queue in canonical (ascending request) order, identical on every
// rank (acceptance flags come from the merged X1 data).  One block.
// One block of 1024 threads (B <= kMaxB): thread b's position is the exclusive
// count of flagged requests before it (warp ballots + a scan of warp totals).
__global__ void __launch_bounds__(1024) k_qcanon(const int32_t* req_flags, int B, int32_t* fb_count,
                                                 int32_t* fb_list, int force_all) {
    __shared__ int wtot[32];
    const int b = threadIdx.x;
    const bool f = b < B && (force_all || (__ldcg(&req_flags[b]) & 0x100));
    const unsigned m = __ballot_sync(0xffffffffu, f);
    const int lane = (int)lane_id(), w = (int)warp_id();
    if (lane == 0) wtot[w] = __popc(m);
    __syncthreads();
    int off = 0;
    for (int k = 0; k < w; ++k) off += wtot[k];
    if (f) fb_list[off + __popc(m & ((1u << lane) - 1u))] = b;
    if (b == 0) {
        int n = 0;
        for (int k = 0; k < (int)(blockDim.x / 32); ++k) n += wtot[k];
        *fb_count = n;
    }
}

// After X3: next_token / flags = max / or over the ranks' gathered entries
// (rank stride rs int32s, tokens at [0, B), flags at [mb, mb + B)).  One block.
__global__ void k_xfinish2(const int32_t* x3r, int nranks, int64_t rs, int mb, int B, int32_t* next_token,
                           int32_t* dbg_flags) {
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
        int32_t t = -1, f = 0;
        for (int r = 0; r < nranks; ++r) {
            t = max(t, x3r[(int64_t)r * rs + b]);
            f |= x3r[(int64_t)r * rs + mb + b];
        }
        next_token[b] = t;
        if (dbg_flags) dbg_flags[b] = f & 0xff;
    }
}

// In-place max over n rank buffers (nj_group's allreduce-MAX): dst = max_r src[r].
__global__ void k_imax(const int32_t* src, int n, int len, int32_t* dst) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= len) return;
    int32_t v = src[i];
    for (int r = 1; r < n; ++r) v = max(v, src[(int64_t)r * len + i]);
    dst[i] = v;
}

// ------------------------------------------------------------ fp64 fallback
// FBX-1: per queued request, per row j: rank-local fp64 lse and the owned
// draft logit (fb_logits from k_fb_logits over the local shard).
__global__ void __launch_bounds__(256) k_fbx_stats(const FbParams p, const ReqMeta m, int slots, double* s4) {
    __shared__ double sh[32];
    const int nfb = __ldcg(p.fb_count);
    const int V = p.V_local;
    for (int k = blockIdx.x; k < nfb; k += gridDim.x) {
        const int b = __ldcg(&p.fb_list[k]);
        const int ro = m.row_off[b], gam = m.row_off[b + 1] - ro - 1;
        for (int j = 0; j <= gam; ++j) {
            const double* L = p.fb_logits + (int64_t)(ro + j) * V;
            const double l = row_lse_d(L, V, sh);
            if (threadIdx.x == 0) {
                double dl = __longlong_as_double(0x7ff8000000000000ll);
                if (j < gam) {
                    const int x = p.draft_tokens[ro - b + j] - p.v_begin;
                    if (x >= 0 && x < V) dl = L[x];
                }
                s4[((int64_t)k * slots + j) * 2] = l;
                s4[((int64_t)k * slots + j) * 2 + 1] = dl;
            }
        }
    }
}

// FBX-2: merged fp64 lse, acceptance (identical on every rank), local masses
// of the residual / bonus distribution and of p_n (zero-mass rule R6).
__global__ void __launch_bounds__(256) k_fbx_accept(const FbParams p, const ReqMeta m, const double* r4, int64_t rs4,
                                                    int nranks, int slots, double* s5, int32_t* fbn, double* fblse) {
    __shared__ double sh[32];
    __shared__ double s_lse;
    __shared__ int s_n;
    const int nfb = __ldcg(p.fb_count);
    const int V = p.V_local;
    for (int k = blockIdx.x; k < nfb; k += gridDim.x) {
        const int b = __ldcg(&p.fb_list[k]);
        const int ro = m.row_off[b], gam = m.row_off[b + 1] - ro - 1, g0 = ro - b;
        if (threadIdx.x == 0) {
            int n = gam;
            double lse_n = 0.0;
            for (int i = 0; i <= gam; ++i) {
                double dl;
                const double lse = xmerge_lse_s(r4, nranks, rs4, k * slots + i, dl);
                if (i == gam) { lse_n = lse; break; }
                const double pd = exp(dl - lse);
                const double qx = (double)p.q[(int64_t)(g0 + i) * p.ldq + p.draft_tokens[g0 + i]];
                if (!((double)p.u[ro + i] * qx < pd)) { n = i; lse_n = lse; break; }
            }
            s_n = n;
            s_lse = lse_n;
        }
        __syncthreads();
        const int n = s_n;
        const double ln = s_lse;
        const bool resid = n < gam;
        const double* L = p.fb_logits + (int64_t)(ro + n) * V;
        const float* qrow = p.q + (int64_t)(g0 + n) * p.ldq + p.v_begin;
        double Wl = 0.0, Wp = 0.0;
        for (int x = threadIdx.x; x < V; x += blockDim.x) {
            const double pe = exp(L[x] - ln);
            Wp += pe;
            if (resid) { const double d = pe - (double)qrow[x]; Wl += d > 0.0 ? d : 0.0; }
            else Wl += pe;
        }
        Wl = block_sum_d(Wl, sh);
        Wp = block_sum_d(Wp, sh);
        if (threadIdx.x == 0) {
            s5[2 * k] = Wl;
            s5[2 * k + 1] = Wp;
            fbn[k] = n;
            fblse[k] = ln;
        }
        __syncthreads();
    }
}

// FBX-3: owner rank of the draw (prefix over ranks in rank order) scans its
// local fp64 weights in ascending id.  x6[k] = global token or -1,
// x6[qcap + k] = flag bits (2 zero mass, 4 clamp).
__global__ void __launch_bounds__(256) k_fbx_locate(const FbParams p, const ReqMeta m, const double* r5, int64_t rs5,
                                                    int nranks, int rank, int qcap, const int32_t* fbn,
                                                    const double* fblse, int32_t* x6) {
    __shared__ double sh[32];
    __shared__ double s_t, sbase;
    __shared__ int s_own, s_clamp, s_zero, st;
    const int nfb = __ldcg(p.fb_count);
    const int V = p.V_local;
    for (int k = blockIdx.x; k < nfb; k += gridDim.x) {
        const int b = __ldcg(&p.fb_list[k]);
        const int ro = m.row_off[b], gam = m.row_off[b + 1] - ro - 1, g0 = ro - b;
        const int n = fbn[k];
        const double ln = fblse[k];
        if (threadIdx.x == 0) {
            double Tot = 0.0;
            for (int r = 0; r < nranks; ++r) Tot += r5[(int64_t)r * rs5 + (int64_t)k * 2];
            const int zero = !(Tot > 0.0);
            const int col = zero ? 1 : 0;
            if (zero) { Tot = 0.0; for (int r = 0; r < nranks; ++r) Tot += r5[(int64_t)r * rs5 + (int64_t)k * 2 + 1]; }
            const double T = (double)p.u[ro + gam] * Tot;
            double P = 0.0;
            int own = -1, last = -1;
            double Pown = 0.0;
            for (int r = 0; r < nranks; ++r) {
                const double A = r5[(int64_t)r * rs5 + (int64_t)k * 2 + col];
                if (A > 0.0) {
                    last = r;
                    if (own < 0 && T < P + A) { own = r; Pown = P; }
                }
                P += A;
            }
            int clamp = 0;
            if (own < 0) { own = last; clamp = 1; }
            s_own = own;
            s_clamp = clamp;
            s_zero = zero;
            s_t = T - Pown;
            sbase = 0.0;
            st = 0x7fffffff;
        }
        __syncthreads();
        const bool resid = (n < gam) && !s_zero;
        if (s_own != rank) {
            if (threadIdx.x == 0) { x6[k] = -1; x6[qcap + k] = 0; }
            __syncthreads();
            continue;
        }
        const double* L = p.fb_logits + (int64_t)(ro + n) * V;
        const float* qrow = p.q + (int64_t)(g0 + n) * p.ldq + p.v_begin;
        auto weight = [&](int x) -> double {
            const double pe = exp(L[x] - ln);
            if (!resid) return pe;
            const double d = pe - (double)qrow[x];
            return d > 0.0 ? d : 0.0;
        };
        const double T = s_t;
        if (!s_clamp) {
            for (int x0 = 0; x0 < V; x0 += blockDim.x) {
                const int x = x0 + threadIdx.x;
                const double w = x < V ? weight(x) : 0.0;
                const double inc = warp_incl_scan_d(w);
                double exc = __shfl_up_sync(0xffffffffu, inc, 1);
                if (lane_id() == 0) exc = 0.0;
                if (lane_id() == 31) sh[warp_id()] = inc;
                __syncthreads();
                double off = sbase;
                for (int k2 = 0; k2 < (int)warp_id(); ++k2) off += sh[k2];
                double tot = sbase;
                for (int k2 = 0; k2 < (int)(blockDim.x / 32); ++k2) tot += sh[k2];
                __syncthreads();
                if (w > 0.0 && off + exc <= T && T < off + inc) atomicMin(&st, x);
                if (threadIdx.x == 0) sbase = tot;
                __syncthreads();
                if (st != 0x7fffffff) break;
            }
        }
        int clampf = s_clamp;
        if (st == 0x7fffffff) {   // overshoot (R5): last positive weight of this (last positive) shard
            clampf = 1;
            if (threadIdx.x == 0) {
                int lastx = 0;
                for (int x = V - 1; x >= 0; --x)
                    if (weight(x) > 0.0) { lastx = x; break; }
                st = lastx;
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            x6[k] = st + p.v_begin;
            x6[qcap + k] = (s_zero ? 2 : 0) | (clampf ? 4 : 0);
        }
        __syncthreads();
    }
}

// FBX-4: write the fallback's outputs (after the MAX exchange of x6).
__global__ void k_fbx_write(const FbParams p, const int32_t* fbn, const int32_t* x6, int qcap) {
    const int nfb = __ldcg(p.fb_count);
    for (int k = threadIdx.x; k < nfb; k += blockDim.x) {
        const int b = p.fb_list[k];
        p.accept_len[b] = fbn[k];
        p.next_token[b] = x6[k];
        if (p.dbg_flags) p.dbg_flags[b] = 1 | x6[qcap + k];
        p.req_flags[b] = 0;
    }
}

}  // namespace nj
