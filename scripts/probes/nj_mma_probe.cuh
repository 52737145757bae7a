// nj_mma_probe.cuh — test-only microbenchmark of the single-thread tcgen05.mma
// issue loop (DESIGN.md §5 "what bounds k_gemm_big"): one CTA per SM, the
// operand tiles stay resident in shared memory (no TMA), one thread issues
// `iters` groups of 4 MMAs (M = 128, N = n, K = 16 each; one 64-deep
// k-block) into one TMEM accumulator, optionally committing to an mbarrier
// after every group and waiting for it (`mode` 1), committing without waiting
// (2, as the ring does), or only at the end (0).
// Reports clock64 cycles per group in out[blockIdx.x].
#pragma once
#include "nj_gemm.cuh"

namespace nj {

__global__ void __launch_bounds__(128, 1) k_mma_probe(int n, int iters, int mode, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sA = smem;                       // 16 KB: 128 x 64 bf16 (contents irrelevant)
    uint8_t* sB = smem + kTileBytesA;         // n x 128 B
    uint64_t* bar = reinterpret_cast<uint64_t*>(sB + 256 * 128);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
    for (int i = threadIdx.x; i < (kTileBytesA + 256 * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    if (threadIdx.x == 0) { mbar_init(bar, 1); mbar_init(bar + 1, 1); fence_barrier_init(); mbar_arrive(bar + 1); }
    if (warp_id() == 0) tmem_alloc(slot, 256);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *slot;
    if (mode >= 4 && warp_id() == 1) {
        // modes 4 / 5: the whole warp runs the loop (convergent), one elected lane issues
        // (mma_bf16_w / mma_kblock_w, as k_gemm_big / k_lmhead do); commit per group
        const uint32_t idesc = idesc_bf16_f32(128, (uint32_t)n);
        const uint64_t ad = sdesc_sw128(sA), bd = sdesc_sw128(sB);
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (mode == 6 || mode == 7) {
                // an operand-ready wait on an already completed barrier before every k-block:
                // 6 warp-uniform try_wait + vote (mbar_wait_w), 7 test_wait by every lane + vote
                if (mode == 6) mbar_wait_w(bar + 1, 0);
                else while (!__all_sync(0xffffffffu, mbar_test_wait(smem_u32(bar + 1), 0))) {}
#pragma unroll
                for (int k = 0; k < 4; ++k) mma_bf16_w(tbase, ad + 2 * k, bd + 2 * k, idesc, (it | k) != 0);
            } else if (mode == 4) {
#pragma unroll
                for (int k = 0; k < 4; ++k) mma_bf16_w(tbase, ad + 2 * k, bd + 2 * k, idesc, (it | k) != 0);
            } else {
                mma_kblock_w<1>(tbase, ad, bd, idesc, it != 0);
            }
            mma_commit_w(bar);
        }
        if (lane_id() == 0) out[blockIdx.x] = (clock64() - t0) / iters;
    } else if (mode < 4 && threadIdx.x == 32) {
        const uint32_t idesc = idesc_bf16_f32(128, (uint32_t)n);
        const uint64_t ad = sdesc_sw128(sA), bd = sdesc_sw128(sB);
        uint32_t ph = 0;
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 4; ++k) mma_bf16(tbase, ad + 2 * k, bd + 2 * k, idesc, (it | k) != 0);
            if (mode == 1) {
                mma_commit(bar);
                mbar_wait(bar, ph);
                ph ^= 1;
            } else if (mode == 2) {
                mma_commit(bar);   // like the ring's per-stage commit, not waited for
            }
        }
        if (mode != 2) {
            mma_commit(bar);
            mbar_wait(bar, ph);
        } else {
            tc_fence_before();   // (mode 2: the barrier phase count is not tracked)
        }
        out[blockIdx.x] = (clock64() - t0) / iters;
    }
    tc_fence_before();
    __syncthreads();
    if (warp_id() == 0) tmem_dealloc(tbase, 256);
}

// The same issue loop for a CTA pair (cta_group::2, M = 256 over two SMs, each CTA
// holding its 128 A rows and HALF of the N B rows): the leader issues, the
// commit is multicast to both CTAs.  Reports the leader's cycles per group.
__global__ void __launch_bounds__(128, 1) k_mma_probe_cg2(int n, int iters, int mode, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sA = smem;                       // 16 KB (mode 3: 4 stages of A 16 KB | B 16 KB)
    uint8_t* sB = smem + kTileBytesA;         // (n / 2) x 128 B
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 4 * (kTileBytesA + 128 * 128));
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    const bool leader = cluster_ctarank() == 0;
    for (int i = threadIdx.x; i < 4 * (kTileBytesA + 128 * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); }
    if (warp_id() == 0) tmem_alloc_cg2(slot, 256);
    fence_proxy_async();
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tbase = *slot;
    if (leader && threadIdx.x == 32) {
        const uint32_t idesc = idesc_bf16_f32(256, (uint32_t)n);
        uint32_t ph = 0;
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const int stg = mode == 3 ? (it & 3) : 0;
            const uint64_t ad = sdesc_sw128(sA + stg * (kTileBytesA + 128 * 128));
            const uint64_t bd = sdesc_sw128(sB + stg * (kTileBytesA + 128 * 128));
#pragma unroll
            for (int k = 0; k < 4; ++k) mma_bf16_cg2(tbase, ad + 2 * k, bd + 2 * k, idesc, (it | k) != 0);
            if (mode == 1) {
                mma_commit_mc2(bar, 3);
                mbar_wait(bar, ph);
                ph ^= 1;
            } else if (mode == 2) {
                mma_commit_mc2(bar, 3);
            }
        }
        if (mode != 2) {
            mma_commit_mc2(bar, 3);
            mbar_wait(bar, ph);
        }
        out[blockIdx.x] = (clock64() - t0) / iters;
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();   // the peer's barrier / TMEM stay alive until the leader is done
    if (warp_id() == 0) tmem_dealloc_cg2(tbase, 256);
}

}  // namespace nj
