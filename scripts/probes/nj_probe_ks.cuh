// nj_probe_ks.cuh — accuracy probe: LM-head GEMM whose TMEM accumulator is
// restarted every KS MMA steps (K = 16 each) and whose partials are summed in
// fp64 by the epilogue.  Used to measure the error of tcgen05 fp32
// accumulation vs. fresh-accumulator granularity.
// Test-only export nj_lmhead_logits_ks.  N <= 32 rows per launch.
#pragma once
#include "nj_gemm.cuh"

namespace nj {

constexpr int kProbeBufs = 4;

struct ProbeKsParams {
    int32_t R, V_local, U, num_kb, nstages, ks;   // ks = MMA steps per partial (>= 1)
    double* logits;   // fp64 output (the fp64 sum of partials, unrounded)
    int64_t ld_out;
};

__global__ void __launch_bounds__(kThreads, 1)
k_probe_ks(const __grid_constant__ CUtensorMap tmW128, const __grid_constant__ CUtensorMap tmW16,
           const __grid_constant__ CUtensorMap tmH, const ProbeKsParams p) {
    constexpr int NPAD = 32;
    constexpr int kBBytes = NPAD * 128;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int S = p.nstages;
    uint8_t* sA = smem;
    uint8_t* sB = smem + (size_t)S * kTileBytesA;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + (size_t)S * kBBytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + S;
    uint64_t* pfull = bars + 2 * S;                 // [kProbeBufs]
    uint64_t* pempty = pfull + kProbeBufs;          // [kProbeBufs]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pempty + kProbeBufs);
    const int warp = (int)warp_id(), lane = (int)lane_id();
    int r0, rows;
    vocab_range(p.U, gridDim.x, blockIdx.x, p.V_local, r0, rows);
    const int ntiles = (rows + kTileV - 1) / kTileV;
    const int steps = p.num_kb * (kBK / 16);
    const int nparts = (steps + p.ks - 1) / p.ks;
    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmW128); tma_prefetch_desc(&tmW16); tma_prefetch_desc(&tmH);
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int b = 0; b < kProbeBufs; ++b) { mbar_init(&pfull[b], 1); mbar_init(&pempty[b], 4); }
        fence_barrier_init();
        fence_proxy_async();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 128);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;
    if (warp == 0 && lane == 0) {
        const uint64_t pol_w = policy_evict_first(), pol_h = policy_evict_last();
        int s = 0;
        uint32_t ph = 0;
        for (int t = 0; t < ntiles; ++t) {
            const int trows = min(kTileV, rows - t * kTileV);
            for (int kb = 0; kb < p.num_kb; ++kb) {
                mbar_wait(&empty[s], ph ^ 1);
                mbar_arrive_expect_tx(&full[s], w_tile_bytes(trows) + kBBytes);
                load_w_tile(sA + (size_t)s * kTileBytesA, &tmW128, &tmW16, &full[s], kb, r0 + t * kTileV, trows, pol_w);
                tma_load_2d(sB + (size_t)s * kBBytes, &tmH, &full[s], kb * kBK, 0, pol_h);
                if (++s == S) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1 && lane == 0) {
        constexpr uint32_t idesc = idesc_bf16_f32(128, NPAD);
        int s = 0;
        uint32_t ph = 0;
        int part = 0;   // global partial counter (buffer = part % kProbeBufs)
        for (int t = 0; t < ntiles; ++t) {
            int step = 0;
            for (int kb = 0; kb < p.num_kb; ++kb) {
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint64_t ad = sdesc_sw128(sA + (size_t)s * kTileBytesA);
                const uint64_t bd = sdesc_sw128(sB + (size_t)s * kBBytes);
                for (int k = 0; k < kBK / 16; ++k, ++step) {
                    const int buf = part % kProbeBufs;
                    if (step % p.ks == 0) {   // new partial: wait for its buffer to be drained
                        mbar_wait(&pempty[buf], ((part / kProbeBufs) & 1) ^ 1);
                        tc_fence_after();
                    }
                    mma_bf16(tbase + (uint32_t)(buf * NPAD), ad + 2 * k, bd + 2 * k, idesc, (step % p.ks) != 0);
                    if ((step + 1) % p.ks == 0 || step + 1 == steps) { mma_commit(&pfull[buf]); ++part; }
                }
                mma_commit(&empty[s]);
                if (++s == S) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp >= 4) {
        const int q = warp & 3;
        const uint32_t lane_base = tbase + ((uint32_t)(q * 32) << 16);
        int part = 0;
        for (int t = 0; t < ntiles; ++t) {
            double acc[NPAD];
#pragma unroll
            for (int j = 0; j < NPAD; ++j) acc[j] = 0.0;
            for (int pp = 0; pp < nparts; ++pp, ++part) {
                const int buf = part % kProbeBufs;
                mbar_wait(&pfull[buf], (part / kProbeBufs) & 1);
                tc_fence_after();
                float v0[16], v1[16];
                tmem_ld16(lane_base + (uint32_t)(buf * NPAD), v0);
                tmem_ld16(lane_base + (uint32_t)(buf * NPAD + 16), v1);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&pempty[buf]);
#pragma unroll
                for (int j = 0; j < 16; ++j) { acc[j] += (double)v0[j]; acc[16 + j] += (double)v1[j]; }
            }
            const int vr = q * 32 + lane;
            if (vr < min(kTileV, rows - t * kTileV)) {
                const int xl = r0 + t * kTileV + vr;
#pragma unroll
                for (int j = 0; j < NPAD; ++j)
                    if (j < p.R) p.logits[(int64_t)j * p.ld_out + xl] = acc[j];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_dealloc(tbase, 128);
}

}  // namespace nj
