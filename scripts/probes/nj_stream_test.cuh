// nj_stream_test.cuh — TMA streaming microbenchmark (test-only export
// nj_stream_test): how fast can one persistent CTA per SM pull its share of
// W through a TMA -> SMEM ring, for different box orders?  Consumer releases
// each stage immediately (no MMA).  Used to pick the LM-head streaming order.
//   mode 0: K-inner  (per 128-row tile: k-blocks 0..nkb-1; box 64x128)
//   mode 1: grouped  (per 128-row tile: 4 k-blocks per stage, 4 boxes)
//   mode 2: packed   (W pre-tiled so each 16-KB box is contiguous; map over
//                     [tiles*nkb*128, 64]; CTA c owns whole tiles)
#pragma once
#include "nj_gemm.cuh"

namespace nj {

struct StreamTestParams {
    int32_t V_local, U, num_kb, nstages, mode, group;
    int32_t ntiles_total;   // mode 2
    int32_t hrows;          // >0: also load an H box of hrows rows per k-block (L2-resident)
};

__global__ void __launch_bounds__(128, 1)
k_stream_test(const __grid_constant__ CUtensorMap tmW128, const __grid_constant__ CUtensorMap tmW16,
              const __grid_constant__ CUtensorMap tmH, const StreamTestParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int S = p.nstages;
    const int G = p.group;
    const size_t stageB = (size_t)G * (kTileBytesA + p.hrows * 128);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)S * stageB);
    uint64_t* full = bars;
    uint64_t* empty = bars + S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int r0, rows;
    vocab_range(p.U, gridDim.x, blockIdx.x, p.V_local, r0, rows);
    int t0 = 0, t1 = 0;
    if (p.mode == 2) {
        const int base = p.ntiles_total / gridDim.x, rem = p.ntiles_total % gridDim.x;
        t0 = blockIdx.x * base + min((int)blockIdx.x, rem);
        t1 = t0 + base + ((int)blockIdx.x < rem ? 1 : 0);
    }
    const int ntiles = p.mode == 2 ? (t1 - t0) : (rows + kTileV - 1) / kTileV;
    const int nsteps = ntiles * ((p.num_kb + G - 1) / G);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        fence_barrier_init();
        fence_proxy_async();
    }
    __syncthreads();
    if (warp == 0 && lane == 0) {
        const uint64_t pol = policy_evict_first();
        int s = 0;
        uint32_t ph = 0;
        for (int st = 0; st < nsteps; ++st) {
            const int t = st / ((p.num_kb + G - 1) / G);
            const int kg = st % ((p.num_kb + G - 1) / G);
            mbar_wait(&empty[s], ph ^ 1);
            uint32_t bytes = 0;
            uint8_t* dst = smem + (size_t)s * stageB;
            uint8_t* hdst = dst + (size_t)G * kTileBytesA;
            for (int g = 0; g < G; ++g) {
                const int kb = kg * G + g;
                if (kb >= p.num_kb) break;
                if (p.mode == 2) bytes += kTileBytesA;
                else bytes += w_tile_bytes(min(kTileV, rows - t * kTileV));
                bytes += p.hrows * 128;
            }
            mbar_arrive_expect_tx(&full[s], bytes);
            for (int g = 0; g < G; ++g) {
                const int kb = kg * G + g;
                if (kb >= p.num_kb) break;
                if (p.mode == 2)
                    tma_load_2d(dst + (size_t)g * kTileBytesA, &tmW128, &full[s], 0,
                                ((t0 + t) * p.num_kb + kb) * kTileV, pol);
                else
                    load_w_tile(dst + (size_t)g * kTileBytesA, &tmW128, &tmW16, &full[s], kb, r0 + t * kTileV,
                                min(kTileV, rows - t * kTileV), pol);
                if (p.hrows) tma_load_2d(hdst + (size_t)g * p.hrows * 128, &tmH, &full[s], kb * kBK, 0, pol);
            }
            if (++s == S) { s = 0; ph ^= 1; }
        }
    } else if (warp == 1 && lane == 0) {
        int s = 0;
        uint32_t ph = 0;
        for (int st = 0; st < nsteps; ++st) {
            mbar_wait(&full[s], ph);
            mbar_arrive(&empty[s]);
            if (++s == S) { s = 0; ph ^= 1; }
        }
    }
    __syncthreads();
}

}  // namespace nj
