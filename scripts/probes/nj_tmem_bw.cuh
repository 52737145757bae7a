// nj_tmem_bw.cuh — TMEM -> register read bandwidth probe (tcgen05.ld): how
// many bytes per cycle can the epilogue drain of a restarted accumulator move?
// One CTA per SM, `nwarps` warps (warp w reads TMEM lane quadrant w % 4), each
// warp reads a column slice of `cols` columns per round, `rounds` times, with
// `inflight` loads of 32x32b.x16 (or .x32 / .x64 by `shape`) issued before one
// tcgen05.wait::ld, and adds the values into registers (as the drain does).
// out[2 * blockIdx.x] = cycles, out[2 * blockIdx.x + 1] = checksum.
#pragma once
#include "nj_gemm.cuh"

namespace nj {

template <int X, int NL>
__device__ __forceinline__ void tmem_ld_batch(uint32_t taddr, float (&acc)[X]) {
    uint32_t r[NL][X];
    if constexpr (X == 16) {
#pragma unroll
        for (int l = 0; l < NL; ++l)
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(r[l][0]), "=r"(r[l][1]), "=r"(r[l][2]), "=r"(r[l][3]), "=r"(r[l][4]), "=r"(r[l][5]),
                  "=r"(r[l][6]), "=r"(r[l][7]), "=r"(r[l][8]), "=r"(r[l][9]), "=r"(r[l][10]), "=r"(r[l][11]),
                  "=r"(r[l][12]), "=r"(r[l][13]), "=r"(r[l][14]), "=r"(r[l][15])
                : "r"(taddr + (uint32_t)(l * X)) : "memory");
    } else {
#pragma unroll
        for (int l = 0; l < NL; ++l)
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(r[l][0]), "=r"(r[l][1]), "=r"(r[l][2]), "=r"(r[l][3]), "=r"(r[l][4]), "=r"(r[l][5]),
                  "=r"(r[l][6]), "=r"(r[l][7]), "=r"(r[l][8]), "=r"(r[l][9]), "=r"(r[l][10]), "=r"(r[l][11]),
                  "=r"(r[l][12]), "=r"(r[l][13]), "=r"(r[l][14]), "=r"(r[l][15]), "=r"(r[l][16]), "=r"(r[l][17]),
                  "=r"(r[l][18]), "=r"(r[l][19]), "=r"(r[l][20]), "=r"(r[l][21]), "=r"(r[l][22]), "=r"(r[l][23]),
                  "=r"(r[l][24]), "=r"(r[l][25]), "=r"(r[l][26]), "=r"(r[l][27]), "=r"(r[l][28]), "=r"(r[l][29]),
                  "=r"(r[l][30]), "=r"(r[l][31])
                : "r"(taddr + (uint32_t)(l * X)) : "memory");
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int l = 0; l < NL; ++l)
#pragma unroll
        for (int i = 0; i < X; ++i) acc[i] += __uint_as_float(r[l][i]);
}

template <int X, int NL>
__global__ void __launch_bounds__(512, 1) k_tmem_bw(int rounds, int cols, long long* out) {
    __shared__ uint32_t slot;
    const int warp = (int)warp_id();
    if (warp == 0) tmem_alloc(&slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = slot;
    const int nw = blockDim.x / 32;
    const int q = warp & 3, set = warp >> 2, nsets = nw / 4;
    // this warp's column slice: the quadrant's columns split over the sets
    const int per = cols / nsets;
    const uint32_t base = tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(set * per);
    float acc[X];
#pragma unroll
    for (int i = 0; i < X; ++i) acc[i] = 0.f;
    __syncthreads();
    const long long t0 = clock64();
    for (int r = 0; r < rounds; ++r)
        for (int c = 0; c + X * NL <= per; c += X * NL) tmem_ld_batch<X, NL>(base + (uint32_t)c, acc);
    __syncthreads();
    const long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < X; ++i) s += acc[i];
    if (threadIdx.x == 0) { out[2 * blockIdx.x] = t1 - t0; out[2 * blockIdx.x + 1] = (long long)s; }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tbase, 512);
}

}  // namespace nj
