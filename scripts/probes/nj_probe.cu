// nj_probe.cu — libnj_probe.so: measurement probes kept OUT of the product
// library (libnj.so).  They include libnj's device headers (PTX wrappers,
// vocabulary split, TMA tile loads) but share no state with it.
//   njp_logits_ks   LM-head GEMM whose TMEM accumulator restarts every ks MMAs,
//                   partials summed in fp64 (tcgen05 accumulation accuracy,
//                   DESIGN.md §6)
//   njp_stream_test TMA streaming of W through an SMEM ring, no compute
//
//   njp_mma_probe   single-thread tcgen05.mma issue rate
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "nj_gemm.cuh"
#include "nj_mma_probe.cuh"
#include "nj_probe_ks.cuh"
#include "nj_stream_test.cuh"
#include "nj_tmem_bw.cuh"

using namespace nj;

namespace {
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
bool encode_2d(CUtensorMap* m, const void* base, int64_t rows, int64_t d, int box_rows) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return false;
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)d * 2};
    cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
int num_sms() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}
// tile-balanced grid of the product (whole 128-row tiles per CTA)
int tile_grid(int V) {
    const int T = (V + kTileV - 1) / kTileV, sms = num_sms();
    const int tpc = (T + sms - 1) / sms;
    return std::max(1, std::min((V + kUnit - 1) / kUnit, (T + tpc - 1) / tpc));
}
}  // namespace

extern "C" {

// out[r, x] (fp64, pitch ld_out) = sum of fresh-accumulator partials of ks
// MMA steps (K = 16) of sum_k W[x,k] h[r,k];  h [n_rows <= 32, d] contiguous.
int njp_logits_ks(void* stream, const uint16_t* W, int32_t V, int32_t d, const uint16_t* h, int32_t n_rows,
                  double* out, int64_t ld_out, int32_t ks) {
    if (!W || !h || !out || n_rows < 1 || n_rows > 32 || ks < 1 || d % 8) return 1;
    CUtensorMap m128, m16, mh;
    if (!encode_2d(&m128, W, V, d, 128) || !encode_2d(&m16, W, V, d, 16) || !encode_2d(&mh, h, n_rows, d, 32))
        return 3;
    ProbeKsParams pp{};
    pp.R = n_rows; pp.V_local = V; pp.U = (V + kUnit - 1) / kUnit; pp.num_kb = (d + kBK - 1) / kBK;
    pp.nstages = 8; pp.ks = ks; pp.logits = out; pp.ld_out = ld_out;
    const size_t smem = (size_t)8 * (kTileBytesA + 32 * 128) + (2 * 8 + 2 * kProbeBufs) * 8 + 16;
    if (cudaFuncSetAttribute(k_probe_ks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 3;
    k_probe_ks<<<tile_grid(V), kThreads, smem, reinterpret_cast<cudaStream_t>(stream)>>>(m128, m16, mh, pp);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

// Every CTA pulls its vocab share of W [V, d] through a ring of nstages stages
// of `group` 64x128 boxes (mode 0/1; mode 2 = W pre-tiled), optionally with an
// H box of hrows rows per k-block.  grid <= 0: the product's tile-balanced grid.
int njp_stream_test(void* stream, const uint16_t* W, int32_t V, int32_t d, int32_t mode, int32_t group,
                    int32_t nstages, const uint16_t* H, int32_t hrows, int32_t grid) {
    if (!W) return 1;
    StreamTestParams sp{};
    sp.V_local = V; sp.U = (V + kUnit - 1) / kUnit; sp.num_kb = (d + kBK - 1) / kBK; sp.nstages = nstages;
    sp.mode = mode; sp.group = group; sp.ntiles_total = V / kTileV;
    CUtensorMap m128, m16;
    if (mode == 2) {
        if (!encode_2d(&m128, W, (int64_t)sp.ntiles_total * sp.num_kb * kTileV, kBK, 128)) return 3;
        m16 = m128;
    } else if (!encode_2d(&m128, W, V, d, 128) || !encode_2d(&m16, W, V, d, 16)) {
        return 3;
    }
    sp.hrows = H ? hrows : 0;
    CUtensorMap mh = m128;
    if (H && !encode_2d(&mh, H, hrows, d, hrows)) return 3;
    const size_t smem = (size_t)nstages * group * (kTileBytesA + sp.hrows * 128) + 2 * nstages * 8 + 16;
    if (smem > (size_t)kSmemLimit) return 2;
    if (cudaFuncSetAttribute(k_stream_test, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return 3;
    const int g = grid > 0 ? grid : tile_grid(V);
    k_stream_test<<<g, 128, smem, reinterpret_cast<cudaStream_t>(stream)>>>(m128, m16, mh, sp);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

// One CTA per SM issues `iters` groups of 4 MMAs (M = 128, N = n, K = 16)
// from resident smem operands; cycles_out[num_SMs] = cycles per group.
int njp_mma_probe(void* stream, int32_t n, int32_t iters, int32_t mode, int64_t* cycles_out) {
    if (!cycles_out || n < 16 || n > 256 || n % 16 || iters < 1) return 1;
    const size_t smem = kTileBytesA + 256 * 128 + 64 + 16;
    if (cudaFuncSetAttribute(k_mma_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return 3;
    k_mma_probe<<<num_sms(), 128, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
        n, iters, mode, reinterpret_cast<long long*>(cycles_out));
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

int njp_mma_probe_cg2(void* stream, int32_t n, int32_t iters, int32_t mode, int64_t* cycles_out) {
    if (!cycles_out || n < 32 || n > 256 || n % 16 || iters < 1) return 1;
    const size_t smem = 4 * (kTileBytesA + 128 * 128) + 64;
    if (cudaFuncSetAttribute(k_mma_probe_cg2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return 3;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((num_sms() / 2) * 2);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = reinterpret_cast<cudaStream_t>(stream);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, k_mma_probe_cg2, (int)n, (int)iters, (int)mode,
                           reinterpret_cast<long long*>(cycles_out)) != cudaSuccess)
        return 3;
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

// TMEM read bandwidth: one CTA per SM, nwarps (4..16) warps each reading its
// slice of `cols` (<= 512) columns of its lane quadrant `rounds` times with
// 32x32b.x{16,32} loads, `inflight` (1, 2, 4) per tcgen05.wait::ld.
// out[2 * SMs] = (cycles, checksum) per CTA.
int njp_tmem_bw(void* stream, int32_t nwarps, int32_t x, int32_t inflight, int32_t cols, int32_t rounds,
                int64_t* out) {
    if (!out || nwarps < 4 || nwarps > 16 || nwarps % 4 || cols < 16 || cols > 512) return 1;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    long long* o = reinterpret_cast<long long*>(out);
    const dim3 g(num_sms()), b(32 * nwarps);
#define L(X, N) k_tmem_bw<X, N><<<g, b, 0, st>>>(rounds, cols, o)
    if (x == 16 && inflight == 1) L(16, 1);
    else if (x == 16 && inflight == 2) L(16, 2);
    else if (x == 16 && inflight == 4) L(16, 4);
    else if (x == 32 && inflight == 1) L(32, 1);
    else if (x == 32 && inflight == 2) L(32, 2);
    else if (x == 32 && inflight == 4) L(32, 4);
    else return 1;
#undef L
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // extern "C"
