// fp32 mode on the bf16 tensor cores ("bf16x3"): operand splits.
//
// An fp32 value a is split into bf16 pieces a1 = bf16(a), a2 = bf16(a - a1)
// (|a - a1 - a2| <= 2^-16 |a|). With activations laid out as A' = [a1 | a1 | a2]
// and weights as W' = [w1 | w2 | w1] along the reduction axis (K' = 3K),
//   A' W'^T = a1 w1 + a1 w2 + a2 w1  =  a w  -  O(2^-16 |a w|)
// so the unchanged bf16 tcgen05 grouped GEMM (fp32 TMEM accumulation) computes
// the fp32 expert GEMMs to ~4e-6 relative (the dropped terms a2 w2, a1 w3, ...),
// inside the fp32 mode's 1e-4 bar, at a third of the bf16 rate instead of the
// CUDA-core fp32 kernel's. GEMM1 writes `pre` split the same way (its
// epilogue, bank flag kSplit3Out); GEMM2 writes fp32 rows (kF32Out).
#include "common.cuh"
#include "nimg_internal.h"

namespace nimg {

NIMG_DEV void split2(float a, bf16& hi, bf16& lo) {
  hi = __float2bfloat16_rn(a);
  lo = __float2bfloat16_rn(a - __bfloat162float(hi));
}

// dst[r] = pattern(src[idx ? idx[r] : r]) : pattern 0 (activations) writes
// [hi | hi | lo], pattern 1 (weights) [hi | lo | hi]; K % 8 == 0.
// Row per block-y, 8 columns per thread.
__global__ void __launch_bounds__(256)
split3_rows_kernel(const float* __restrict__ src, const int32_t* __restrict__ idx, bf16* __restrict__ dst,
                   int64_t rows, int K, int pattern) {
  pdl_trigger();
  pdl_wait();
  const int64_t r = blockIdx.y + (int64_t)gridDim.y * blockIdx.z;
  if (r >= rows) return;
  const float* s = src + (idx ? (int64_t)idx[r] : r) * K;
  bf16* d = dst + r * (int64_t)(3 * K);
  for (int k = (blockIdx.x * blockDim.x + threadIdx.x) * 8; k < K; k += gridDim.x * blockDim.x * 8) {
    const float4 v0 = *reinterpret_cast<const float4*>(s + k);
    const float4 v1 = *reinterpret_cast<const float4*>(s + k + 4);
    const float f[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
    __align__(16) bf16 hi[8], lo[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) split2(f[i], hi[i], lo[i]);
    const uint4 H = *reinterpret_cast<const uint4*>(hi), L = *reinterpret_cast<const uint4*>(lo);
    *reinterpret_cast<uint4*>(d + k) = H;
    *reinterpret_cast<uint4*>(d + K + k) = pattern ? L : H;
    *reinterpret_cast<uint4*>(d + 2 * K + k) = pattern ? H : L;
  }
}

cudaError_t launch_split3_rows(const float* src, const int32_t* idx, void* dst, int64_t rows, int K,
                               int pattern, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  const int per_block = 256 * 8;
  const unsigned gx = (unsigned)((K + per_block - 1) / per_block);
  const int64_t gy = rows < 65535 ? rows : 65535;
  const int64_t gz = (rows + gy - 1) / gy;
  return launch_pdl(split3_rows_kernel, dim3(gx, (unsigned)gy, (unsigned)gz), dim3(256), 0, s, src, idx,
                    static_cast<bf16*>(dst), rows, K, pattern);
}

}  // namespace nimg
