// CUDA-core grouped SwiGLU GEMMs (fp32 accumulate, no TF32).
//
// Used for the fp32 parity mode (the reference computes experts in f64 and
// rounds to fp32, moe.py:42-51; this path keeps rel-err ~1e-6, inside the
// north star's 1e-4 bar) and for shapes the TMA path cannot take (d or h not
// a multiple of 16, e.g. the reference's tiny unit-test shapes). Same
// segment/bank tables as the tensor-core kernel.
//   MODE 0: pre[r, n] = SiLU(x W1^T) * (x W3^T)  (fp32 out)
//   MODE 1: y[r, n]   = pre W2^T                  (fp32 out; `pre` is fp32)
// The f64 storage mode (f64_kernels.cu) instantiates the same kernel with f64
// operands, accumulators and outputs (ACC = double), as the reference's
// swiglu computes with an f64 `pre` that is never rounded (moe.py:42-51).
#include "common.cuh"
#include "nimg_internal.h"

namespace nimg {
namespace simt {

constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

template <typename ACC, typename T> NIMG_DEV ACC to_acc(T v) { return (ACC)to_f32(v); }
template <> NIMG_DEV double to_acc<double, double>(double v) { return v; }
NIMG_DEV float silu_mul(float v, float g) { return v / (1.0f + expf(-v)) * g; }
// moe.py:45-48: h1 * (1 / (1 + exp(-h1))) * h3 in f64
NIMG_DEV double silu_mul(double v, double g) { return v * (1.0 / (1.0 + exp(-v))) * g; }

template <int MODE, typename TA, typename TW, typename ACC = float>
__global__ void __launch_bounds__(NT) grouped_simt_kernel(const __grid_constant__ SimtParams p) {
  __shared__ ACC As[BK][BM + 4];
  __shared__ ACC Bs[BK][BN + 4];
  __shared__ ACC B3s[MODE == 0 ? BK : 1][BN + 4];

  const int t = blockIdx.x;
  int lo = 0, hi = p.nseg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (p.seg_tile0[mid] <= t) lo = mid; else hi = mid - 1;
  }
  const int bank = lo >= p.nseg0 ? 1 : 0;
  const SimtBank& bk = p.bank[bank];
  const int local = t - p.seg_tile0[lo];
  const int m_blk = local / bk.ntn, n_blk = local % bk.ntn;
  const int row0 = p.seg_row0[lo] + m_blk * BM;
  const int rows = min(BM, p.seg_rows[lo] - m_blk * BM);
  const int n0 = n_blk * BN;
  const int64_t e = p.seg_expert[lo];
  const TA* A = reinterpret_cast<const TA*>(bk.a);
  const TW* W = reinterpret_cast<const TW*>(bk.w) + e * (int64_t)bk.N * bk.K;
  const TW* W3 = MODE == 0 ? reinterpret_cast<const TW*>(bk.w3) + e * (int64_t)bk.N * bk.K : nullptr;

  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  ACC acc[4][4], acc3[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) { acc[i][j] = ACC(0); acc3[i][j] = ACC(0); }

  for (int k0 = 0; k0 < bk.K; k0 += BK) {
    for (int i = threadIdx.x; i < BM * BK; i += NT) {
      const int r = i / BK, kk = i % BK;
      ACC v = ACC(0);
      if (r < rows && k0 + kk < bk.K) v = to_acc<ACC>(A[(int64_t)(row0 + r) * bk.a_ld + k0 + kk]);
      As[kk][r] = v;
    }
    for (int i = threadIdx.x; i < BN * BK; i += NT) {
      const int c = i / BK, kk = i % BK;
      ACC v = ACC(0), v3 = ACC(0);
      if (n0 + c < bk.N && k0 + kk < bk.K) {
        const int64_t off = (int64_t)(n0 + c) * bk.K + k0 + kk;
        v = to_acc<ACC>(W[off]);
        if (MODE == 0) v3 = to_acc<ACC>(W3[off]);
      }
      Bs[kk][c] = v;
      if (MODE == 0) B3s[kk][c] = v3;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      ACC a[4], b[4], b3[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        b[j] = Bs[kk][tx * 4 + j];
        if (MODE == 0) b3[j] = B3s[kk][tx * 4 + j];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[i][j] = fma(a[i], b[j], acc[i][j]);
          if (MODE == 0) acc3[i][j] = fma(a[i], b3[j], acc3[i][j]);
        }
    }
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = ty * 4 + i;
    if (r >= rows) continue;
    ACC* o = static_cast<ACC*>(bk.out) + (int64_t)(row0 + r) * bk.out_ld;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = n0 + tx * 4 + j;
      if (c >= bk.N) continue;
      ACC v = acc[i][j];
      if (MODE == 0) {
        if (sizeof(ACC) == 4 && bk.h_out != nullptr) {   // training forward: keep h1 | h3
          float* hrow = bk.h_out + (int64_t)(row0 + r) * (2 * bk.N);
          hrow[c] = (float)v;
          hrow[bk.N + c] = (float)acc3[i][j];
        }
        v = silu_mul(v, acc3[i][j]);
      }
      o[c] = v;
    }
  }
}

}  // namespace simt

int simt_bm() { return simt::BM; }
int simt_bn() { return simt::BN; }

cudaError_t launch_grouped_simt(int mode, bool in_bf16, const SimtParams& p, cudaStream_t stream,
                                bool f64) {
  if (p.total_tiles <= 0) return cudaSuccess;
  const int grid = p.total_tiles;
  if (f64) {
    if (mode == 0) simt::grouped_simt_kernel<0, double, double, double><<<grid, simt::NT, 0, stream>>>(p);
    else simt::grouped_simt_kernel<1, double, double, double><<<grid, simt::NT, 0, stream>>>(p);
    return cudaGetLastError();
  }
  if (mode == 0) {
    if (in_bf16) simt::grouped_simt_kernel<0, bf16, bf16><<<grid, simt::NT, 0, stream>>>(p);
    else simt::grouped_simt_kernel<0, float, float><<<grid, simt::NT, 0, stream>>>(p);
  } else {
    if (in_bf16) simt::grouped_simt_kernel<1, float, bf16><<<grid, simt::NT, 0, stream>>>(p);
    else simt::grouped_simt_kernel<1, float, float><<<grid, simt::NT, 0, stream>>>(p);
  }
  return cudaGetLastError();
}

}  // namespace nimg
