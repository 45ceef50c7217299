// The backbone's MoE branch around the layer:
//
//   h      = x + tanh(sa_gate) * r_attn                       backbone.py:584, 42-59
//   x_norm = rmsnorm(h) * (1/sqrt(layer+1))                   backbone.py:585-586, tensor.py:518-531
//   x_mod  = x_norm * (1 + ff_scale)                          backbone.py:587-589
//   ...layer...  moe = moe_forward(h, x_norm, x_mod, t_vec)   backbone.py:595-597
//   x_out  = h + tanh(ff_gate) * moe                          backbone.py:606
//
// block_modvec: per-sample f64 tanh of the two gates and fp32(1 + ff_scale).
// block_prologue: warp per token, one pass over x and r_attn producing h,
// x_norm and x_mod with the reference's per-op rounding chain (f64 compute,
// round to storage dtype), including numpy's pairwise order for the
// mean of squares. The x_out residual is fused into the combine kernel.
#include "common.cuh"
#include "nimg_internal.h"

namespace nimg {

__global__ void block_modvec_kernel(const float* __restrict__ sa_gate,
                                    const float* __restrict__ ff_scale,
                                    const float* __restrict__ ff_gate, double* __restrict__ th_sa,
                                    double* __restrict__ th_ff, float* __restrict__ onep,
                                    int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  th_sa[i] = tanh((double)sa_gate[i]);
  th_ff[i] = tanh((double)ff_gate[i]);
  onep[i] = (float)((double)ff_scale[i] + 1.0);   // add(ff_scale, 1.0): as_tensor(1.0) -> fp32
}

constexpr int BP_WARPS = 4;

// squares staged per warp in leaf-padded smem: leaf l (128 elements) at
// l * 129 doubles, so lane l reading its leaf is bank-conflict free.
template <typename T>
__global__ void __launch_bounds__(BP_WARPS * 32)
block_prologue_kernel(const T* __restrict__ x, const T* __restrict__ r_attn,
                      const double* __restrict__ th_sa, const float* __restrict__ onep,
                      T* __restrict__ h_out, T* __restrict__ xn_out, T* __restrict__ xm_out,
                      int64_t T_tok, int S, int d, float scale_t, int balanced) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nleaf = (d + 127) / 128;
  double* sq = reinterpret_cast<double*>(sm) + (size_t)warp * nleaf * 129;
  const int64_t t = (int64_t)blockIdx.x * BP_WARPS + warp;
  if (t >= T_tok) return;
  const int64_t b = t / S;
  const T* xr = x + t * d;
  const T* rr = r_attn + t * d;
  const double* ths = th_sa + b * d;
  // pass 1: h (rounded to storage), squares to smem
  for (int j = lane; j < d; j += 32) {
    // numpy rounds the product and the sum separately: no FMA contraction
    const T hv = from_f32<T>((float)__dadd_rn((double)to_f32(xr[j]), __dmul_rn(ths[j], (double)to_f32(rr[j]))));
    h_out[t * d + j] = hv;
    const double hd = (double)to_f32(hv);
    sq[(j >> 7) * 129 + (j & 127)] = hd * hd;
  }
  __syncwarp();
  double sum;
  if (balanced) {
    // d = 128 * 2^k (<= 4096): numpy's recursion bottoms out in 2^k equal
    // leaves of 128 and folds them as a balanced tree == an xor-shuffle tree.
    double v = 0.0;
    if (lane < nleaf) v = np_pairwise_sum(sq + lane * 129, 128);
    for (int o = 1; o < nleaf; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    sum = __shfl_sync(0xffffffffu, v, 0);
  } else {
    // general d: lane 0 walks numpy's recursion over a contiguous copy
    double s0 = 0.0;
    if (lane == 0) {
      // compact the padded leaves in place (leaf l starts at l*129 -> l*128)
      for (int l = 1; l < nleaf; ++l)
        for (int i = 0; i < 128 && l * 128 + i < d; ++i) sq[l * 128 + i] = sq[l * 129 + i];
      s0 = np_pairwise_sum(sq, d);
    }
    sum = __shfl_sync(0xffffffffu, s0, 0);
  }
  const double inv = 1.0 / sqrt(sum / (double)d + 1e-6);    // tensor.py:527-528
  const double sc = (double)scale_t;
  const float* op = onep + b * d;
  for (int j = lane; j < d; j += 32) {
    const double hd = (double)to_f32(h_out[t * d + j]);
    const T xn0 = from_f32<T>((float)(hd * inv));                         // rmsnorm -> dtype
    const T xn = from_f32<T>((float)((double)to_f32(xn0) * sc));          // * fp32(scale)
    xn_out[t * d + j] = xn;
    xm_out[t * d + j] = from_f32<T>((float)((double)to_f32(xn) * (double)op[j]));  // * (1+ff_scale)
  }
}

cudaError_t launch_block_modvec(const float* sa_gate, const float* ff_scale, const float* ff_gate,
                                double* th_sa, double* th_ff, float* onep, int64_t n,
                                cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  block_modvec_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(sa_gate, ff_scale, ff_gate, th_sa,
                                                                   th_ff, onep, n);
  return cudaGetLastError();
}

cudaError_t launch_block_prologue(bool bf, const void* x, const void* r_attn, const double* th_sa,
                                  const float* onep, void* h, void* xn, void* xm, int64_t T, int S,
                                  int d, float scale_t, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  const int nleaf = (d + 127) / 128;
  const int balanced = (d % 128 == 0) && nleaf <= 32 && (nleaf & (nleaf - 1)) == 0;
  const size_t smem = (size_t)BP_WARPS * nleaf * 129 * 8;
  const unsigned grid = (unsigned)((T + BP_WARPS - 1) / BP_WARPS);
  cudaError_t e;
  if (bf) {
    e = cudaFuncSetAttribute(block_prologue_kernel<bf16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    block_prologue_kernel<bf16><<<grid, BP_WARPS * 32, smem, s>>>(
        (const bf16*)x, (const bf16*)r_attn, th_sa, onep, (bf16*)h, (bf16*)xn, (bf16*)xm, T, S, d,
        scale_t, balanced);
  } else {
    e = cudaFuncSetAttribute(block_prologue_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    block_prologue_kernel<float><<<grid, BP_WARPS * 32, smem, s>>>(
        (const float*)x, (const float*)r_attn, th_sa, onep, (float*)h, (float*)xn, (float*)xm, T,
        S, d, scale_t, balanced);
  }
  return cudaGetLastError();
}

}  // namespace nimg
