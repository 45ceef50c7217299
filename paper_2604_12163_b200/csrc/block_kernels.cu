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

// th_* in f64 for the fp32 (reference-exact) chain and rounded to fp32 for
// the bf16 path, which computes in fp32.
__global__ void block_modvec_kernel(const float* __restrict__ sa_gate,
                                    const float* __restrict__ ff_scale,
                                    const float* __restrict__ ff_gate, double* __restrict__ th_sa,
                                    double* __restrict__ th_ff, float* __restrict__ onep,
                                    float* __restrict__ th_sa_f, float* __restrict__ th_ff_f,
                                    int64_t n) {
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double a = tanh((double)sa_gate[i]), g = tanh((double)ff_gate[i]);
  th_sa[i] = a;
  th_ff[i] = g;
  th_sa_f[i] = (float)a;
  th_ff_f[i] = (float)g;
  onep[i] = (float)((double)ff_scale[i] + 1.0);   // add(ff_scale, 1.0): as_tensor(1.0) -> fp32
}

// bf16 storage: the same op sequence in fp32 registers (no f64 chain -- the
// bf16 mode's bar is tolerance + bit-exact routing of the x_norm produced).
constexpr int BPF_WARPS = 8;
__global__ void __launch_bounds__(BPF_WARPS * 32)
block_prologue_bf16_kernel(const bf16* __restrict__ x, const bf16* __restrict__ r_attn,
                           const float* __restrict__ th_sa, const float* __restrict__ onep,
                           bf16* __restrict__ h_out, bf16* __restrict__ xn_out,
                           bf16* __restrict__ xm_out, int64_t T_tok, int S, int d, float scale_t) {
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * BPF_WARPS + warp;
  if (t >= T_tok) return;
  const int64_t b = t / S;
  const bf16* xr = x + t * d;
  const bf16* rr = r_attn + t * d;
  const float* ths = th_sa + b * d;
  const float* op = onep + b * d;
  constexpr int MAXV = 8;                       // up to 8 x 16-B vectors per lane (d <= 2048)
  float hf[MAXV][8];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < MAXV; ++k) {
    const int c0 = (k * 32 + lane) * 8;
    if (c0 < d) {
      const uint4 xv = __ldg(reinterpret_cast<const uint4*>(xr + c0));
      const uint4 rv = __ldg(reinterpret_cast<const uint4*>(rr + c0));
      const bf16* xe = reinterpret_cast<const bf16*>(&xv);
      const bf16* re = reinterpret_cast<const bf16*>(&rv);
      float g[8];   // per-sample gate: two 16-B loads instead of eight scalar ones
      *reinterpret_cast<float4*>(g) = __ldg(reinterpret_cast<const float4*>(ths + c0));
      *reinterpret_cast<float4*>(g + 4) = __ldg(reinterpret_cast<const float4*>(ths + c0) + 1);
      bf16 hv[8];
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        hv[v] = __float2bfloat16_rn(__fadd_rn(__bfloat162float(xe[v]),
                                              __fmul_rn(g[v], __bfloat162float(re[v]))));
        hf[k][v] = __bfloat162float(hv[v]);
        ss = fmaf(hf[k][v], hf[k][v], ss);
      }
      *reinterpret_cast<uint4*>(h_out + t * d + c0) = *reinterpret_cast<const uint4*>(hv);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float inv = rsqrtf(ss / (float)d + 1e-6f);
#pragma unroll
  for (int k = 0; k < MAXV; ++k) {
    const int c0 = (k * 32 + lane) * 8;
    if (c0 < d) {
      bf16 xn[8], xm[8];
      float o1[8];
      *reinterpret_cast<float4*>(o1) = __ldg(reinterpret_cast<const float4*>(op + c0));
      *reinterpret_cast<float4*>(o1 + 4) = __ldg(reinterpret_cast<const float4*>(op + c0) + 1);
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const float xn0 = __bfloat162float(__float2bfloat16_rn(hf[k][v] * inv));
        xn[v] = __float2bfloat16_rn(xn0 * scale_t);
        xm[v] = __float2bfloat16_rn(__bfloat162float(xn[v]) * o1[v]);
      }
      *reinterpret_cast<uint4*>(xn_out + t * d + c0) = *reinterpret_cast<const uint4*>(xn);
      *reinterpret_cast<uint4*>(xm_out + t * d + c0) = *reinterpret_cast<const uint4*>(xm);
    }
  }
}

// bf16, block per token: thread c owns the 8 elements [8c, 8c+8) (d / 8
// threads, d <= 8192); the sum of squares is reduced lane-sequentially, over
// the warp (xor tree) and over the warps in index order. No 64-float row in
// registers, so many tokens are in flight per SM (the warp-per-token kernel
// above keeps a whole row per warp).
__global__ void block_prologue_bf16_blk_kernel(const bf16* __restrict__ x, const bf16* __restrict__ r_attn,
                                               const float* __restrict__ th_sa, const float* __restrict__ onep,
                                               bf16* __restrict__ h_out, bf16* __restrict__ xn_out,
                                               bf16* __restrict__ xm_out, int S, int d, float scale_t) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[32];
  const int64_t t = blockIdx.x;
  const int c = threadIdx.x, lane = c & 31, warp = c >> 5, nw = blockDim.x >> 5;
  const int64_t b = t / S;
  const int64_t o = t * d + (int64_t)c * 8;
  const uint4 xv = __ldg(reinterpret_cast<const uint4*>(x + o));
  const uint4 rv = __ldg(reinterpret_cast<const uint4*>(r_attn + o));
  float g[8], o1[8];
  *reinterpret_cast<float4*>(g) = __ldg(reinterpret_cast<const float4*>(th_sa + b * d + c * 8));
  *reinterpret_cast<float4*>(g + 4) = __ldg(reinterpret_cast<const float4*>(th_sa + b * d + c * 8) + 1);
  *reinterpret_cast<float4*>(o1) = __ldg(reinterpret_cast<const float4*>(onep + b * d + c * 8));
  *reinterpret_cast<float4*>(o1 + 4) = __ldg(reinterpret_cast<const float4*>(onep + b * d + c * 8) + 1);
  const bf16* xe = reinterpret_cast<const bf16*>(&xv);
  const bf16* re = reinterpret_cast<const bf16*>(&rv);
  bf16 hv[8];
  float hf[8], ss = 0.f;
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    hv[v] = __float2bfloat16_rn(__fadd_rn(__bfloat162float(xe[v]), __fmul_rn(g[v], __bfloat162float(re[v]))));
    hf[v] = __bfloat162float(hv[v]);
    ss = fmaf(hf[v], hf[v], ss);
  }
  *reinterpret_cast<uint4*>(h_out + o) = *reinterpret_cast<const uint4*>(hv);
#pragma unroll
  for (int k = 16; k > 0; k >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, k);
  if (lane == 0) red[warp] = ss;
  __syncthreads();
  float tot = red[0];
  for (int w = 1; w < nw; ++w) tot += red[w];
  const float inv = rsqrtf(tot / (float)d + 1e-6f);
  bf16 xn[8], xm[8];
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    const float xn0 = __bfloat162float(__float2bfloat16_rn(hf[v] * inv));
    xn[v] = __float2bfloat16_rn(xn0 * scale_t);
    xm[v] = __float2bfloat16_rn(__bfloat162float(xn[v]) * o1[v]);
  }
  *reinterpret_cast<uint4*>(xn_out + o) = *reinterpret_cast<const uint4*>(xn);
  *reinterpret_cast<uint4*>(xm_out + o) = *reinterpret_cast<const uint4*>(xm);
}

static bool bp_block() {
  static const bool on = [] {
    const char* e = getenv("NIMG_BP_BLOCK");
    return !(e && e[0] == '0');
  }();
  return on;
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
  pdl_trigger();
  pdl_wait();
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
  T* hr = h_out + t * d;
  const float* op = onep + b * d;
  constexpr int VEC = 16 / sizeof(T);           // elements per 16-B vector
  const bool vec = (d % (32 * VEC) == 0);
  // pass 1: h (rounded to storage), squares to smem. numpy rounds the product
  // and the sum separately: no FMA contraction (__dmul_rn / __dadd_rn).
  if (vec) {
#pragma unroll 4
    for (int c0 = lane * VEC; c0 < d; c0 += 32 * VEC) {
      const uint4 xv = __ldg(reinterpret_cast<const uint4*>(xr + c0));
      const uint4 rv = __ldg(reinterpret_cast<const uint4*>(rr + c0));
      const T* xe = reinterpret_cast<const T*>(&xv);
      const T* re = reinterpret_cast<const T*>(&rv);
      T hv[VEC];
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        hv[v] = from_f32<T>((float)__dadd_rn((double)to_f32(xe[v]),
                                             __dmul_rn(ths[c0 + v], (double)to_f32(re[v]))));
        const double hd = (double)to_f32(hv[v]);
        const int j = c0 + v;
        sq[(j >> 7) * 129 + (j & 127)] = hd * hd;
      }
      *reinterpret_cast<uint4*>(hr + c0) = *reinterpret_cast<const uint4*>(hv);
    }
  } else {
    for (int j = lane; j < d; j += 32) {
      const T hv = from_f32<T>((float)__dadd_rn((double)to_f32(xr[j]), __dmul_rn(ths[j], (double)to_f32(rr[j]))));
      hr[j] = hv;
      const double hd = (double)to_f32(hv);
      sq[(j >> 7) * 129 + (j & 127)] = hd * hd;
    }
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
  if (vec) {
#pragma unroll 4
    for (int c0 = lane * VEC; c0 < d; c0 += 32 * VEC) {
      const uint4 hv4 = *reinterpret_cast<const uint4*>(hr + c0);
      const T* he = reinterpret_cast<const T*>(&hv4);
      T xn[VEC], xm[VEC];
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const T xn0 = from_f32<T>((float)((double)to_f32(he[v]) * inv));     // rmsnorm -> dtype
        xn[v] = from_f32<T>((float)((double)to_f32(xn0) * sc));              // * as_tensor(scale)
        xm[v] = from_f32<T>((float)((double)to_f32(xn[v]) * (double)op[c0 + v]));  // * (1+ff_scale)
      }
      *reinterpret_cast<uint4*>(xn_out + t * d + c0) = *reinterpret_cast<const uint4*>(xn);
      *reinterpret_cast<uint4*>(xm_out + t * d + c0) = *reinterpret_cast<const uint4*>(xm);
    }
  } else {
    for (int j = lane; j < d; j += 32) {
      const double hd = (double)to_f32(hr[j]);
      const T xn0 = from_f32<T>((float)(hd * inv));
      const T xn = from_f32<T>((float)((double)to_f32(xn0) * sc));
      xn_out[t * d + j] = xn;
      xm_out[t * d + j] = from_f32<T>((float)((double)to_f32(xn) * (double)op[j]));
    }
  }
}

cudaError_t launch_block_modvec(const float* sa_gate, const float* ff_scale, const float* ff_gate,
                                double* th_sa, double* th_ff, float* onep, float* th_sa_f,
                                float* th_ff_f, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  block_modvec_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(sa_gate, ff_scale, ff_gate, th_sa,
                                                                   th_ff, onep, th_sa_f, th_ff_f, n);
  return cudaGetLastError();
}

cudaError_t launch_block_prologue(bool bf, const void* x, const void* r_attn, const double* th_sa,
                                  const float* th_sa_f, const float* onep, void* h, void* xn,
                                  void* xm, int64_t T, int S, int d, float scale_t, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  if (bf && bp_block() && d % 256 == 0 && d <= 8192)
    return launch_pdl(block_prologue_bf16_blk_kernel, dim3((unsigned)T), dim3(d / 8), 0, s,
                      (const bf16*)x, (const bf16*)r_attn, th_sa_f, onep, (bf16*)h, (bf16*)xn,
                      (bf16*)xm, S, d, scale_t);
  if (bf && d % 256 == 0 && d <= 2048) {
    return launch_pdl(block_prologue_bf16_kernel, dim3((unsigned)((T + BPF_WARPS - 1) / BPF_WARPS)),
                      dim3(BPF_WARPS * 32), 0, s, (const bf16*)x, (const bf16*)r_attn, th_sa_f, onep,
                      (bf16*)h, (bf16*)xn, (bf16*)xm, T, S, d, scale_t);
  }
  const int nleaf = (d + 127) / 128;
  const int balanced = (d % 128 == 0) && nleaf <= 32 && (nleaf & (nleaf - 1)) == 0;
  const size_t smem = (size_t)BP_WARPS * nleaf * 129 * 8;
  const unsigned grid = (unsigned)((T + BP_WARPS - 1) / BP_WARPS);
  cudaError_t e;
  if (bf) {
    e = cudaFuncSetAttribute(block_prologue_kernel<bf16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = launch_pdl(block_prologue_kernel<bf16>, dim3(grid), dim3(BP_WARPS * 32), smem, s,
                   (const bf16*)x, (const bf16*)r_attn, th_sa, onep, (bf16*)h, (bf16*)xn, (bf16*)xm,
                   T, S, d, scale_t, balanced);
  } else {
    e = cudaFuncSetAttribute(block_prologue_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = launch_pdl(block_prologue_kernel<float>, dim3(grid), dim3(BP_WARPS * 32), smem, s,
                   (const float*)x, (const float*)r_attn, th_sa, onep, (float*)h, (float*)xn,
                   (float*)xm, T, S, d, scale_t, balanced);
  }
  return e;
}

}  // namespace nimg
