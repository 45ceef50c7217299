// Fused element-wise kernels of the denoising-step stack (dit.py), SURVEY
// 8(f) row 3: the per-block chains around attention and the dense FFN that
// PyTorch would run as 6-10 separate passes over (B*S, d):
//
//   ln_modulate          out = LN(x) * (1 + scale[b]) + shift[b]      (backbone.py:76-88, :559-560)
//   gate_res_ln_modulate h = x + th[b] * r;  m = LN(h) * (1 + scale[b]) (backbone.py:91-121)
//   gated_residual       out = x + th[b] * r                          (backbone.py:42-59)
//   qk_norm_rope         per (token, head): RMSNorm over d_h, then the
//                        2-axis rotary rotation with per-token tables  (tensor.py:518-531,
//                                                                       backbone.py:128-182)
// th = tanh(gate) is precomputed per (sample, channel). One warp per row,
// 16-byte vectors, fp32 statistics (two passes over the row, the second
// from L1); HBM traffic = one read of each operand and one write.
#include "common.cuh"
#include "nimg_internal.h"

namespace nimg {

template <typename T> struct V8;
template <> struct V8<bf16> { static constexpr int N = 8; };
template <> struct V8<float> { static constexpr int N = 4; };

template <typename T>
NIMG_DEV void load_vec(const T* p, float* v) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  if constexpr (sizeof(T) == 2) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      v[2 * q] = __uint_as_float(w[q] << 16);
      v[2 * q + 1] = __uint_as_float(w[q] & 0xFFFF0000u);
    }
  } else {
    v[0] = __uint_as_float(u.x); v[1] = __uint_as_float(u.y);
    v[2] = __uint_as_float(u.z); v[3] = __uint_as_float(u.w);
  }
}
template <typename T>
NIMG_DEV void store_vec(T* p, const float* v) {
  if constexpr (sizeof(T) == 2) {
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const __nv_bfloat162 b2 = __floats2bfloat162_rn(v[2 * q], v[2 * q + 1]);
      w[q] = *reinterpret_cast<const uint32_t*>(&b2);
    }
    *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  } else {
    *reinterpret_cast<uint4*>(p) = make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]),
                                              __float_as_uint(v[2]), __float_as_uint(v[3]));
  }
}

NIMG_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr int SK_WARPS = 8;

// MODE 0: ln_modulate(x) ; MODE 1: gate_res_ln_modulate ; MODE 2: gated_residual
template <typename T, int MODE>
__global__ void __launch_bounds__(SK_WARPS * 32)
row_mod_kernel(const T* __restrict__ x, const T* __restrict__ r, const float* __restrict__ th,
               const float* __restrict__ scale, const float* __restrict__ shift,
               T* __restrict__ h_out, T* __restrict__ m_out, int64_t rows, int S, int d, float eps) {
  pdl_trigger();
  pdl_wait();
  constexpr int N = V8<T>::N;
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * SK_WARPS + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int64_t b = row / S;
  const T* xr = x + row * d;
  const T* rr = MODE >= 1 ? r + row * d : nullptr;
  const float* thb = MODE >= 1 ? th + b * d : nullptr;
  T* hr = MODE >= 1 ? h_out + row * d : nullptr;
  // pass 1: (gated residual ->) row sum
  float sum = 0.f;
  for (int c = lane * N; c < d; c += 32 * N) {
    float v[N];
    load_vec<T>(xr + c, v);
    if constexpr (MODE >= 1) {
      float rv[N];
      load_vec<T>(rr + c, rv);
#pragma unroll
      for (int j = 0; j < N; ++j) v[j] = to_f32(from_f32<T>(v[j] + thb[c + j] * rv[j]));
      store_vec<T>(hr + c, v);          // the residual stream, rounded to the activation dtype
    }
#pragma unroll
    for (int j = 0; j < N; ++j) sum += v[j];
  }
  if constexpr (MODE == 2) return;
  const T* src = MODE == 1 ? hr : xr;   // a lane re-reads only what it wrote
  const float mu = warp_sum(sum) / (float)d;
  float sq = 0.f;
  for (int c = lane * N; c < d; c += 32 * N) {
    float v[N];
    load_vec<T>(src + c, v);
#pragma unroll
    for (int j = 0; j < N; ++j) { const float t = v[j] - mu; sq += t * t; }
  }
  const float inv = rsqrtf(warp_sum(sq) / (float)d + eps);
  const float* sc = scale + b * d;
  const float* sh = shift ? shift + b * d : nullptr;
  T* mr = m_out + row * d;
  for (int c = lane * N; c < d; c += 32 * N) {
    float v[N];
    load_vec<T>(src + c, v);
#pragma unroll
    for (int j = 0; j < N; ++j) {
      v[j] = (v[j] - mu) * inv * (1.f + sc[c + j]);
      if (sh) v[j] += sh[c + j];
    }
    store_vec<T>(mr + c, v);
  }
}

// One warp per (token, head) row of d_h: RMSNorm then rotary pairs.
// x: token t's heads start at x + t * xs (xs >= H * dh: a column slice of a
// fused QKV projection); out: contiguous (rows, d_h); cos/sin (S, d_h) fp32.
template <typename T>
__global__ void __launch_bounds__(SK_WARPS * 32)
qk_norm_rope_kernel(const T* x, int64_t xs, const float* __restrict__ cs,
                    const float* __restrict__ sn, T* out, int64_t rows, int S, int H, int dh,
                    float eps) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * SK_WARPS + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int64_t tok = row / H;
  const int s = (int)(tok % S);
  const T* xr = x + tok * xs + (row % H) * dh;
  T* orow = out + row * dh;
  const float* c = cs + (int64_t)s * dh;
  const float* sg = sn + (int64_t)s * dh;
  // each lane owns pairs (2p, 2p+1) for p = lane, lane + 32, ...
  float sq = 0.f;
  for (int p = lane; 2 * p < dh; p += 32) {
    const float a = to_f32(xr[2 * p]), bb = to_f32(xr[2 * p + 1]);
    sq += a * a + bb * bb;
  }
  const float inv = rsqrtf(warp_sum(sq) / (float)dh + eps);
  for (int p = lane; 2 * p < dh; p += 32) {
    const float a = to_f32(xr[2 * p]) * inv, bb = to_f32(xr[2 * p + 1]) * inv;
    // rotate_pairs: (x0, x1) -> (-x1, x0)
    orow[2 * p] = from_f32<T>(a * c[2 * p] - bb * sg[2 * p]);
    orow[2 * p + 1] = from_f32<T>(bb * c[2 * p + 1] + a * sg[2 * p + 1]);
  }
}

template <typename T, int MODE>
static cudaError_t launch_row_mod(const void* x, const void* r, const float* th, const float* scale,
                                  const float* shift, void* h, void* m, int64_t rows, int S, int d,
                                  float eps, cudaStream_t s) {
  const unsigned grid = (unsigned)((rows + SK_WARPS - 1) / SK_WARPS);
  return launch_pdl(row_mod_kernel<T, MODE>, dim3(grid), dim3(SK_WARPS * 32), 0, s,
                    (const T*)x, (const T*)r, th, scale, shift, (T*)h, (T*)m, rows, S, d, eps);
}

cudaError_t launch_row_modulate(int mode, bool bf, const void* x, const void* r, const float* th,
                                const float* scale, const float* shift, void* h, void* m,
                                int64_t rows, int S, int d, float eps, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
#define NIMG_RM(T)                                                                          \
  (mode == 0 ? launch_row_mod<T, 0>(x, r, th, scale, shift, h, m, rows, S, d, eps, s)     \
   : mode == 1 ? launch_row_mod<T, 1>(x, r, th, scale, shift, h, m, rows, S, d, eps, s)   \
               : launch_row_mod<T, 2>(x, r, th, scale, shift, h, m, rows, S, d, eps, s))
  return bf ? NIMG_RM(bf16) : NIMG_RM(float);
#undef NIMG_RM
}

cudaError_t launch_qk_norm_rope(bool bf, const void* x, int64_t xs, const float* cs, const float* sn,
                                void* out, int64_t rows, int S, int H, int dh, float eps,
                                cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  const unsigned grid = (unsigned)((rows + SK_WARPS - 1) / SK_WARPS);
  if (bf)
    return launch_pdl(qk_norm_rope_kernel<bf16>, dim3(grid), dim3(SK_WARPS * 32), 0, s,
                      (const bf16*)x, xs, cs, sn, (bf16*)out, rows, S, H, dh, eps);
  return launch_pdl(qk_norm_rope_kernel<float>, dim3(grid), dim3(SK_WARPS * 32), 0, s,
                    (const float*)x, xs, cs, sn, (float*)out, rows, S, H, dh, eps);
}

}  // namespace nimg
