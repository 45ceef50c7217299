// The reference's float64 storage mode on the GPU (act_dtype == NIMG_F64).
//
// The reference stores float64 end to end under NIMG_VERIFY=1 /
// set_default_dtype(float64) (tensor.py:39-47), and its backbone promotes the
// MoE inputs to float64 even in the float32 mode (sinusoidal_features and RoPE
// multiply by f64 constants, backbone.py:259-261, :176-177): route_full then
// keeps f64 logits, scores and gates (router.py:120-143) and swiglu returns
// f64 (moe.py:42-51). Rounding every intermediate to fp32 would change which
// tokens win near-ties, so this mode keeps every value in f64:
//
//   router_logits_f64   [x_norm | t_emb] W_r as one f64 dot over 2d per
//                       (token, expert)                     router.py:120-122
//   softmax_f64         max-subtract, exp, numpy pairwise sum, divide
//                                                           tensor.py:467-473
//   select_f64          per (sample, expert) column: stable descending order
//                       of the f64 scores, NaN last, ties by lower token index
//                       (argsort(-x, kind="stable")[:cap])  router.py:98-101
//   gates_f64           expert-ascending f64 totals (np.add.at order), then
//                       raw / (tot + eps) * alpha           router.py:137-143
//   combine_f64         0 + sum_e (y * gate) in expert-ascending order, + shared
//                                                moe.py:156-161, tensor.py:366-378
//
// The expert GEMMs run the CUDA-core grouped kernel with f64 operands and
// accumulators (grouped_gemm_simt.cu). Only the f64 summation order differs
// from OpenBLAS, so values agree to ~1e-15 relative; a selection can differ
// from the reference only where two f64 scores tie to within that.
#include "common.cuh"
#include "nimg_internal.h"

namespace nimg {
namespace f64m {

template <typename T> NIMG_DEV double ld64(const T* p, int64_t i);
template <> NIMG_DEV double ld64<double>(const double* p, int64_t i) { return p[i]; }
template <> NIMG_DEV double ld64<float>(const float* p, int64_t i) { return (double)p[i]; }

// ---- logits: L[t, e] = sum_{k < 2d} A[t, k] W[k, e], A = [x_norm[t] | t_emb[t / S]]
constexpr int LBM = 64, LBN = 64, LBK = 16, LNT = 256;
__global__ void __launch_bounds__(LNT)
router_logits_f64_kernel(const double* __restrict__ x, const double* __restrict__ t_emb,
                         const double* __restrict__ w, double* __restrict__ logits, int64_t T,
                         int S, int d, int E) {
  __shared__ double As[LBK][LBM + 1];
  __shared__ double Bs[LBK][LBN + 1];
  const int64_t m0 = (int64_t)blockIdx.x * LBM;
  const int n0 = blockIdx.y * LBN;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  const int K = 2 * d;
  for (int k0 = 0; k0 < K; k0 += LBK) {
    for (int i = threadIdx.x; i < LBM * LBK; i += LNT) {
      const int r = i / LBK, kk = i % LBK;
      const int64_t t = m0 + r;
      const int k = k0 + kk;
      double v = 0.0;
      if (t < T && k < K) v = k < d ? x[t * d + k] : t_emb[(t / S) * d + (k - d)];
      As[kk][r] = v;
    }
    for (int i = threadIdx.x; i < LBN * LBK; i += LNT) {
      const int kk = i / LBN, c = i % LBN;
      const int k = k0 + kk;
      Bs[kk][c] = (k < K && n0 + c < E) ? w[(int64_t)k * E + n0 + c] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < LBK; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t t = m0 + ty * 4 + i;
    if (t >= T) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int e = n0 + tx * 4 + j;
      if (e < E) logits[t * E + e] = acc[i][j];
    }
  }
}

// ---- softmax over E per token (tensor.py:467-473), warp per token; writes the
// scores expert-major (B, E, S) for the per-column selection.
constexpr int SM_WARPS = 8;
__global__ void __launch_bounds__(SM_WARPS * 32)
softmax_f64_kernel(const double* __restrict__ logits, double* __restrict__ scores_bes, int64_t T,
                   int S, int E) {
  extern __shared__ double sm_e[];   // SM_WARPS * E
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t t = (int64_t)blockIdx.x * SM_WARPS + warp;
  if (t >= T) return;
  double* ev = sm_e + warp * E;
  const double* l = logits + t * E;
  double m = -INFINITY;
  bool nan = false;
  for (int e = lane; e < E; e += 32) {
    const double v = l[e];
    nan |= v != v;
    m = fmax(m, v);
  }
  for (int o = 16; o; o >>= 1) {
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    nan |= __shfl_xor_sync(0xffffffffu, (int)nan, o) != 0;
  }
  if (nan) m = __longlong_as_double(0x7ff8000000000000ll);  // numpy max propagates NaN
  for (int e = lane; e < E; e += 32) ev[e] = exp(l[e] - m);
  __syncwarp();
  double sum = 0.0;
  if (lane == 0) sum = np_pairwise_sum(ev, E);
  sum = __shfl_sync(0xffffffffu, sum, 0);
  const int64_t b = t / S, s = t % S;
  for (int e = lane; e < E; e += 32) scores_bes[(b * E + e) * S + s] = ev[e] / sum;
}

// ---- per (sample, expert) column: top-cap of S f64 scores in the order of
// argsort(-x, kind="stable"): descending, NaN last, ties (incl. -0 == +0) by
// ascending token index. One CTA per column; bitonic sort of (key, index) in
// shared memory (S <= 16384).
NIMG_DEV uint64_t desc_key(double v) {
  if (v != v) return 0ull;                    // NaN ranks after everything
  if (v == 0.0) v = 0.0;                      // -0 == +0
  const uint64_t b = (uint64_t)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);   // larger value -> larger key
}
// a before b: larger key first, then lower index
NIMG_DEV bool before(uint64_t ka, int ia, uint64_t kb, int ib) {
  return ka > kb || (ka == kb && ia < ib);
}

__global__ void __launch_bounds__(1024)
select_f64_kernel(const double* __restrict__ scores_bes, int32_t* __restrict__ token_flat,
                  double* __restrict__ gate_raw, int16_t* __restrict__ slot_of, int B, int S, int E,
                  int cap, int n) {
  extern __shared__ uint64_t sel_sm[];
  uint64_t* key = sel_sm;
  int* idx = reinterpret_cast<int*>(sel_sm + n);
  const int col = blockIdx.x;   // b * E + e
  const int b = col / E, e = col % E;
  const double* sc = scores_bes + (int64_t)col * S;
  int16_t* slot = slot_of + (int64_t)col * S;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    key[i] = i < S ? desc_key(sc[i]) : 0ull;
    idx[i] = i;   // padding indices >= S sort after every real NaN entry
    if (i < S) slot[i] = -1;
  }
  __syncthreads();
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int p = i ^ j;
        if (p > i) {
          const bool up = (i & k) == 0;   // this pair sorts into "before" order
          const bool swap = up ? before(key[p], idx[p], key[i], idx[i])
                               : before(key[i], idx[i], key[p], idx[p]);
          if (swap) {
            const uint64_t tk = key[i]; key[i] = key[p]; key[p] = tk;
            const int ti = idx[i]; idx[i] = idx[p]; idx[p] = ti;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int j = threadIdx.x; j < cap; j += blockDim.x) {
    const int s = idx[j];
    const int64_t row = ((int64_t)e * B + b) * cap + j;   // expert-major (e, b, slot)
    token_flat[row] = b * S + s;
    gate_raw[row] = sc[s];
    slot[s] = (int16_t)j;
  }
}

// ---- gates: thread per token. totals in expert-ascending order from 0.0
// (np.add.at over the expert-major token_flat), then raw / (tot + eps) * alpha.
__global__ void gates_f64_kernel(const double* __restrict__ gate_raw,
                                 const int16_t* __restrict__ slot_of, double* __restrict__ gates,
                                 int32_t* __restrict__ comb_rows, int32_t* __restrict__ comb_cnt,
                                 int B, int S, int E, int cap, double eps, double alpha) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)B * S) return;
  const int b = (int)(t / S), s = (int)(t % S);
  double tot = 0.0;
  int n = 0;
  for (int e = 0; e < E; ++e) {
    const int j = slot_of[((int64_t)b * E + e) * S + s];
    if (j < 0) continue;
    const int32_t row = (int32_t)(((int64_t)e * B + b) * cap + j);
    comb_rows[t * E + n++] = row;
    tot += gate_raw[row];
  }
  comb_cnt[t] = n;
  const double den = tot + eps;
  for (int k = 0; k < n; ++k) {
    const int32_t row = comb_rows[t * E + k];
    gates[row] = gate_raw[row] / den * alpha;
  }
}

// ---- combine: warp per token, lanes over d.
__global__ void combine_f64_kernel(const double* __restrict__ yr, const double* __restrict__ ys,
                                   const double* __restrict__ gates,
                                   const int32_t* __restrict__ comb_rows,
                                   const int32_t* __restrict__ comb_cnt, double* __restrict__ out,
                                   int64_t T, int d, int E) {
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (t >= T) return;
  const int lane = threadIdx.x % 32;
  const int n = comb_cnt[t];
  for (int c = lane; c < d; c += 32) {
    double acc = 0.0;
    for (int k = 0; k < n; ++k) {
      const int32_t r = comb_rows[t * E + k];
      acc += yr[(int64_t)r * d + c] * gates[r];
    }
    out[t * d + c] = acc + ys[t * d + c];
  }
}

}  // namespace f64m

cudaError_t launch_route_f64(const double* x_norm, const double* t_emb, const double* w_r,
                             double* logits, double* scores_bes, int32_t* token_flat,
                             double* gate_raw, double* gates, int32_t* comb_rows,
                             int32_t* comb_cnt, int16_t* slot_of, int B, int S, int d, int E,
                             int cap, double eps, double alpha, cudaStream_t st) {
  using namespace f64m;
  const int64_t T = (int64_t)B * S;
  {
    dim3 grid((unsigned)((T + LBM - 1) / LBM), (unsigned)((E + LBN - 1) / LBN));
    router_logits_f64_kernel<<<grid, LNT, 0, st>>>(x_norm, t_emb, w_r, logits, T, S, d, E);
  }
  {
    const size_t smem = (size_t)SM_WARPS * E * sizeof(double);
    cudaError_t err = cudaFuncSetAttribute(softmax_f64_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    softmax_f64_kernel<<<(unsigned)((T + SM_WARPS - 1) / SM_WARPS), SM_WARPS * 32, smem, st>>>(
        logits, scores_bes, T, S, E);
  }
  {
    int n = 1;
    while (n < S) n <<= 1;
    const size_t smem = (size_t)n * (sizeof(uint64_t) + sizeof(int));
    cudaError_t err = cudaFuncSetAttribute(select_f64_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    const int threads = n < 1024 ? (n < 32 ? 32 : n) : 1024;
    select_f64_kernel<<<B * E, threads, smem, st>>>(scores_bes, token_flat, gate_raw, slot_of, B, S,
                                                    E, cap, n);
  }
  gates_f64_kernel<<<(unsigned)((T + 127) / 128), 128, 0, st>>>(gate_raw, slot_of, gates, comb_rows,
                                                                comb_cnt, B, S, E, cap, eps, alpha);
  return cudaGetLastError();
}

cudaError_t launch_combine_f64(const double* yr, const double* ys, const double* gates,
                               const int32_t* comb_rows, const int32_t* comb_cnt, double* out,
                               int64_t T, int d, int E, cudaStream_t st) {
  f64m::combine_f64_kernel<<<(unsigned)((T + 7) / 8), 256, 0, st>>>(yr, ys, gates, comb_rows,
                                                                      comb_cnt, out, T, d, E);
  return cudaGetLastError();
}

}  // namespace nimg
