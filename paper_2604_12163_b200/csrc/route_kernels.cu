// Routing and data-movement kernels of the expert-choice MoE layer.
//
//   router_tbias   t_emb . W_r[d:]  per sample, f64            (router.py:120-122, t half)
//   router_scores  x_norm . W_r[:d] + tbias in f64 -> fp32 logits; f64 softmax
//                  in numpy's exact summation order -> fp32 scores (router.py:122-123,
//                  tensor.py:280-287, 467-473). HBM-light, FP64-pipe bound.
//   ec_select      per (sample, expert) column: radix-select of the top-`cap`
//                  64-bit keys (score desc, token index asc), bitonic ordering of
//                  the winners (router.py:98-101, 126-136).
//   gate_norm      per-token totals in expert-ascending f64 order and the
//                  reference's fp32 rounding chain (router.py:137-143).
//   gather_rows    x_mod rows into expert-major order (moe.py:152-153).
//   combine        deterministic expert-ascending weighted sum + shared expert
//                  (moe.py:156-161, tensor.py:366-378).
#include "common.cuh"
#include "nimg_internal.h"

namespace nimg {

// ------------------------------------------------------------------ numpy sum
// Exact restatement of numpy's pairwise summation (used by `e.sum(axis=-1)`
// in tensor.py:471): < 8 terms sequential from 0.0; <= 128 terms with eight
// stride-8 accumulators folded as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a
// sequential tail; larger n split at n/2 rounded down to a multiple of 8.
__device__ double np_pairwise_sum(const double* a, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res += a[i];
    return res;
  }
  if (n <= 128) {
    double r0 = a[0], r1 = a[1], r2 = a[2], r3 = a[3], r4 = a[4], r5 = a[5], r6 = a[6], r7 = a[7];
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
      r0 += a[i + 0]; r1 += a[i + 1]; r2 += a[i + 2]; r3 += a[i + 3];
      r4 += a[i + 4]; r5 += a[i + 5]; r6 += a[i + 6]; r7 += a[i + 7];
    }
    double res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
}

// ------------------------------------------------------------------ t bias
// tb[b, e] = sum_k t_emb[b, k] * W_r[d + k, e] in f64. Block = (b, 32 experts),
// 8 k-slices per expert folded in a fixed order.
__global__ void router_tbias_kernel(const float* __restrict__ t_emb, const float* __restrict__ w_r,
                                    double* __restrict__ tb, int d, int E) {
  __shared__ double part[8][32];
  const int b = blockIdx.x;
  const int el = threadIdx.x & 31, ks = threadIdx.x >> 5;
  const int e = blockIdx.y * 32 + el;
  double acc = 0.0;
  if (e < E) {
    const float* t = t_emb + (int64_t)b * d;
    const float* w = w_r + (int64_t)d * E + e;
    for (int k = ks; k < d; k += 8) acc = fma((double)t[k], (double)w[(int64_t)k * E], acc);
  }
  part[ks][el] = acc;
  __syncthreads();
  if (ks == 0 && e < E) {
    double s = part[0][el];
    for (int j = 1; j < 8; ++j) s += part[j][el];
    tb[(int64_t)b * E + e] = s;
  }
}

// ------------------------------------------------------------------ router
// CTA = TM tokens x all E experts; thread = 4 tokens x 4 experts of f64
// accumulators. K staged through smem in KC-chunks as f64.
constexpr int RT_THREADS = 128;
constexpr int RT_KC = 32;

struct RouterGeom {
  int EG, TG, TM, EP;
};
__host__ __device__ inline RouterGeom router_geom(int E) {
  RouterGeom g;
  g.EG = (E + 3) / 4;
  g.TG = RT_THREADS / g.EG;
  g.TM = g.TG * 4;
  g.EP = g.EG * 4;
  return g;
}
__host__ __device__ inline size_t router_smem(int E) {
  RouterGeom g = router_geom(E);
  size_t loop = (size_t)RT_KC * g.TM * 8 + (size_t)RT_KC * g.EP * 8;
  size_t post = (size_t)g.TM * E * 8 + (size_t)g.TM * E * 4;  // ex (f64) + sc (f32)
  size_t r1 = loop > post ? loop : post;
  return r1 + (size_t)g.TM * E * 4 /*lg*/ + (size_t)g.TM * 16 /*mx, sum*/;
}

template <typename TX>
__global__ void __launch_bounds__(RT_THREADS)
router_scores_kernel(const TX* __restrict__ x, const float* __restrict__ w_r,
                     const double* __restrict__ tb, float* __restrict__ logits,
                     float* __restrict__ scores_bes, int B, int S, int d, int E) {
  extern __shared__ __align__(16) uint8_t sm[];
  const RouterGeom g = router_geom(E);
  const int64_t T = (int64_t)B * S;
  const int64_t t0 = (int64_t)blockIdx.x * g.TM;
  double* xs = reinterpret_cast<double*>(sm);            // [KC][TM]
  double* ws = xs + RT_KC * g.TM;                        // [KC][EP]
  const size_t r1 = router_smem(E) - (size_t)g.TM * E * 4 - (size_t)g.TM * 16;
  float* lg = reinterpret_cast<float*>(sm + r1);         // [TM][E]
  double* mx = reinterpret_cast<double*>(sm + r1 + (size_t)g.TM * E * 4);
  double* sum = mx + g.TM;
  double* ex = reinterpret_cast<double*>(sm);            // [TM][E]  (reuses loop region)
  float* sc = reinterpret_cast<float*>(sm + (size_t)g.TM * E * 8);  // [TM][E]

  const int tid = threadIdx.x;
  const bool active = tid < g.TG * g.EG;
  const int tg = active ? tid / g.EG : 0, eg = active ? tid % g.EG : 0;

  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;

  for (int k0 = 0; k0 < d; k0 += RT_KC) {
    for (int i = tid; i < g.TM * RT_KC; i += RT_THREADS) {
      const int tok = i / RT_KC, kk = i % RT_KC;
      const int64_t t = t0 + tok;
      double v = 0.0;
      if (t < T && k0 + kk < d) v = (double)to_f32(x[t * d + k0 + kk]);
      xs[kk * g.TM + tok] = v;
    }
    for (int i = tid; i < RT_KC * g.EP; i += RT_THREADS) {
      const int kk = i / g.EP, e = i % g.EP;
      double v = 0.0;
      if (e < E && k0 + kk < d) v = (double)w_r[(int64_t)(k0 + kk) * E + e];
      ws[kk * g.EP + e] = v;
    }
    __syncthreads();
    if (active) {
      const int kmax = min(RT_KC, d - k0);
      for (int kk = 0; kk < kmax; ++kk) {
        const double2 xa = *reinterpret_cast<const double2*>(&xs[kk * g.TM + tg * 4]);
        const double2 xb = *reinterpret_cast<const double2*>(&xs[kk * g.TM + tg * 4 + 2]);
        const double2 wa = *reinterpret_cast<const double2*>(&ws[kk * g.EP + eg * 4]);
        const double2 wb = *reinterpret_cast<const double2*>(&ws[kk * g.EP + eg * 4 + 2]);
        const double xv[4] = {xa.x, xa.y, xb.x, xb.y};
        const double wv[4] = {wa.x, wa.y, wb.x, wb.y};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(xv[i], wv[j], acc[i][j]);
      }
    }
    __syncthreads();
  }

  // logits = fp32(x-part + t-part)   (matmul f64 -> fp32, tensor.py:286-287)
  if (active) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int tok = tg * 4 + i;
      const int64_t t = t0 + tok;
      if (t >= T) continue;
      const int b = (int)(t / S);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int e = eg * 4 + j;
        if (e < E) lg[tok * E + e] = (float)(acc[i][j] + tb[(int64_t)b * E + e]);
      }
    }
  }
  __syncthreads();
  // row max (exact in any order)
  for (int tok = tid; tok < g.TM; tok += RT_THREADS) {
    double m = -INFINITY;
    for (int e = 0; e < E; ++e) m = fmax(m, (double)lg[tok * E + e]);
    mx[tok] = m;
  }
  __syncthreads();
  for (int i = tid; i < g.TM * E; i += RT_THREADS) {
    const int tok = i / E;
    ex[i] = exp((double)lg[i] - mx[tok]);
  }
  __syncthreads();
  for (int tok = tid; tok < g.TM; tok += RT_THREADS) sum[tok] = np_pairwise_sum(ex + tok * E, E);
  __syncthreads();
  for (int i = tid; i < g.TM * E; i += RT_THREADS) {
    const int tok = i / E;
    sc[i] = (float)(ex[i] / sum[tok]);
  }
  __syncthreads();
  // logits (B,S,E): contiguous run of TM*E floats
  for (int i = tid; i < g.TM * E; i += RT_THREADS) {
    const int64_t t = t0 + i / E;
    if (t < T) logits[t * E + (i % E)] = lg[i];
  }
  // scores transposed to (B,E,S): coalesced along tokens
  for (int i = tid; i < g.TM * E; i += RT_THREADS) {
    const int e = i / g.TM, tok = i % g.TM;
    const int64_t t = t0 + tok;
    if (t < T) {
      const int64_t b = t / S, s = t % S;
      scores_bes[(b * E + e) * S + s] = sc[tok * E + e];
    }
  }
}

// ------------------------------------------------------------------ select
constexpr int SEL_THREADS = 256;

NIMG_DEV uint32_t score_key(float v) {
  uint32_t u = __float_as_uint(v);
  if ((u & 0x7FFFFFFFu) > 0x7F800000u) return 0u;   // NaN sorts last (numpy argsort)
  if (u == 0x80000000u) u = 0u;                      // -0 == +0
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

template <int NT>
NIMG_DEV int block_excl_scan(int v, int* scratch /*[NT/32 + 1]*/, int& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += n;
  }
  if (lane == 31) scratch[w] = incl;
  __syncthreads();
  if (w == 0) {
    int s = lane < NT / 32 ? scratch[lane] : 0;
    int si = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, si, o);
      if (lane >= o) si += n;
    }
    if (lane < NT / 32) scratch[lane] = si - s;
    if (lane == 31) scratch[NT / 32] = si;
  }
  __syncthreads();
  const int res = scratch[w] + incl - v;
  total = scratch[NT / 32];
  __syncthreads();
  return res;
}

__host__ __device__ inline int next_pow2(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}
inline size_t select_smem(int S, int cap) {
  return (size_t)S * 4 + (size_t)next_pow2(cap) * 8 + 256 * 4 + 64 * 4;
}

__global__ void __launch_bounds__(SEL_THREADS)
ec_select_kernel(const float* __restrict__ scores_bes, int32_t* __restrict__ token_flat,
                 float* __restrict__ gate_raw, int16_t* __restrict__ slot_of, int B, int S, int E,
                 int cap) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int P = next_pow2(cap);
  uint64_t* win = reinterpret_cast<uint64_t*>(sm);                  // [P]
  uint32_t* keys = reinterpret_cast<uint32_t*>(sm + (size_t)P * 8);  // [S]
  uint32_t* hist = keys + S;                                        // [256]
  int* scratch = reinterpret_cast<int*>(hist + 256);                // [64]
  __shared__ uint32_t s_digit;
  __shared__ int s_k;

  const int b = blockIdx.x, e = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* col = scores_bes + ((int64_t)b * E + e) * S;
  for (int i = tid; i < S; i += SEL_THREADS) keys[i] = score_key(col[i]);

  // ---- radix select of the cap-th largest key, 8 bits per pass from the MSB
  uint32_t prefix = 0, pmask = 0;
  int k = cap;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += SEL_THREADS) hist[i] = 0;
    __syncthreads();
    for (int i = tid; i < S; i += SEL_THREADS) {
      const uint32_t key = keys[i];
      if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (warp == 0) {
      int cnt[8], local = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) { cnt[j] = (int)hist[255 - 8 * lane - j]; local += cnt[j]; }
      int incl = local;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += n;
      }
      const int excl = incl - local;
      if (excl < k && k <= incl) {
        int c = excl;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (c < k && c + cnt[j] >= k) { s_digit = 255u - 8u * lane - j; s_k = k - c; }
          c += cnt[j];
        }
      }
    }
    __syncthreads();
    prefix |= s_digit << shift;
    pmask |= 0xFFu << shift;
    k = s_k;
    __syncthreads();
  }
  const uint32_t thr = prefix;
  const int need_eq = k;

  // ---- compaction in token order: all keys > thr, the first need_eq == thr
  const int per = (S + SEL_THREADS - 1) / SEL_THREADS;
  const int lo = min(S, tid * per), hi = min(S, lo + per);
  int n_gt = 0, n_eq = 0;
  for (int i = lo; i < hi; ++i) {
    const uint32_t key = keys[i];
    n_gt += key > thr;
    n_eq += key == thr;
  }
  int tot;
  const int gt_before = block_excl_scan<SEL_THREADS>(n_gt, scratch, tot);
  int eq_before = block_excl_scan<SEL_THREADS>(n_eq, scratch, tot);
  int pos = gt_before + min(eq_before, need_eq);
  for (int i = lo; i < hi; ++i) {
    const uint32_t key = keys[i];
    const uint64_t comp = ((uint64_t)key << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)i);
    if (key > thr) {
      win[pos++] = comp;
    } else if (key == thr) {
      if (eq_before < need_eq) win[pos++] = comp;
      ++eq_before;
    }
  }
  for (int i = cap + tid; i < P; i += SEL_THREADS) win[i] = 0ull;
  __syncthreads();

  // ---- bitonic sort, descending composite key (score desc, index asc)
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < P / 2; i += SEL_THREADS) {
        const int a = 2 * i - (i & (stride - 1));
        const int c = a + stride;
        const bool desc = (a & size) == 0;
        const uint64_t va = win[a], vc = win[c];
        if ((va < vc) == desc) { win[a] = vc; win[c] = va; }
      }
      __syncthreads();
    }
  }

  // ---- outputs in expert-major (e, b, slot) order (router.py:131-133)
  const int64_t T = (int64_t)B * S;
  for (int j = tid; j < cap; j += SEL_THREADS) {
    const uint32_t idx = 0xFFFFFFFFu - (uint32_t)(win[j] & 0xFFFFFFFFull);
    const int64_t o = ((int64_t)e * B + b) * cap + j;
    token_flat[o] = (int32_t)((int64_t)b * S + idx);
    gate_raw[o] = col[idx];
    slot_of[(int64_t)e * T + (int64_t)b * S + idx] = (int16_t)j;
  }
}

// ------------------------------------------------------------------ gates
// Per token (router.py:137-143): totals = fp32(sum_e f64(raw)) in expert order
// (np.add.at order), den = fp32(f64(tot) + f64(fp32 eps)),
// gate = fp32(f64(fp32(f64(raw) / f64(den))) * f64(fp32 alpha)).
__global__ void gate_norm_kernel(const float* __restrict__ scores_bes,
                                 const int16_t* __restrict__ slot_of, float* __restrict__ gates,
                                 int32_t* __restrict__ comb_rows, int32_t* __restrict__ comb_cnt,
                                 int B, int S, int E, int cap, float eps32, float alpha32) {
  const int64_t T = (int64_t)B * S;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int64_t b = t / S, s = t % S;
  double tot = 0.0;
  int cnt = 0;
  for (int e = 0; e < E; ++e) {
    const int j = slot_of[(int64_t)e * T + t];
    if (j >= 0) {
      tot += (double)scores_bes[(b * E + e) * S + s];
      comb_rows[(int64_t)cnt * T + t] = (int32_t)(((int64_t)e * B + b) * cap + j);
      ++cnt;
    }
  }
  comb_cnt[t] = cnt;
  const float tot32 = (float)tot;
  const float den = (float)((double)tot32 + (double)eps32);
  for (int k = 0; k < cnt; ++k) {
    const int32_t row = comb_rows[(int64_t)k * T + t];
    const int e = (int)(row / ((int64_t)B * cap));
    const float raw = scores_bes[(b * E + e) * S + s];
    const float q = (float)((double)raw / (double)den);
    gates[row] = (float)((double)q * (double)alpha32);
  }
}

// ------------------------------------------------------------------ gather
// dst[i, :] = src[idx[i], :]; one warp per row, 16-B vectors, all loads first.
__global__ void gather_rows_vec_kernel(const int4* __restrict__ src, int64_t row_vecs,
                                       const int32_t* __restrict__ idx, int64_t n_idx,
                                       int4* __restrict__ dst) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= n_idx) return;
  const int lane = threadIdx.x & 31;
  const int4* s = src + (int64_t)idx[row] * row_vecs;
  int4* o = dst + row * row_vecs;
  int64_t v = lane;
  for (; v + 96 < row_vecs; v += 128) {
    const int4 a0 = __ldg(s + v), a1 = __ldg(s + v + 32), a2 = __ldg(s + v + 64), a3 = __ldg(s + v + 96);
    o[v] = a0; o[v + 32] = a1; o[v + 64] = a2; o[v + 96] = a3;
  }
  for (; v < row_vecs; v += 32) o[v] = __ldg(s + v);
}
__global__ void gather_rows_byte_kernel(const uint8_t* __restrict__ src, int64_t row_bytes,
                                        const int32_t* __restrict__ idx, int64_t n_idx,
                                        uint8_t* __restrict__ dst) {
  const int64_t row = blockIdx.x;
  if (row >= n_idx) return;
  const uint8_t* s = src + (int64_t)idx[row] * row_bytes;
  for (int64_t i = threadIdx.x; i < row_bytes; i += blockDim.x) dst[row * row_bytes + i] = s[i];
}

// ------------------------------------------------------------------ combine
// moe.py:156-161 with the reference's rounding chain: gated = fp32(Y*gate),
// combined = fp32(sum over selecting experts in ascending order, f64),
// out = round(f64(combined) + f64(shared)).
template <typename TY, typename TO, int VEC>
__global__ void __launch_bounds__(256)
combine_kernel(const TY* __restrict__ yr, const TY* __restrict__ ys, const float* __restrict__ gates,
               const int32_t* __restrict__ comb_rows, const int32_t* __restrict__ comb_cnt,
               TO* __restrict__ out, int64_t T, int d) {
  const int64_t t = blockIdx.x;
  const int cnt = comb_cnt[t];
  for (int c = threadIdx.x * VEC; c < d; c += blockDim.x * VEC) {
    double acc[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[v] = 0.0;
    for (int k = 0; k < cnt; ++k) {
      const int32_t row = comb_rows[(int64_t)k * T + t];
      const float gte = gates[row];
      const TY* y = yr + (int64_t)row * d + c;
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[v] += (double)(to_f32(y[v]) * gte);
    }
    const TY* sh = ys + t * d + c;
    TO* o = out + t * d + c;
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      const float comb = (float)acc[v];
      o[v] = from_f32<TO>((float)((double)comb + (double)to_f32(sh[v])));
    }
  }
}

// ------------------------------------------------------------------ launchers
cudaError_t launch_router_tbias(const float* t_emb, const float* w_r, double* tb, int B, int d,
                                int E, cudaStream_t s) {
  dim3 grid(B, (E + 31) / 32);
  router_tbias_kernel<<<grid, 256, 0, s>>>(t_emb, w_r, tb, d, E);
  return cudaGetLastError();
}

cudaError_t launch_router_scores(bool x_bf16, const void* x_norm, const float* w_r,
                                 const double* tb, float* logits, float* scores_bes, int B, int S,
                                 int d, int E, cudaStream_t s) {
  const RouterGeom g = router_geom(E);
  const int64_t T = (int64_t)B * S;
  const int grid = (int)((T + g.TM - 1) / g.TM);
  const size_t smem = router_smem(E);
  cudaError_t err;
  if (x_bf16) {
    err = cudaFuncSetAttribute(router_scores_kernel<bf16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    router_scores_kernel<bf16><<<grid, RT_THREADS, smem, s>>>(
        reinterpret_cast<const bf16*>(x_norm), w_r, tb, logits, scores_bes, B, S, d, E);
  } else {
    err = cudaFuncSetAttribute(router_scores_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    router_scores_kernel<float><<<grid, RT_THREADS, smem, s>>>(
        reinterpret_cast<const float*>(x_norm), w_r, tb, logits, scores_bes, B, S, d, E);
  }
  return cudaGetLastError();
}

cudaError_t launch_ec_select(const float* scores_bes, int32_t* token_flat, float* gate_raw,
                             int16_t* slot_of, int B, int S, int E, int cap, cudaStream_t s) {
  const size_t smem = select_smem(S, cap);
  cudaError_t err = cudaFuncSetAttribute(ec_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  dim3 grid(B, E);
  ec_select_kernel<<<grid, SEL_THREADS, smem, s>>>(scores_bes, token_flat, gate_raw, slot_of, B,
                                                   S, E, cap);
  return cudaGetLastError();
}

cudaError_t launch_gate_norm(const float* scores_bes, const int16_t* slot_of, float* gates,
                             int32_t* comb_rows, int32_t* comb_cnt, int B, int S, int E, int cap,
                             float gate_eps, float gate_scale, cudaStream_t s) {
  const int64_t T = (int64_t)B * S;
  const int grid = (int)((T + 127) / 128);
  gate_norm_kernel<<<grid, 128, 0, s>>>(scores_bes, slot_of, gates, comb_rows, comb_cnt, B, S, E,
                                        cap, gate_eps, gate_scale);
  return cudaGetLastError();
}

cudaError_t launch_gather_rows(const void* src, int64_t row_bytes, const int32_t* idx,
                               int64_t n_idx, void* dst, cudaStream_t s) {
  if (n_idx <= 0) return cudaSuccess;
  const bool vec = (row_bytes % 16 == 0) && ((uintptr_t)src % 16 == 0) && ((uintptr_t)dst % 16 == 0);
  if (vec) {
    const int rows_per_cta = 8;
    const int64_t grid = (n_idx + rows_per_cta - 1) / rows_per_cta;
    gather_rows_vec_kernel<<<(unsigned)grid, 32 * rows_per_cta, 0, s>>>(
        reinterpret_cast<const int4*>(src), row_bytes / 16, idx, n_idx, reinterpret_cast<int4*>(dst));
  } else {
    gather_rows_byte_kernel<<<(unsigned)n_idx, 128, 0, s>>>(
        reinterpret_cast<const uint8_t*>(src), row_bytes, idx, n_idx, reinterpret_cast<uint8_t*>(dst));
  }
  return cudaGetLastError();
}

template <typename TY, typename TO>
static void combine_dispatch(const void* yr, const void* ys, const float* gates,
                             const int32_t* rows, const int32_t* cnt, void* out, int64_t T, int d,
                             cudaStream_t s) {
  if (d % 8 == 0)
    combine_kernel<TY, TO, 8><<<(unsigned)T, 256, 0, s>>>(
        (const TY*)yr, (const TY*)ys, gates, rows, cnt, (TO*)out, T, d);
  else
    combine_kernel<TY, TO, 1><<<(unsigned)T, 256, 0, s>>>(
        (const TY*)yr, (const TY*)ys, gates, rows, cnt, (TO*)out, T, d);
}

cudaError_t launch_combine(bool y_bf16, bool out_bf16, const void* y_routed, const void* y_shared,
                           const float* gates, const int32_t* comb_rows, const int32_t* comb_cnt,
                           void* out, int64_t T, int d, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  if (y_bf16 && out_bf16) combine_dispatch<bf16, bf16>(y_routed, y_shared, gates, comb_rows, comb_cnt, out, T, d, s);
  else if (y_bf16) combine_dispatch<bf16, float>(y_routed, y_shared, gates, comb_rows, comb_cnt, out, T, d, s);
  else if (out_bf16) combine_dispatch<float, bf16>(y_routed, y_shared, gates, comb_rows, comb_cnt, out, T, d, s);
  else combine_dispatch<float, float>(y_routed, y_shared, gates, comb_rows, comb_cnt, out, T, d, s);
  return cudaGetLastError();
}

}  // namespace nimg
