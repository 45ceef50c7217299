// Backward of the expert-choice MoE layer: the pullbacks
// the reference's tape applies to moe_forward (moe.py:138-164), in reverse:
//
//   combine_bwd   add / scatter_add_rows / mul / broadcast_to bwd
//                 (tensor.py:235-260, :321-328, :366-382): dY_r = gate * g_out[token],
//                 dgate = <g_out[token], Y_r>; then the gate chain
//                 gates = (raw / (tot + eps)) * alpha (router.py:137-143; div/add/
//                 gather_rows/scatter_add_rows bwd) and the softmax pullback
//                 s * (g - <g, s>) on the f64 probabilities (tensor.py:467-477) ->
//                 dlogits (T, E) fp32.
//   router_bwd_*  matmul / concat / broadcast_to bwd of logits = [x_norm | t] W_r
//                 (tensor.py:280-296, :321-345): dx_norm = dlogits W_r[:d]^T,
//                 dt_emb = (sum_s dlogits) W_r[d:]^T, dW_r = [x_norm | t]^T dlogits
//                 (token-chunk partials folded in a fixed order: deterministic).
//   grouped_simt_bwd  the swiglu pullback (moe.py:53-62) per expert segment on
//                 CUDA cores (fp32 parity mode, and shapes the tcgen05 path does not
//                 take): dgrad of GEMM2 with the SwiGLU derivative in the epilogue,
//                 dgrad of GEMM1, and both weight gradients.
// The gather pullback (gather_rows bwd, tensor.py:358-361) is the forward
// combine kernel with unit gates (route_kernels.cu).
#include <type_traits>

#include "common.cuh"
#include "nimg_internal.h"

namespace nimg {

// ------------------------------------------------------------------ combine / gates / softmax
constexpr int CBB_WARPS = 8;

NIMG_DEV float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
NIMG_DEV double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
NIMG_DEV double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <typename T> struct V8 {   // 8 elements
  typename std::conditional<sizeof(T) == 2, uint4, float4[2]>::type raw;
  NIMG_DEV void load(const T* p) {
    if constexpr (sizeof(T) == 2) raw = __ldg(reinterpret_cast<const uint4*>(p));
    else { raw[0] = __ldg(reinterpret_cast<const float4*>(p)); raw[1] = __ldg(reinterpret_cast<const float4*>(p) + 1); }
  }
  NIMG_DEV float at(int i) const { return to_f32(reinterpret_cast<const T*>(&raw)[i]); }
};
template <typename T> NIMG_DEV void store8(T* p, const float (&v)[8]) {
  if constexpr (sizeof(T) == 2) {
    uint4 u = make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]),
                         pack_bf16x2(v[6], v[7]));
    *reinterpret_cast<uint4*>(p) = u;
  } else {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
}

// Warp per token. VEC8: d % 8 == 0 and 16-B aligned rows (vector loads).
template <typename TG, typename TY, typename TD, bool VEC8>
__global__ void __launch_bounds__(CBB_WARPS * 32)
combine_bwd_kernel(const TG* __restrict__ g_out, const TY* __restrict__ yr,
                   const float* __restrict__ gates, const float* __restrict__ gate_raw,
                   const int32_t* __restrict__ comb_rows, const int32_t* __restrict__ comb_cnt,
                   const float* __restrict__ logits, TD* __restrict__ dyr, TD* __restrict__ dys,
                   float* __restrict__ dlogits, bf16* __restrict__ dl16, int64_t T, int d, int E,
                   int rows_per_expert, float eps32, float alpha32) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(16) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* gsc = reinterpret_cast<double*>(sm) + (size_t)warp * E;                 // d loss / d score
  int32_t* rows = reinterpret_cast<int32_t*>(sm + (size_t)CBB_WARPS * E * 8) + (size_t)warp * E;
  float* dg = reinterpret_cast<float*>(sm + (size_t)CBB_WARPS * E * 12) + (size_t)warp * E;
  const int64_t t = (int64_t)blockIdx.x * CBB_WARPS + warp;
  if (t >= T) return;
  const int cnt = comb_cnt[t];
  for (int k = lane; k < cnt; k += 32) rows[k] = comb_rows[t * E + k];
  for (int e = lane; e < E; e += 32) gsc[e] = 0.0;
  __syncwarp();
  const TG* g = g_out + t * d;
  // dY rows (mul bwd: g * gate) and dgate = sum_c g * Y (mul + broadcast_to bwd);
  // NB rows at a time so their loads are in flight together
  if constexpr (VEC8) {
    constexpr int NB = 4;
    for (int k0 = 0; k0 < cnt; k0 += NB) {
      float gate[NB], dot[NB];
      const TY* y[NB];
      TD* o[NB];
#pragma unroll
      for (int q = 0; q < NB; ++q) {
        const int64_t r = rows[k0 + q < cnt ? k0 + q : k0];
        gate[q] = __ldg(gates + r);
        y[q] = yr + r * d;
        o[q] = dyr + r * d;
        dot[q] = 0.f;
      }
      for (int c = lane * 8; c < d; c += 256) {
        V8<TG> gv; gv.load(g + c);
        V8<TY> yv[NB];
#pragma unroll
        for (int q = 0; q < NB; ++q)
          if (k0 + q < cnt) yv[q].load(y[q] + c);
#pragma unroll
        for (int q = 0; q < NB; ++q) {
          if (k0 + q >= cnt) continue;
          float res[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            dot[q] = fmaf(gv.at(i), yv[q].at(i), dot[q]);
            res[i] = gv.at(i) * gate[q];
          }
          store8(o[q] + c, res);
        }
      }
#pragma unroll
      for (int q = 0; q < NB; ++q) {
        const float v = warp_sum_f(dot[q]);
        if (lane == 0 && k0 + q < cnt) dg[k0 + q] = v;
      }
    }
  } else {
    for (int k = 0; k < cnt; ++k) {
      const int64_t r = rows[k];
      const float gate = __ldg(gates + r);
      const TY* y = yr + r * d;
      TD* o = dyr + r * d;
      float dot = 0.f;
      for (int c = lane; c < d; c += 32) {
        const float gvv = to_f32(g[c]);
        dot = fmaf(gvv, to_f32(y[c]), dot);
        o[c] = from_f32<TD>(gvv * gate);
      }
      dot = warp_sum_f(dot);
      if (lane == 0) dg[k] = dot;
    }
  }
  if (dys != nullptr) {   // shared-expert upstream gradient in the dY dtype
    TD* o = dys + t * d;
    if constexpr (VEC8) {
      for (int c = lane * 8; c < d; c += 256) {
        V8<TG> gv; gv.load(g + c);
        float res[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) res[i] = gv.at(i);
        store8(o + c, res);
      }
    } else {
      for (int c = lane; c < d; c += 32) o[c] = from_f32<TD>(to_f32(g[c]));
    }
  }
  __syncwarp();
  // gate chain pullback (router.py:140-143), f64 like the reference's closures
  double tot = 0.0;
  if (lane == 0)
    for (int k = 0; k < cnt; ++k) tot += (double)__ldg(gate_raw + rows[k]);   // np.add.at order
  const float tot32 = __shfl_sync(0xffffffffu, (float)tot, 0);
  const double den = (double)(float)((double)tot32 + (double)eps32);
  double gden = 0.0;
  for (int k = lane; k < cnt; k += 32) {
    const double gq = (double)dg[k] * (double)alpha32;
    gden += -gq * (double)__ldg(gate_raw + rows[k]) / (den * den);
  }
  const double gtot = warp_sum_d(gden);
  for (int k = lane; k < cnt; k += 32) {
    const double gq = (double)dg[k] * (double)alpha32;
    gsc[rows[k] / rows_per_expert] = gq / den + gtot;
  }
  __syncwarp();
  // softmax pullback on the f64 probabilities of the fp32 logits
  const float* lg = logits + t * E;
  double m = -INFINITY;
  for (int e = lane; e < E; e += 32) m = fmax(m, (double)__ldg(lg + e));
  m = warp_max_d(m);
  double se = 0.0;
  for (int e = lane; e < E; e += 32) se += exp((double)__ldg(lg + e) - m);
  se = warp_sum_d(se);
  double gs = 0.0;
  for (int e = lane; e < E; e += 32) gs += gsc[e] * (exp((double)__ldg(lg + e) - m) / se);
  gs = warp_sum_d(gs);
  for (int e = lane; e < E; e += 32) {
    const double s = exp((double)__ldg(lg + e) - m) / se;
    const float v = (float)(s * (gsc[e] - gs));
    dlogits[t * E + e] = v;
    if (dl16 != nullptr) dl16[t * E + e] = __float2bfloat16_rn(v);
  }
}

// ------------------------------------------------------------------ router pullback
// dx_norm[t, j] = sum_e dl[t, e] * W_r[j, e]   (64 tokens x 64 columns per CTA)
constexpr int RB_T = 64, RB_J = 64, RB_K = 16;
template <typename TX>
__global__ void __launch_bounds__(256)
router_bwd_dx_kernel(const float* __restrict__ dl, const float* __restrict__ w_r, TX* __restrict__ dx,
                     int64_t T, int d, int E) {
  pdl_trigger();
  pdl_wait();
  __shared__ float As[RB_K][RB_T + 4];
  __shared__ float Bs[RB_K][RB_J + 4];
  const int64_t t0 = (int64_t)blockIdx.x * RB_T;
  const int j0 = blockIdx.y * RB_J;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < E; k0 += RB_K) {
    for (int i = threadIdx.x; i < RB_T * RB_K; i += 256) {
      const int r = i / RB_K, kk = i % RB_K;
      As[kk][r] = (t0 + r < T && k0 + kk < E) ? dl[(t0 + r) * E + k0 + kk] : 0.f;
      Bs[kk][r] = (j0 + r < d && k0 + kk < E) ? w_r[(int64_t)(j0 + r) * E + k0 + kk] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < RB_K; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = As[kk][ty * 4 + i]; b[i] = Bs[kk][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t t = t0 + ty * 4 + i;
    if (t >= T) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = j0 + tx * 4 + j;
      if (c < d) dx[t * d + c] = from_f32<TX>(acc[i][j]);
    }
  }
}

// part[c][j][e] = sum over tokens of chunk c of x_norm[t, j] * dl[t, e]
constexpr int RW_CHUNK = 256;
template <typename TX>
__global__ void __launch_bounds__(256)
router_bwd_dw_partial_kernel(const TX* __restrict__ xn, const float* __restrict__ dl,
                             float* __restrict__ part, int64_t T, int d, int E) {
  pdl_trigger();
  pdl_wait();
  __shared__ float Xs[RB_K][RB_J + 4];
  __shared__ float Ls[RB_K][RB_J + 4];
  const int j0 = blockIdx.x * RB_J, e0 = blockIdx.y * RB_J;
  const int64_t c = blockIdx.z;
  const int64_t tb = c * RW_CHUNK;
  const int64_t te = tb + RW_CHUNK < T ? tb + RW_CHUNK : T;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int64_t k0 = tb; k0 < te; k0 += RB_K) {
    for (int i = threadIdx.x; i < RB_K * RB_J; i += 256) {
      const int kk = i / RB_J, r = i % RB_J;
      const int64_t t = k0 + kk;
      Xs[kk][r] = (t < te && j0 + r < d) ? to_f32(xn[t * d + j0 + r]) : 0.f;
      Ls[kk][r] = (t < te && e0 + r < E) ? dl[t * E + e0 + r] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < RB_K; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = Xs[kk][ty * 4 + i]; b[i] = Ls[kk][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  float* pc = part + c * (int64_t)d * E;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int j = j0 + ty * 4 + i;
    if (j >= d) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = e0 + tx * 4 + q;
      if (e < E) pc[(int64_t)j * E + e] = acc[i][q];
    }
  }
}

// colsum[b, e] = sum_s dl[b, s, e] (fixed order: 8 strided partial sums folded in order)
__global__ void __launch_bounds__(256)
router_bwd_colsum_kernel(const float* __restrict__ dl, float* __restrict__ colsum, int S, int E) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[8][33];
  const int b = blockIdx.y, e = blockIdx.x * 32 + (threadIdx.x & 31), sl = threadIdx.x >> 5;
  float acc = 0.f;
  if (e < E)
    for (int s = sl; s < S; s += 8) acc += dl[((int64_t)b * S + s) * E + e];
  red[sl][threadIdx.x & 31] = acc;
  __syncthreads();
  if (sl == 0 && e < E) {
    float v = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) v += red[i][threadIdx.x & 31];
    colsum[(int64_t)b * E + e] = v;
  }
}

// g_w_r[:d] = sum_c part[c] (fixed order); g_w_r[d + j, e] = sum_b t[b, j] colsum[b, e];
// g_t[b, j] = sum_e colsum[b, e] W_r[d + j, e]
__global__ void __launch_bounds__(256)
router_bwd_fold_kernel(const float* __restrict__ part, int nchunks, const float* __restrict__ colsum,
                       const float* __restrict__ t_emb, const float* __restrict__ w_r,
                       float* __restrict__ g_wr, float* __restrict__ g_t, int B, int d, int E) {
  pdl_trigger();
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nx = (int64_t)d * E;
  if (i < nx) {
    float v = 0.f;
    for (int c = 0; c < nchunks; ++c) v += part[(int64_t)c * nx + i];
    g_wr[i] = v;
    const int j = (int)(i / E), e = (int)(i % E);
    float vt = 0.f;
    for (int b = 0; b < B; ++b) vt = fmaf(t_emb[(int64_t)b * d + j], colsum[(int64_t)b * E + e], vt);
    g_wr[nx + i] = vt;
  }
  if (i < (int64_t)B * d) {
    const int b = (int)(i / d), j = (int)(i % d);
    float v = 0.f;
    for (int e = 0; e < E; ++e) v = fmaf(colsum[(int64_t)b * E + e], w_r[(int64_t)(d + j) * E + e], v);
    g_t[i] = v;
  }
}

// ------------------------------------------------------------------ SIMT grouped pullbacks
// Per expert segment (rows r of a bank, expert e), the swiglu pullback of
// moe.py:53-62 with h1|h3 saved by the forward (H rows of width 2h):
//   BWD_D2: dH[r, n] = (dY W2_e)[r, n] -> dH1 = v h3 sig (1 + h1 (1 - sig)), dH3 = v act
//   BWD_D1: dX[r, n] = sum_k dH[r, k] [W1_e; W3_e][k, n]          (K = 2h)
//   BWD_W2: dW2_e[m, n] = sum_r dY[r, m] pre[r, n]
//   BWD_W1: [dW1_e; dW3_e][m, n] = sum_r dH[r, m] X[r, n]          (M = 2h)
namespace sb {
constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

template <int MODE> NIMG_DEV bool is_w() { return MODE == BWD_W2 || MODE == BWD_W1; }

template <int MODE, typename TA, typename TB>
__global__ void __launch_bounds__(NT) grouped_simt_bwd_kernel(const __grid_constant__ BwdParams p) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x;
  int lo = 0, hi = p.nseg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (p.seg_tile0[mid] <= t) lo = mid; else hi = mid - 1;
  }
  const BwdBank& bk = p.bank[p.seg_bank[lo]];
  const int local = t - p.seg_tile0[lo];
  const int m_blk = local / bk.ntn, n_blk = local % bk.ntn;
  const int64_t row0 = p.seg_row0[lo];
  const int seg_rows = p.seg_rows[lo];
  const int64_t e = p.seg_expert[lo];
  const int m0 = m_blk * BM, n0 = n_blk * BN;
  const int M = is_w<MODE>() ? bk.M : seg_rows;
  const int K = is_w<MODE>() ? seg_rows : bk.K;
  const int N = bk.N, h = bk.h;
  const TA* A = reinterpret_cast<const TA*>(bk.a);
  const TB* Bp = reinterpret_cast<const TB*>(bk.b);
  const TB* B3 = reinterpret_cast<const TB*>(bk.b3);
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += BK) {
    for (int i = threadIdx.x; i < BM * BK; i += NT) {
      int r, kk;
      if (is_w<MODE>()) { r = i % BM; kk = i / BM; } else { kk = i % BK; r = i / BK; }
      const int m = m0 + r, k = k0 + kk;
      float v = 0.f;
      if (m < M && k < K) {
        if (is_w<MODE>()) v = to_f32(A[(row0 + k) * bk.a_ld + m]);      // A(m, k) = rowop[k][m]
        else v = to_f32(A[(row0 + m) * bk.a_ld + k]);                   // A(m, k) = rows[m][k]
      }
      As[kk][r] = v;
    }
    for (int i = threadIdx.x; i < BN * BK; i += NT) {
      const int c = i % BN, kk = i / BN;        // n fastest: every B operand here is N-contiguous
      const int n = n0 + c, k = k0 + kk;
      float v = 0.f;
      if (n < N && k < K) {
        if (MODE == BWD_D2) v = to_f32(Bp[e * (int64_t)N * K + (int64_t)k * N + n]);          // W2_e[k][n]
        else if (MODE == BWD_D1)
          v = k < h ? to_f32(Bp[e * (int64_t)h * N + (int64_t)k * N + n])                     // W1_e[k][n]
                    : to_f32(B3[e * (int64_t)h * N + (int64_t)(k - h) * N + n]);              // W3_e[k-h][n]
        else v = to_f32(Bp[(row0 + k) * bk.b_ld + n]);                                        // rowop[k][n]
      }
      Bs[kk][c] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = As[kk][ty * 4 + i]; b[i] = Bs[kk][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      const float v = acc[i][j];
      if (MODE == BWD_D2) {
        const float* hr = reinterpret_cast<const float*>(bk.aux) + (row0 + m) * (int64_t)(2 * h);
        const float h1 = hr[n], h3 = hr[h + n];
        const float sig = 1.0f / (1.0f + expf(-h1));
        float* o = reinterpret_cast<float*>(bk.out) + (row0 + m) * (int64_t)(2 * h);
        o[n] = v * h3 * sig * (1.0f + h1 * (1.0f - sig));
        o[h + n] = v * h1 * sig;
      } else if (MODE == BWD_D1) {
        reinterpret_cast<float*>(bk.out)[(row0 + m) * bk.out_ld + n] = v;
      } else if (MODE == BWD_W2) {
        reinterpret_cast<float*>(bk.out)[e * (int64_t)M * N + (int64_t)m * N + n] = v;
      } else {
        float* o = m < h ? reinterpret_cast<float*>(bk.out) + e * (int64_t)h * N + (int64_t)m * N
                         : reinterpret_cast<float*>(bk.out3) + e * (int64_t)h * N + (int64_t)(m - h) * N;
        o[n] = v;
      }
    }
  }
}
}  // namespace sb

int simt_bwd_bm() { return sb::BM; }
int simt_bwd_bn() { return sb::BN; }

cudaError_t launch_grouped_simt_bwd(int mode, bool b_bf16, const BwdParams& p, cudaStream_t s) {
  if (p.total_tiles <= 0) return cudaSuccess;
  const dim3 grid(p.total_tiles), block(sb::NT);
#define NIMG_SB(M)                                                                                  \
  return b_bf16 ? launch_pdl(sb::grouped_simt_bwd_kernel<M, float, bf16>, grid, block, 0, s, p)   \
                : launch_pdl(sb::grouped_simt_bwd_kernel<M, float, float>, grid, block, 0, s, p)
  switch (mode) {
    case BWD_D2: NIMG_SB(BWD_D2);
    case BWD_D1: NIMG_SB(BWD_D1);
    case BWD_W2: NIMG_SB(BWD_W2);
    default: NIMG_SB(BWD_W1);
  }
#undef NIMG_SB
}

// ------------------------------------------------------------------ launchers
cudaError_t launch_combine_bwd(bool g_bf16, bool y_bf16, bool dy_bf16, const void* g_out,
                               const void* yr, const float* gates, const float* gate_raw,
                               const int32_t* comb_rows, const int32_t* comb_cnt,
                               const float* logits, void* dyr, void* dys, float* dlogits,
                               bf16_raw* dl16_raw, int64_t T, int d, int E, int rows_per_expert,
                               float eps32, float alpha32, cudaStream_t s) {
  bf16* dl16 = reinterpret_cast<bf16*>(dl16_raw);
  if (T <= 0) return cudaSuccess;
  const unsigned grid = (unsigned)((T + CBB_WARPS - 1) / CBB_WARPS);
  const size_t smem = (size_t)CBB_WARPS * E * 16;
  const bool v8 = d % 8 == 0;
#define NIMG_CBB(TG, TY, TD)                                                                       \
  return v8 ? launch_pdl(combine_bwd_kernel<TG, TY, TD, true>, dim3(grid), dim3(CBB_WARPS * 32),  \
                         smem, s, (const TG*)g_out, (const TY*)yr, gates, gate_raw, comb_rows,    \
                         comb_cnt, logits, (TD*)dyr, (TD*)dys, dlogits, dl16, T, d, E,                  \
                         rows_per_expert, eps32, alpha32)                                          \
            : launch_pdl(combine_bwd_kernel<TG, TY, TD, false>, dim3(grid), dim3(CBB_WARPS * 32), \
                         smem, s, (const TG*)g_out, (const TY*)yr, gates, gate_raw, comb_rows,    \
                         comb_cnt, logits, (TD*)dyr, (TD*)dys, dlogits, dl16, T, d, E,                  \
                         rows_per_expert, eps32, alpha32)
  // supported combos: tcgen05 path (all bf16); SIMT path (g act, y/dY fp32)
  if (g_bf16 && y_bf16 && dy_bf16) { NIMG_CBB(bf16, bf16, bf16); }
  if (g_bf16 && !y_bf16 && !dy_bf16) { NIMG_CBB(bf16, float, float); }
  if (!g_bf16 && !y_bf16 && !dy_bf16) { NIMG_CBB(float, float, float); }
#undef NIMG_CBB
  return cudaErrorInvalidValue;
}

size_t router_bwd_part_bytes(int64_t T, int d, int E) {
  return (size_t)((T + RW_CHUNK - 1) / RW_CHUNK) * d * E * 4;
}

cudaError_t launch_router_bwd_simt(bool x_bf16, const void* x_norm, const float* w_r,
                                   const float* dl, void* dx, float* part, int64_t T, int d, int E,
                                   cudaStream_t s, int* nchunks) {
  *nchunks = (int)((T + RW_CHUNK - 1) / RW_CHUNK);
  if (T <= 0) return cudaSuccess;
  const dim3 gdx((unsigned)((T + RB_T - 1) / RB_T), (unsigned)((d + RB_J - 1) / RB_J));
  cudaError_t err = x_bf16
      ? launch_pdl(router_bwd_dx_kernel<bf16>, gdx, dim3(256), 0, s, dl, w_r, (bf16*)dx, T, d, E)
      : launch_pdl(router_bwd_dx_kernel<float>, gdx, dim3(256), 0, s, dl, w_r, (float*)dx, T, d, E);
  if (err != cudaSuccess) return err;
  const dim3 gdw((unsigned)((d + RB_J - 1) / RB_J), (unsigned)((E + RB_J - 1) / RB_J), (unsigned)*nchunks);
  return x_bf16 ? launch_pdl(router_bwd_dw_partial_kernel<bf16>, gdw, dim3(256), 0, s,
                             (const bf16*)x_norm, dl, part, T, d, E)
                : launch_pdl(router_bwd_dw_partial_kernel<float>, gdw, dim3(256), 0, s,
                             (const float*)x_norm, dl, part, T, d, E);
}

cudaError_t launch_router_bwd_fold(const float* dl, const float* t_emb, const float* w_r,
                                   const float* part, int nchunks, float* colsum, float* g_wr,
                                   float* g_t, int B, int S, int d, int E, cudaStream_t s) {
  if ((int64_t)B * S <= 0) return cudaSuccess;
  cudaError_t err = launch_pdl(router_bwd_colsum_kernel, dim3((unsigned)((E + 31) / 32), (unsigned)B),
                               dim3(256), 0, s, dl, colsum, S, E);
  if (err != cudaSuccess) return err;
  const int64_t n = (int64_t)d * E > (int64_t)B * d ? (int64_t)d * E : (int64_t)B * d;
  return launch_pdl(router_bwd_fold_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s,
                    part, nchunks, (const float*)colsum, t_emb, w_r, g_wr, g_t, B, d, E);
}

// out[i] = sum_c part[c][i], c ascending (fixed order): fold of the shared
// bank's row-chunk weight-gradient partials
__global__ void sum_partials_kernel(const float4* __restrict__ part, int ks, int64_t n4,
                                    float4* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n4) return;
  float4 a = __ldg(part + i);
  for (int c = 1; c < ks; ++c) {
    const float4 b = __ldg(part + (int64_t)c * n4 + i);
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
  }
  out[i] = a;
}

cudaError_t launch_sum_partials(const float* part, int ks, int64_t n, float* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int64_t n4 = n / 4;   // n % 4 == 0 (weight shapes are multiples of 64)
  return launch_pdl(sum_partials_kernel, dim3((unsigned)((n4 + 255) / 256)), dim3(256), 0, s,
                    reinterpret_cast<const float4*>(part), ks, n4, reinterpret_cast<float4*>(out));
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ src, bf16* __restrict__ dst, int64_t n) {
  pdl_trigger();
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = __float2bfloat16_rn(src[i]);
}

cudaError_t launch_f32_to_bf16(const float* src, bf16_raw* dst, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  return launch_pdl(f32_to_bf16_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, src,
                    reinterpret_cast<bf16*>(dst), n);
}

}  // namespace nimg
