// Routing and data-movement kernels of the expert-choice MoE layer.
//
//   router_prep    t_emb . W_r[d:] per sample in f64 (router.py:120-122, t half)
//                  and an f64 copy of W_r[:d]
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
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "nimg_internal.h"

namespace nimg {

// ------------------------------------------------------------------ router prep
// (a) wd[k, e] = f64(W_r[k, e]) for the x half (k < d), E padded to EP;
// (b) tb[b, e] = sum_k t_emb[b, k] * W_r[d + k, e] in f64 (the t half of the
//     concatenated router input, router.py:120-122). Block (chunk c, sample b)
//     folds one 64-row k-chunk into part[b, c, e]; the last of a sample's nkc
//     blocks (per-sample counter, armed to 0xFFFFFFFF by the caller's memset)
//     sums its chunks in ascending order -- deterministic -- and re-arms.
constexpr int RP_KCH = 64;
constexpr int RP_CONV_BLOCKS = 32;
__global__ void __launch_bounds__(64)
router_prep_kernel(const float* __restrict__ t_emb, const float* __restrict__ w_r,
                   double* __restrict__ tb, double* __restrict__ part, double* __restrict__ wd,
                   unsigned* __restrict__ counters, int B, int d, int E, int EP) {
  const int nkc = (d + RP_KCH - 1) / RP_KCH;
  if ((int)blockIdx.x >= nkc) {  // conversion blocks: grid.x == nkc + RP_CONV_BLOCKS
    const int64_t n = (int64_t)d * EP;
    const int64_t stride = (int64_t)RP_CONV_BLOCKS * gridDim.y * blockDim.x;
    for (int64_t i = ((int64_t)(blockIdx.x - nkc) * gridDim.y + blockIdx.y) * blockDim.x + threadIdx.x;
         i < n; i += stride) {
      const int64_t k = i / EP;
      const int e = (int)(i % EP);
      wd[i] = e < E ? (double)w_r[k * E + e] : 0.0;
    }
    return;
  }
  const int c = blockIdx.x, b = blockIdx.y;
  const int k0 = c * RP_KCH, k1 = min(d, k0 + RP_KCH);
  __shared__ float ts[RP_KCH];
  for (int k = k0 + threadIdx.x; k < k1; k += blockDim.x) ts[k - k0] = t_emb[(int64_t)b * d + k];
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    double acc = 0.0;
    const float* w = w_r + (int64_t)(d + k0) * E + e;
#pragma unroll 16
    for (int k = 0; k < k1 - k0; ++k) acc = fma((double)ts[k], (double)w[(int64_t)k * E], acc);
    part[((int64_t)b * nkc + c) * E + e] = acc;
  }
  __threadfence();
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(&counters[b], 1u) == (unsigned)(nkc - 2);  // from 0xFFFFFFFF
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const double* pp = part + (int64_t)b * nkc * E + e;
    double sacc = 0.0;
    for (int j = 0; j < nkc; ++j) sacc += __ldcg(pp + (int64_t)j * E);
    tb[(int64_t)b * E + e] = sacc;
  }
  if (threadIdx.x == 0) counters[b] = 0xFFFFFFFFu;
}

// ------------------------------------------------------------------ router
// FP64-pipe bound GEMM-let: logits[t, e] = sum_k x[t, k] * W[k, e] + tb[b, e].
// CTA = TM tokens x EP experts, thread = 4 tokens (strided by TG) x 8 experts
// (pairs strided by 2*EG) of f64 accumulators, so every shared load of a warp
// is a single conflict-free wavefront. K is staged in KC-chunks, double
// buffered: W (pre-converted f64) by cp.async, x by a register prefetch that
// is converted to f64 once per element.
constexpr int RT_THREADS = 128;
constexpr int RT_KC = 32;
constexpr int RT_XS = RT_KC + 2;  // x row stride (doubles): 272 B == 16 mod 128

struct RouterGeom {
  int EG, TG, TM, EP, NT;
};
__host__ __device__ inline RouterGeom router_geom(int E) {
  RouterGeom g;
  g.EG = (E + 7) / 8;
  g.EP = g.EG * 8;
  g.TG = RT_THREADS / g.EG;
  if (g.TG > 16) g.TG = 16;
  if (g.TG < 1) g.TG = 1;
  g.TM = g.TG * 4;
  g.NT = g.EG * g.TG;
  return g;
}
__host__ __device__ inline size_t router_stage_bytes(const RouterGeom& g) {
  return (size_t)RT_KC * g.EP * 8 + (size_t)g.TM * RT_XS * 8;
}
__host__ __device__ inline size_t router_smem(int E) {
  const RouterGeom g = router_geom(E);
  const size_t stage = 2 * router_stage_bytes(g);
  const size_t post = (size_t)g.TM * E * (8 + 4 + 4);  // ex (f64) + sc + lg (f32)
  return (stage > post ? stage : post) + (size_t)g.TM * 16;
}

NIMG_DEV void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
NIMG_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> NIMG_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <typename TX> struct XVec;
template <> struct XVec<bf16> { static constexpr int N = 8; };
template <> struct XVec<float> { static constexpr int N = 4; };

template <typename TX>
NIMG_DEV void cvt_store_x(double* dst, const uint4& v) {
  if constexpr (sizeof(TX) == 2) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double lo = (double)__uint_as_float(w[q] << 16);
      const double hi = (double)__uint_as_float(w[q] & 0xFFFF0000u);
      *reinterpret_cast<double2*>(dst + 2 * q) = make_double2(lo, hi);
    }
  } else {
    *reinterpret_cast<double2*>(dst) = make_double2((double)__uint_as_float(v.x), (double)__uint_as_float(v.y));
    *reinterpret_cast<double2*>(dst + 2) = make_double2((double)__uint_as_float(v.z), (double)__uint_as_float(v.w));
  }
}

template <typename TX, bool VEC>
__global__ void __launch_bounds__(RT_THREADS)
router_scores_kernel(const TX* __restrict__ x, const double* __restrict__ wd,
                     const double* __restrict__ tb, float* __restrict__ logits,
                     float* __restrict__ scores_bes, int B, int S, int d, int E) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(16) uint8_t sm[];
  const RouterGeom g = router_geom(E);
  constexpr int XV = XVec<TX>::N;            // elements per 16-B vector
  constexpr int VPR = RT_KC / XV;            // vectors per token row per chunk
  const int64_t T = (int64_t)B * S;
  const int64_t t0 = (int64_t)blockIdx.x * g.TM;
  const size_t SB = router_stage_bytes(g);
  auto wsb = [&](int buf) { return reinterpret_cast<double*>(sm + buf * SB); };
  auto xsb = [&](int buf) { return reinterpret_cast<double*>(sm + buf * SB + (size_t)RT_KC * g.EP * 8); };

  const int tid = threadIdx.x;
  const bool active = tid < g.NT;
  const int tg = active ? tid / g.EG : 0, eg = active ? tid % g.EG : 0;
  const int nvec_x = g.TM * VPR;             // x vectors per chunk
  const int nvec_w = RT_KC * g.EP / 2;       // 16-B W vectors per chunk
  const int nc = (d + RT_KC - 1) / RT_KC;

  // x prefetch registers: TM <= 64 tokens x RT_KC / XV vectors over RT_THREADS threads
  constexpr int XR = 64 * RT_KC / XV / RT_THREADS;
  uint4 xr[XR];
  auto load_x = [&](int c) {
    const int k0 = c * RT_KC;
#pragma unroll
    for (int r = 0; r < XR; ++r) {
      const int i = tid + r * RT_THREADS;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (i < nvec_x) {
        const int tok = i / VPR, kv = i % VPR;
        const int64_t t = t0 + tok;
        const int k = k0 + kv * XV;
        if (t < T) {
          if (VEC) {
            if (k < d) v = __ldg(reinterpret_cast<const uint4*>(x + t * d + k));
          } else {
            TX tmp[XV];
#pragma unroll
            for (int q = 0; q < XV; ++q) tmp[q] = (k + q < d) ? x[t * d + k + q] : from_f32<TX>(0.f);
            v = *reinterpret_cast<uint4*>(tmp);
          }
        }
      }
      xr[r] = v;
    }
  };
  auto store_x = [&](int buf) {
    double* xs = xsb(buf);
#pragma unroll
    for (int r = 0; r < XR; ++r) {
      const int i = tid + r * RT_THREADS;
      if (i < nvec_x) {
        const int tok = i / VPR, kv = i % VPR;
        cvt_store_x<TX>(xs + tok * RT_XS + kv * XV, xr[r]);
      }
    }
  };
  auto load_w = [&](int c, int buf) {
    const int k0 = c * RT_KC;
    double* ws = wsb(buf);
    for (int i = tid; i < nvec_w; i += RT_THREADS) {
      const int kk = (2 * i) / g.EP, e = (2 * i) % g.EP;
      if (k0 + kk < d) cp_async16(ws + kk * g.EP + e, wd + (int64_t)(k0 + kk) * g.EP + e);
      else *reinterpret_cast<double2*>(ws + kk * g.EP + e) = make_double2(0.0, 0.0);
    }
  };

  double acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;

  load_x(0);
  load_w(0, 0);
  cp_async_commit();
  store_x(0);
  for (int c = 0; c < nc; ++c) {
    const int buf = c & 1;
    if (c + 1 < nc) {
      load_x(c + 1);
      load_w(c + 1, buf ^ 1);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (active) {
      const double* xs = xsb(buf);
      const double* ws = wsb(buf);
#pragma unroll 4
      for (int kk = 0; kk < RT_KC; kk += 2) {
        double2 xv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          xv[i] = *reinterpret_cast<const double2*>(xs + (tg + g.TG * i) * RT_XS + kk);
        double2 w0[4], w1[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          w0[q] = *reinterpret_cast<const double2*>(ws + kk * g.EP + 2 * eg + 2 * g.EG * q);
          w1[q] = *reinterpret_cast<const double2*>(ws + (kk + 1) * g.EP + 2 * eg + 2 * g.EG * q);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            acc[i][2 * q] = fma(xv[i].x, w0[q].x, acc[i][2 * q]);
            acc[i][2 * q + 1] = fma(xv[i].x, w0[q].y, acc[i][2 * q + 1]);
            acc[i][2 * q] = fma(xv[i].y, w1[q].x, acc[i][2 * q]);
            acc[i][2 * q + 1] = fma(xv[i].y, w1[q].y, acc[i][2 * q + 1]);
          }
      }
    }
    if (c + 1 < nc) store_x(buf ^ 1);
    __syncthreads();
  }

  // ---- epilogue (reuses the staging smem): fp32 logits, f64 softmax
  double* ex = reinterpret_cast<double*>(sm);                           // [TM][E]
  float* sc = reinterpret_cast<float*>(sm + (size_t)g.TM * E * 8);      // [TM][E]
  float* lg = sc + (size_t)g.TM * E;                                    // [TM][E]
  double* mx = reinterpret_cast<double*>(sm + (router_smem(E) - (size_t)g.TM * 16));
  double* sum = mx + g.TM;
  if (active) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int tok = tg + g.TG * i;
      const int64_t t = t0 + tok;
      if (t >= T) continue;
      const int64_t b = t / S;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int e = 2 * eg + 2 * g.EG * (j >> 1) + (j & 1);
        // matmul f64 -> fp32 (tensor.py:286-287)
        if (e < E) lg[tok * E + e] = (float)(acc[i][j] + tb[b * E + e]);
      }
    }
  }
  __syncthreads();
  for (int tok = tid; tok < g.TM; tok += RT_THREADS) {
    double m = -INFINITY;
    for (int e = 0; e < E; ++e) m = fmax(m, (double)lg[tok * E + e]);
    mx[tok] = m;
  }
  __syncthreads();
  for (int i = tid; i < g.TM * E; i += RT_THREADS) ex[i] = exp((double)lg[i] - mx[i / E]);
  __syncthreads();
  for (int tok = tid; tok < g.TM; tok += RT_THREADS) sum[tok] = np_pairwise_sum(ex + tok * E, E);
  __syncthreads();
  for (int i = tid; i < g.TM * E; i += RT_THREADS) sc[i] = (float)(ex[i] / sum[i / E]);
  __syncthreads();
  for (int i = tid; i < g.TM * E; i += RT_THREADS) {
    const int64_t t = t0 + i / E;
    if (t < T) logits[t * E + (i % E)] = lg[i];
  }
  for (int i = tid; i < g.TM * E; i += RT_THREADS) {
    const int e = i / g.TM, tok = i % g.TM;
    const int64_t t = t0 + tok;
    if (t < T) {
      const int64_t b = t / S, s = t % S;
      scores_bes[(b * E + e) * S + s] = sc[tok * E + e];
    }
  }
}

// ------------------------------------------------------------------ router (DMMA, E <= 64)
// Same contraction on the FP64 tensor pipe: mma.sync m8n8k4 f64 (one
// instruction = 256 f64 FMAs). CTA = 4 warps x 16 tokens, all 64 (padded)
// experts; warp tile = 2 x 8 fragments of 8x8, 32 f64 accumulators per lane.
// Staging strides make every fragment load an optimal 2-wavefront LDS.64:
// x rows of 36 doubles (288 B == 32 mod 128), W rows of 72 doubles (576 B ==
// 64 mod 128).
constexpr int DM_TM = 64, DM_KC = 32, DM_XS = 36, DM_WS = 72, DM_EP = 64;
// Router prep for the DMMA router (E <= 64), one short kernel, no counters:
// blocks [0, B * KS): block (b, ks) sums its k-range of the t half
// part[b, ks, e] = sum_k t_emb[b, k] * W_r[d + k, e] in f64 (router.py:120-122)
// -- thread (e, q) sums one of 4 sub-slices, folded in a fixed order; the
// scores kernel folds the KS partials per sample in ks order (deterministic).
// Blocks [B * KS, + RP2_CONV) write wd[k, e] = f64(W_r[k, e]) for the x half,
// E padded to 64. Short dependent chains: the kernel is latency-bound.
constexpr int RP2_CONV = 64;
__host__ __device__ inline int rp2_ks(int d) { return router_tpart_ks(d); }
__global__ void __launch_bounds__(256)
router_prep_dmma_kernel(const float* __restrict__ t_emb, const float* __restrict__ w_r,
                        double* __restrict__ part, double* __restrict__ wd, int B, int d, int E) {
  pdl_trigger();
  const int KS = rp2_ks(d);
  if ((int)blockIdx.x >= B * KS) {
    const int64_t n = (int64_t)d * DM_EP;
    const int64_t stride = (int64_t)RP2_CONV * blockDim.x;
    for (int64_t i = (int64_t)(blockIdx.x - B * KS) * blockDim.x + threadIdx.x; i < n; i += stride) {
      const int64_t k = i / DM_EP;
      const int e = (int)(i % DM_EP);
      wd[i] = e < E ? (double)__ldg(w_r + k * E + e) : 0.0;
    }
    return;
  }
  router_tpart_block(t_emb, w_r, part, blockIdx.x / KS, blockIdx.x % KS, d, E);
}

__host__ __device__ inline size_t dmma_stage_bytes() {
  return (size_t)DM_KC * DM_WS * 8 + (size_t)DM_TM * DM_XS * 8;
}
// epilogue smem: ex/sc/lg (TM * E * 16) + folded t-bias of the <= TM samples a
// CTA can span (TM * E * 8) + max/sum (TM * 16)
__host__ __device__ inline size_t dmma_tbs_offset(int E) { return (size_t)DM_TM * E * 16; }
__host__ __device__ inline size_t dmma_router_smem(int E) {
  const size_t stage = 2 * dmma_stage_bytes();
  const size_t post = (size_t)DM_TM * E * (8 + 4 + 4) + (size_t)DM_TM * E * 8;
  const size_t need = (stage > post ? stage : post) + (size_t)DM_TM * 16;
  // The grid is sized for exactly 2 CTAs per SM; registers and 74 KB would
  // admit 3, and a CTA placed early (PDL) on a half-busy GPU would then stack
  // 3 on some SMs and 1 on others. >= 76 KB caps residency at 2 per SM.
  constexpr size_t kTwoPerSm = 76 * 1024;
  return need > kTwoPerSm ? need : kTwoPerSm;
}

NIMG_DEV void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <typename TX, bool VEC>
__global__ void __launch_bounds__(128)
router_scores_dmma_kernel(const TX* __restrict__ x, const double* __restrict__ wd,
                          const double* __restrict__ part, float* __restrict__ logits,
                          float* __restrict__ scores_bes, int B, int S, int d, int E,
                          int frags_per_cta) {
  // PDL secondary of router_prep_dmma_kernel: only the layer input x_norm is
  // read before pdl_wait(); wd and the t-bias partials come from the prep.
  pdl_trigger();
  // CTA c owns 8-row fragments [c*fpc, (c+1)*fpc) (fpc <= 8); the grid is sized
  // to whole multiples of the SM count (>= 2 CTAs per SM) so per-SM DMMA work
  // is balanced. Warp w computes fragments w and w+4 of the CTA (when present).
  extern __shared__ __align__(16) uint8_t sm[];
  constexpr int XV = XVec<TX>::N;
  constexpr int VPR = DM_KC / XV;
  constexpr int XR = DM_TM * VPR / 128;
  constexpr int WR = DM_KC * DM_EP / 2 / 128;
  const int64_t T = (int64_t)B * S;
  const int64_t t0 = (int64_t)blockIdx.x * frags_per_cta * 8;
  const int64_t rows_left = T - t0;
  const int rows = (int)(rows_left < (int64_t)frags_per_cta * 8 ? rows_left : (int64_t)frags_per_cta * 8);
  const size_t SB = dmma_stage_bytes();
  auto wsb = [&](int buf) { return reinterpret_cast<double*>(sm + buf * SB); };
  auto xsb = [&](int buf) { return reinterpret_cast<double*>(sm + buf * SB + (size_t)DM_KC * DM_WS * 8); };
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nc = (d + DM_KC - 1) / DM_KC;
  const int nfr = (rows + 7) / 8;
  const bool has0 = warp < nfr, has1 = warp + 4 < nfr;

  uint4 xr[XR];
  auto load_x = [&](int c) {
    const int k0 = c * DM_KC;
#pragma unroll
    for (int r = 0; r < XR; ++r) {
      const int i = tid + r * 128;
      const int tok = i / VPR, kv = i % VPR;
      const int k = k0 + kv * XV;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (tok < rows) {
        const int64_t t = t0 + tok;
        if (VEC) {
          if (k < d) v = __ldg(reinterpret_cast<const uint4*>(x + t * d + k));
        } else {
          TX tmp[XV];
#pragma unroll
          for (int q = 0; q < XV; ++q) tmp[q] = (k + q < d) ? x[t * d + k + q] : from_f32<TX>(0.f);
          v = *reinterpret_cast<uint4*>(tmp);
        }
      }
      xr[r] = v;
    }
  };
  auto store_x = [&](int buf) {
    double* xs = xsb(buf);
#pragma unroll
    for (int r = 0; r < XR; ++r) {
      const int i = tid + r * 128;
      cvt_store_x<TX>(xs + (i / VPR) * DM_XS + (i % VPR) * XV, xr[r]);
    }
  };
  auto load_w = [&](int c, int buf) {
    const int k0 = c * DM_KC;
    double* ws = wsb(buf);
#pragma unroll
    for (int r = 0; r < WR; ++r) {
      const int i = tid + r * 128;
      const int kk = i / (DM_EP / 2), e = (i % (DM_EP / 2)) * 2;
      if (k0 + kk < d) cp_async16(ws + kk * DM_WS + e, wd + (int64_t)(k0 + kk) * DM_EP + e);
      else *reinterpret_cast<double2*>(ws + kk * DM_WS + e) = make_double2(0.0, 0.0);
    }
  };

  double acc[2][8][2];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int n = 0; n < 8; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;

  const int ar = lane >> 2, ac = lane & 3;   // A frag: (row, k); B frag: (k = ac, col = ar)
  load_x(0);
  pdl_wait();   // prep kernel complete: wd and tb are ready
  load_w(0, 0);
  cp_async_commit();
  store_x(0);
  for (int c = 0; c < nc; ++c) {
    const int buf = c & 1;
    if (c + 1 < nc) {
      load_x(c + 1);
      load_w(c + 1, buf ^ 1);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* xs = xsb(buf) + (warp * 8 + ar) * DM_XS + ac;
    const double* ws = wsb(buf) + ac * DM_WS + ar;
    if (has0) {
#pragma unroll
      for (int k4 = 0; k4 < DM_KC; k4 += 4) {
        const double a0 = xs[k4];
        const double a1 = has1 ? xs[32 * DM_XS + k4] : 0.0;   // fragment w+4
        double bf[8];
#pragma unroll
        for (int n = 0; n < 8; ++n) bf[n] = ws[k4 * DM_WS + n * 8];
#pragma unroll
        for (int n = 0; n < 8; ++n) dmma_8x8x4(acc[0][n][0], acc[0][n][1], a0, bf[n]);
        if (has1) {
#pragma unroll
          for (int n = 0; n < 8; ++n) dmma_8x8x4(acc[1][n][0], acc[1][n][1], a1, bf[n]);
        }
      }
    }
    if (c + 1 < nc) store_x(buf ^ 1);
    __syncthreads();
  }

  // t-bias of the samples this CTA spans: fold the prep's KS partials in ks
  // order (deterministic) into smem once (the staging buffers are free now)
  const int64_t b_first = t0 / S;
  const int nb = (int)((t0 + rows - 1) / S - b_first + 1);
  double* tbs = reinterpret_cast<double*>(sm + dmma_tbs_offset(E));
  {
    for (int i = tid; i < nb * E; i += 128) tbs[i] = router_tbias(part, b_first + i / E, i % E, d, E);
  }
  __syncthreads();

  if (E == DM_EP) {
    // ---- register epilogue (E == 64). Lane (ar, ac) holds, for row ar of each
    // fragment, columns n*8 + 2*ac + j. numpy's pairwise sum over 64 terms uses
    // accumulators r[c mod 8] folded ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)); each
    // r[c mod 8] lives in one lane (summed over n in order), so two xor-shuffles
    // reproduce the exact order (IEEE add is commutative).
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      if (!(m == 0 ? has0 : has1)) continue;
      const int tok = (warp + 4 * m) * 8 + ar;
      const bool tv = tok < rows;
      const int64_t t = t0 + (tv ? tok : 0);
      const int64_t b = t / S, srow = t % S;
      float lg[8][2];
      double mx = -INFINITY;
#pragma unroll
      for (int n = 0; n < 8; ++n)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int e = n * 8 + 2 * ac + j;
          lg[n][j] = (float)(acc[m][n][j] + tbs[(b - b_first) * E + e]);   // tensor.py:286-287
          mx = fmax(mx, (double)lg[n][j]);
        }
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      double ex[8][2], r[2] = {0.0, 0.0};
#pragma unroll
      for (int n = 0; n < 8; ++n)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          ex[n][j] = exp((double)lg[n][j] - mx);
          r[j] = n == 0 ? ex[n][j] : r[j] + ex[n][j];
        }
      double q = r[0] + r[1];
      q = q + __shfl_xor_sync(0xffffffffu, q, 1);
      const double sum = q + __shfl_xor_sync(0xffffffffu, q, 2);
      if (tv) {
#pragma unroll
        for (int n = 0; n < 8; ++n) {
          *reinterpret_cast<float2*>(logits + t * E + n * 8 + 2 * ac) = make_float2(lg[n][0], lg[n][1]);
#pragma unroll
          for (int j = 0; j < 2; ++j)
            scores_bes[(b * E + n * 8 + 2 * ac + j) * S + srow] = (float)(ex[n][j] / sum);
        }
      }
    }
    return;
  }

  // ---- general epilogue (E < 64) through smem (reuses the staging buffers)
  double* ex = reinterpret_cast<double*>(sm);
  float* sc = reinterpret_cast<float*>(sm + (size_t)DM_TM * E * 8);
  float* lg = sc + (size_t)DM_TM * E;
  double* mx = reinterpret_cast<double*>(sm + (dmma_router_smem(E) - (size_t)DM_TM * 16));
  double* sum = mx + DM_TM;
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    const int tok = (warp + 4 * m) * 8 + ar;
    if (tok < rows) {
      const int64_t b = (t0 + tok) / S;
#pragma unroll
      for (int n = 0; n < 8; ++n)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int e = n * 8 + ac * 2 + j;
          if (e < E) lg[tok * E + e] = (float)(acc[m][n][j] + tbs[(b - b_first) * E + e]);  // tensor.py:286-287
        }
    }
  }
  __syncthreads();
  for (int tok = tid; tok < rows; tok += 128) {
    double mv = -INFINITY;
    for (int e = 0; e < E; ++e) mv = fmax(mv, (double)lg[tok * E + e]);
    mx[tok] = mv;
  }
  __syncthreads();
  for (int i = tid; i < rows * E; i += 128) ex[i] = exp((double)lg[i] - mx[i / E]);
  __syncthreads();
  for (int tok = tid; tok < rows; tok += 128) sum[tok] = np_pairwise_sum(ex + tok * E, E);
  __syncthreads();
  for (int i = tid; i < rows * E; i += 128) sc[i] = (float)(ex[i] / sum[i / E]);
  __syncthreads();
  for (int i = tid; i < rows * E; i += 128) logits[(t0 + i / E) * E + (i % E)] = lg[i];
  for (int i = tid; i < rows * E; i += 128) {
    const int e = i / rows, tok = i % rows;
    const int64_t t = t0 + tok;
    const int64_t b = t / S, sr = t % S;
    scores_bes[(b * E + e) * S + sr] = sc[tok * E + e];
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
                 int cap, int* __restrict__ cursor) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int P = next_pow2(cap);
  uint64_t* win = reinterpret_cast<uint64_t*>(sm);                  // [P]
  uint32_t* keys = reinterpret_cast<uint32_t*>(sm + (size_t)P * 8);  // [S]
  uint32_t* hist = keys + S;                                        // [256]
  int* scratch = reinterpret_cast<int*>(hist + 256);                // [64]
  __shared__ uint32_t s_digit;
  __shared__ int s_k;

  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.x, e = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (cursor && e == 0 && tid == 0) cursor[b] = 0;
  const float* col = scores_bes + ((int64_t)b * E + e) * S;
  for (int i = tid; i < S; i += SEL_THREADS) keys[i] = score_key(col[i]);

  // ---- radix select of the cap-th largest key, 8 bits per pass from the MSB
  uint32_t prefix = 0, pmask = 0;
  int k = cap;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += SEL_THREADS) hist[i] = 0;
    __syncthreads();
    // warp-aggregated histogram: near-uniform router scores put most keys in
    // one bin, so per-element smem atomics would serialise on one address
    for (int i0 = 0; i0 < S; i0 += SEL_THREADS) {
      const int i = i0 + tid;
      const uint32_t key = i < S ? keys[i] : 0u;
      const bool cand = i < S && (key & pmask) == prefix;
      const uint32_t dig = (key >> shift) & 255u;
      const unsigned grp = __match_any_sync(0xffffffffu, cand ? dig : 0xFFFFFFFFu);
      if (cand && lane == __ffs(grp) - 1) atomicAdd(&hist[dig], (unsigned)__popc(grp));
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
  // keys[] is free from here on: it becomes this column's slot table
  for (int i = tid; i < S; i += SEL_THREADS) keys[i] = 0xFFFFFFFFu;

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
  for (int j = tid; j < cap; j += SEL_THREADS) {
    const uint32_t idx = 0xFFFFFFFFu - (uint32_t)(win[j] & 0xFFFFFFFFull);
    const int64_t o = ((int64_t)e * B + b) * cap + j;
    token_flat[o] = (int32_t)((int64_t)b * S + idx);
    gate_raw[o] = col[idx];
    keys[idx] = (uint32_t)j;
  }
  __syncthreads();
  // the whole (b, e) column of the slot table, -1 where not selected: no
  // separate arming pass over the workspace
  int16_t* scol = slot_of + ((int64_t)b * E + e) * S;
  for (int i = tid; i < S; i += SEL_THREADS) scol[i] = (int16_t)(int32_t)keys[i];
}

// ------------------------------------------------------------------ select, block per column
// One 128-thread block per (b, e) column with the keys in registers (warp w
// holds tokens [w S/4, (w+1) S/4), lane l of it tokens l + 32 j): the cap-th
// largest key is found MSB-first, two bits per step (16 steps, three
// candidate counts per step, one redux.sync each, the four warps' counts
// summed through shared memory behind one barrier). The winners are every key
// > thr plus the first (cap - #gt) keys == thr in token order, then one warp
// sorts them by (score desc, index asc) -- the order of argsort(-x,
// kind="stable")[:cap] (router.py:98-101). Padding keys are 0 (= NaN's key)
// with indices >= S, so they rank after every real element and are never
// taken (cap <= S).
constexpr int SB_WARPS = 4;
#ifndef NIMG_SEL_R8
#define NIMG_SEL_R8 1
#endif
template <int KPL>
__global__ void __launch_bounds__(SB_WARPS * 32)
ec_select_blk_kernel(const float* __restrict__ scores_bes, int32_t* __restrict__ token_flat,
                     float* __restrict__ gate_raw, int16_t* __restrict__ slot_of, int B, int S,
                     int E, int cap, int P, int* __restrict__ cursor,
                     unsigned long long* __restrict__ tokmask, int2* __restrict__ tokent) {
  extern __shared__ __align__(16) uint64_t wsel[];   // [P] winners
  __shared__ int red[2][SB_WARPS][4];
  __shared__ int wcnt[SB_WARPS][2];
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int col = blockIdx.x;                         // b * E + e: scores_bes is (B, E, S)
  const int b = col / E, e = col - b * E;
  if (cursor && e == 0 && threadIdx.x == 0) cursor[b] = 0;   // gate_tile's row allocator
  const float* c = scores_bes + (int64_t)col * S;
  const int i0 = warp * 32 * KPL + lane;              // token of key[0]
  uint32_t key[KPL];
#pragma unroll
  for (int j = 0; j < KPL; ++j) {
    const int i = i0 + 32 * j;
    key[j] = i < S ? score_key(__ldg(c + i)) : 0u;
  }
  // bits every key of the column shares (router scores cluster near 1/E, so
  // the sign and most exponent bits agree): the search starts below them
  uint32_t kand = 0xFFFFFFFFu, kor = 0u;
#pragma unroll
  for (int j = 0; j < KPL; ++j) {
    if (i0 + 32 * j < S) { kand &= key[j]; kor |= key[j]; }
  }
  kand = __reduce_and_sync(0xffffffffu, kand);
  kor = __reduce_or_sync(0xffffffffu, kor);
  if (lane == 0) { red[0][warp][0] = (int)kand; red[1][warp][0] = (int)kor; }
  __syncthreads();
  kand = 0xFFFFFFFFu;
  kor = 0u;
#pragma unroll
  for (int w = 0; w < SB_WARPS; ++w) { kand &= (uint32_t)red[0][w][0]; kor |= (uint32_t)red[1][w][0]; }
  const uint32_t diff = kand ^ kor;        // bits that differ somewhere in the column
  const int top = diff ? 31 - __clz(diff) : -1;
  // every key agrees above bit `top`: the cap-th largest key has those bits
  uint32_t thr = top < 0 ? kand : (top >= 31 ? 0u : (kand & ~((2u << top) - 1u)));
#if NIMG_SEL_R8
  // Radix search, 8 bits per pass below the common prefix: every key that
  // still matches the prefix bumps a shared-memory histogram bin; warp 0 scans
  // the 256 bins from the top for the bin holding the need-th largest key,
  // zeroes the other histogram and publishes (digit, keys above it). Two
  // barriers per pass, ceil((top + 1) / 8) passes.
  __shared__ int hist[2][256];
  __shared__ int rres[2];
  for (int i = threadIdx.x; i < 512; i += SB_WARPS * 32) (&hist[0][0])[i] = 0;
  __syncthreads();   // red[] free, histograms zeroed
  int need = cap;
#pragma unroll 1
  for (int rem = top + 1, buf = 0; rem > 0; buf ^= 1) {
    const int nb = rem < 8 ? rem : 8, sh = rem - nb, hi = rem;
#pragma unroll
    for (int j = 0; j < KPL; ++j) {
      const bool match = hi >= 32 || ((key[j] ^ thr) >> hi) == 0u;
      if (match) atomicAdd(&hist[buf][(key[j] >> sh) & ((1u << nb) - 1u)], 1);
    }
    __syncthreads();
    if (warp == 0) {
      int c[8], ls = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {   // lane l: bins 255 - 8 l - i, descending
        c[i] = hist[buf][255 - 8 * lane - i];
        ls += c[i];
        hist[buf ^ 1][8 * lane + i] = 0;
      }
      int incl = ls;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const int excl = incl - ls;
      if (excl < need && incl >= need) {
        int run = excl, dsel = 0, above = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (run < need && run + c[i] >= need) { dsel = 255 - 8 * lane - i; above = run; }
          run += c[i];
        }
        rres[0] = dsel;
        rres[1] = above;
      }
    }
    __syncthreads();
    thr |= (uint32_t)rres[0] << sh;
    need -= rres[1];
    rem = sh;
  }
#else
  const int sh0 = top < 0 ? -2 : (top | 1) - 1;   // first 2-bit step covering bit `top`
  __syncthreads();   // red[] reused by the search
#pragma unroll 1
  for (int sh = sh0, buf = 0; sh >= 0; sh -= 2, buf ^= 1) {
    int n1 = 0, n2 = 0, n3 = 0;
#pragma unroll
    for (int j = 0; j < KPL; ++j) {
      n1 += key[j] >= (thr | (1u << sh)) ? 1 : 0;
      n2 += key[j] >= (thr | (2u << sh)) ? 1 : 0;
      n3 += key[j] >= (thr | (3u << sh)) ? 1 : 0;
    }
    n1 = (int)__reduce_add_sync(0xffffffffu, (unsigned)n1);
    n2 = (int)__reduce_add_sync(0xffffffffu, (unsigned)n2);
    n3 = (int)__reduce_add_sync(0xffffffffu, (unsigned)n3);
    if (lane == 0) { red[buf][warp][1] = n1; red[buf][warp][2] = n2; red[buf][warp][3] = n3; }
    __syncthreads();   // double-buffered counts: one barrier per step
    int t1 = 0, t2 = 0, t3 = 0;
#pragma unroll
    for (int w = 0; w < SB_WARPS; ++w) { t1 += red[buf][w][1]; t2 += red[buf][w][2]; t3 += red[buf][w][3]; }
    thr |= (t3 >= cap ? 3u : t2 >= cap ? 2u : t1 >= cap ? 1u : 0u) << sh;
  }
#endif
  int n_gt = 0, n_eq = 0;
#pragma unroll
  for (int j = 0; j < KPL; ++j) { n_gt += key[j] > thr ? 1 : 0; n_eq += key[j] == thr ? 1 : 0; }
  n_gt = (int)__reduce_add_sync(0xffffffffu, (unsigned)n_gt);
  n_eq = (int)__reduce_add_sync(0xffffffffu, (unsigned)n_eq);
  if (lane == 0) { wcnt[warp][0] = n_gt; wcnt[warp][1] = n_eq; }
  __syncthreads();
  int gt_all = 0, eq_before = 0, w_before = 0;
#pragma unroll
  for (int w = 0; w < SB_WARPS; ++w) gt_all += wcnt[w][0];
  const int need_eq = cap - gt_all;
  for (int w = 0; w < warp; ++w) {
    eq_before += wcnt[w][1];
    w_before += wcnt[w][0] + max(0, min(wcnt[w][1], need_eq - (eq_before - wcnt[w][1])));
  }
  const unsigned lt = (1u << lane) - 1u;
  int n_w = w_before;
#pragma unroll
  for (int j = 0; j < KPL; ++j) {
    const bool eq = key[j] == thr;
    const unsigned me = __ballot_sync(0xffffffffu, eq);
    const bool take = key[j] > thr || (eq && eq_before + __popc(me & lt) < need_eq);
    const unsigned mt = __ballot_sync(0xffffffffu, take);
    if (take)
      wsel[n_w + __popc(mt & lt)] =
          ((uint64_t)key[j] << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)(i0 + 32 * j));
    n_w += __popc(mt);
    eq_before += __popc(me);
  }
  for (int i = cap + threadIdx.x; i < P; i += SB_WARPS * 32) wsel[i] = 0ull;
  // the column of the slot table: -1, then the winners' slots (after the sort)
  int16_t* scol = slot_of + (int64_t)col * S;
  for (int i = threadIdx.x; i < S; i += SB_WARPS * 32) scol[i] = (int16_t)-1;
  __syncthreads();
  // bitonic sort of P composite keys, descending, by all warps
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P / 2; i += SB_WARPS * 32) {
        const int a = 2 * i - (i & (stride - 1));
        const int cc = a + stride;
        const bool desc = (a & size) == 0;
        const uint64_t va = wsel[a], vc = wsel[cc];
        if ((va < vc) == desc) { wsel[a] = vc; wsel[cc] = va; }
      }
      if (P > 64) __syncthreads(); else __syncwarp();
    }
  }
  if (P <= 64 && warp != 0) return;   // the sort ran in warp 0 alone (P/2 <= 32 pairs)
  for (int j = threadIdx.x; j < cap; j += (P <= 64 ? 32 : SB_WARPS * 32)) {
    const uint32_t idx = 0xFFFFFFFFu - (uint32_t)(wsel[j] & 0xFFFFFFFFull);
    const int64_t o = ((int64_t)e * B + b) * cap + j;
    token_flat[o] = (int32_t)((int64_t)b * S + idx);
    gate_raw[o] = c[idx];
    scol[idx] = (int16_t)j;
    if (tokmask) {
      const int64_t tt = (int64_t)b * S + idx;
      tokent[tt * E + e] = make_int2((int32_t)o, __float_as_int(c[idx]));
      atomicOr(tokmask + tt, 1ull << e);
    }
  }
}

// ------------------------------------------------------------------ gates, tile of 32 tokens
// One block per 32 consecutive tokens of one sample (router.py:137-143): the
// (B, E, S) slot table and scores are read coalesced (32 tokens of one expert
// per warp load) and transposed through shared memory; then warp per token as
// gate_norm_kernel: the selecting experts in ascending order (ballot prefix),
// totals = fp32(sequential f64 sum -- the np.add.at order), den = fp32(f64(tot)
// + f64(fp32 eps)), gate = fp32(f64(fp32(f64(raw) / f64(den))) * f64(fp32
// alpha)); the per-token combine list.
constexpr int GT_TOK = 32, GT_THREADS = 256;
__global__ void __launch_bounds__(GT_THREADS)
gate_tile_kernel(const float* __restrict__ scores_bes, const int16_t* __restrict__ slot_of,
                 float* __restrict__ gates, int32_t* __restrict__ comb_rows,
                 int32_t* __restrict__ comb_cnt, int B, int S, int E, int cap, float eps32,
                 float alpha32, int* __restrict__ bg_flags, int n_bg_flags, TokOrder tko) {
  extern __shared__ __align__(16) uint8_t gsm[];
  constexpr int NW = GT_THREADS / 32;
  int16_t* sl = reinterpret_cast<int16_t*>(gsm);                                  // [E][32]
  const size_t o1 = ((size_t)E * GT_TOK * 2 + 15) & ~size_t(15);
  float* raw = reinterpret_cast<float*>(gsm + o1);                               // [E][32]
  float* raw_l = raw + (size_t)E * GT_TOK;                                       // [NW][E]
  int32_t* row_l = reinterpret_cast<int32_t*>(raw_l + (size_t)NW * E);           // [NW][E]
  pdl_trigger();
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_bg_flags;
       i += (int64_t)gridDim.x * blockDim.x)
    bg_flags[i] = 0;
  const int tiles_per_b = (S + GT_TOK - 1) / GT_TOK;
  const int b = blockIdx.x / tiles_per_b;
  const int s0 = (blockIdx.x - b * tiles_per_b) * GT_TOK;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool in = s0 + lane < S;
  for (int e = warp; e < E; e += NW) {
    const int64_t o = ((int64_t)b * E + e) * S + s0 + lane;
    const int16_t j = in ? slot_of[o] : (int16_t)-1;
    sl[e * GT_TOK + lane] = j;
    raw[e * GT_TOK + lane] = (in && j >= 0) ? scores_bes[o] : 0.f;
  }
  __shared__ int tcnt[GT_TOK], toff[GT_TOK];
  if (tko.tok_off) {
    // token-ordered layout: this tile's rows get a contiguous range of its
    // sample's E * cap rows (tiles in any order: per-sample atomic cursor)
    __syncthreads();
    for (int tok = warp; tok < GT_TOK; tok += NW) {
      int n = 0;
      if (s0 + tok < S)
        for (int e0 = 0; e0 < E; e0 += 32) {
          const int e = e0 + lane;
          n += __popc(__ballot_sync(0xffffffffu, e < E && sl[e * GT_TOK + tok] >= 0));
        }
      if (lane == 0) tcnt[tok] = n;
    }
    __syncthreads();
    if (warp == 0) {
      const int n = tcnt[lane];
      int incl = n;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      int base = 0;
      if (lane == 31) base = atomicAdd(tko.cursor + b, incl);
      base = __shfl_sync(0xffffffffu, base, 31);
      toff[lane] = (int)((int64_t)b * E * cap) + base + incl - n;
    }
  }
  __syncthreads();
  float* rl = raw_l + (size_t)warp * E;
  int32_t* ro = row_l + (size_t)warp * E;
  for (int tok = warp; tok < GT_TOK && s0 + tok < S; tok += NW) {
    const int64_t t = (int64_t)b * S + s0 + tok;
    int cnt = 0;
    for (int e0 = 0; e0 < E; e0 += 32) {
      const int e = e0 + lane;
      const int j = e < E ? (int)sl[e * GT_TOK + tok] : -1;
      const unsigned m = __ballot_sync(0xffffffffu, j >= 0);
      if (j >= 0) {
        const int pos = cnt + __popc(m & ((1u << lane) - 1u));
        rl[pos] = raw[e * GT_TOK + tok];
        ro[pos] = (int32_t)(((int64_t)e * B + b) * cap + j);
      }
      cnt += __popc(m);
    }
    __syncwarp();
    double tot = 0.0;
    if (lane == 0)
      for (int k = 0; k < cnt; ++k) tot += (double)rl[k];
    const float tot32 = __shfl_sync(0xffffffffu, (float)tot, 0);
    const float den = (float)((double)tot32 + (double)eps32);
    for (int k = lane; k < cnt; k += 32) {
      const float q = (float)((double)rl[k] / (double)den);
      const float gk = (float)((double)q * (double)alpha32);
      gates[ro[k]] = gk;
      comb_rows[t * E + k] = ro[k];
      if (tko.tok_off) {
        const int o = toff[tok] + k;
        tko.row_map[ro[k]] = o;
        tko.gate_tok[o] = gk;
      }
    }
    if (lane == 0) {
      comb_cnt[t] = cnt;
      if (tko.tok_off) tko.tok_off[t] = toff[tok];
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ gates
// Warp per token (router.py:137-143): the experts that picked the token, in
// ascending order (ballot + prefix), totals = fp32(sequential f64 sum in that
// order -- np.add.at order), den = fp32(f64(tot) + f64(fp32 eps)),
// gate = fp32(f64(fp32(f64(raw) / f64(den))) * f64(fp32 alpha)). Also emits
// the per-token combine list (rows of the expert-major flat order).
constexpr int GN_WARPS = 8;
__global__ void __launch_bounds__(GN_WARPS * 32)
gate_norm_kernel(const float* __restrict__ scores_bes, const int16_t* __restrict__ slot_of,
                 float* __restrict__ gates, int32_t* __restrict__ comb_rows,
                 int32_t* __restrict__ comb_cnt, int B, int S, int E, int cap, float eps32,
                 float alpha32, int* __restrict__ bg_flags, int n_bg_flags) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* raw_l = reinterpret_cast<float*>(sm) + (size_t)warp * E;
  int32_t* row_l = reinterpret_cast<int32_t*>(sm + (size_t)GN_WARPS * E * 4) + (size_t)warp * E;
  pdl_trigger();
  pdl_wait();
  // arm the next GEMM1's background-gather flags (it waits on this kernel)
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_bg_flags;
       i += (int64_t)gridDim.x * blockDim.x)
    bg_flags[i] = 0;
  const int64_t T = (int64_t)B * S;
  const int64_t t = (int64_t)blockIdx.x * GN_WARPS + warp;
  if (t >= T) return;
  const int64_t b = t / S, s = t % S;
  int cnt = 0;
  for (int e0 = 0; e0 < E; e0 += 32) {
    const int e = e0 + lane;
    const int j = e < E ? (int)slot_of[(b * E + e) * S + s] : -1;   // slot table (B, E, S)
    const unsigned m = __ballot_sync(0xffffffffu, j >= 0);
    if (j >= 0) {
      const int pos = cnt + __popc(m & ((1u << lane) - 1u));
      raw_l[pos] = scores_bes[(b * E + e) * S + s];
      row_l[pos] = (int32_t)(((int64_t)e * B + b) * cap + j);
    }
    cnt += __popc(m);
  }
  __syncwarp();
  double tot = 0.0;
  if (lane == 0)
    for (int k = 0; k < cnt; ++k) tot += (double)raw_l[k];
  const float tot32 = __shfl_sync(0xffffffffu, (float)tot, 0);
  const float den = (float)((double)tot32 + (double)eps32);
  for (int k = lane; k < cnt; k += 32) {
    const float q = (float)((double)raw_l[k] / (double)den);
    gates[row_l[k]] = (float)((double)q * (double)alpha32);
    comb_rows[t * E + k] = row_l[k];
  }
  if (lane == 0) comb_cnt[t] = cnt;
}

// ------------------------------------------------------------------ gather
// dst[i, :] = src[idx[i], :]; one warp per row, 16-B vectors, all loads first.
__global__ void gather_rows_vec_kernel(const int4* __restrict__ src, int64_t row_vecs,
                                       const int32_t* __restrict__ idx, int64_t n_idx,
                                       int4* __restrict__ dst) {
  pdl_trigger();
  pdl_wait();
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
  pdl_trigger();
  pdl_wait();
  const int64_t row = blockIdx.x;
  if (row >= n_idx) return;
  const uint8_t* s = src + (int64_t)idx[row] * row_bytes;
  for (int64_t i = threadIdx.x; i < row_bytes; i += blockDim.x) dst[row * row_bytes + i] = s[i];
}

// ------------------------------------------------------------------ combine
// moe.py:156-161 with the reference's rounding chain: gated = fp32(Y*gate),
// combined = fp32(sum over selecting experts in ascending order), out =
// round(combined + shared). ACC = double for fp32 output (the f64 chain of
// tensor.py:374-376), float for bf16 output (inside its tolerance). Warp per
// token: the token's row list and gates are staged in smem, then each lane
// issues the loads of up to CB_BATCH rows before consuming any of them.
constexpr int CB_WARPS = 8;
#ifndef NIMG_CB_BATCH
#define NIMG_CB_BATCH 8
#endif
constexpr int CB_BATCH = NIMG_CB_BATCH;

template <typename T, int VEC> struct VecIO {
  static_assert(VEC * sizeof(T) % 16 == 0 || VEC == 1, "vector width");
  static constexpr int NV = VEC * sizeof(T) / 16 > 0 ? VEC * (int)sizeof(T) / 16 : 1;
  uint4 v[NV];
  NIMG_DEV void load(const T* p) {
    if constexpr (VEC == 1) {
      *reinterpret_cast<T*>(&v[0]) = *p;
    } else {
#pragma unroll
      for (int i = 0; i < NV; ++i) v[i] = __ldg(reinterpret_cast<const uint4*>(p) + i);
    }
  }
  NIMG_DEV float at(int i) const { return to_f32(reinterpret_cast<const T*>(v)[i]); }
};

// RESID (the backbone's MoE branch, backbone.py:606): instead of the layer
// output, write h + tanh(ff_gate) * round(layer output) (f64, rounded).
// Resident blocks per SM the register allocation must allow. The bf16 combine at
// 3 (80 registers instead of 92: 24 warps per SM instead of 16) measured 90 vs
// 97-101 us in the cfg2 step; 4 spills (profiles/r02_combine_occupancy_ab.txt).
// The variants with fp32 rows or output keep 1 (they would spill).
#ifndef NIMG_CB_MINB
#define NIMG_CB_MINB 3
#endif
template <typename TY, typename TO, int VEC, typename ACC, int UNR, bool RESID>
__global__ void __launch_bounds__(CB_WARPS * 32, (sizeof(TY) == 2 && sizeof(TO) == 2) ? NIMG_CB_MINB : 1)
combine_kernel(const TY* __restrict__ yr, const TY* __restrict__ ys, const float* __restrict__ gates,
               const int32_t* __restrict__ comb_rows, const int32_t* __restrict__ comb_cnt,
               TO* __restrict__ out, int64_t T, int d, int E, const TO* __restrict__ hres,
               const ACC* __restrict__ thg, int S, const int32_t* __restrict__ tok_off, GateFuse gf) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(16) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t* rows = reinterpret_cast<int32_t*>(sm) + (size_t)warp * E;
  float* gl = reinterpret_cast<float*>(sm + (size_t)CB_WARPS * E * 4) + (size_t)warp * E;
  const int64_t t = (int64_t)blockIdx.x * CB_WARPS + warp;
  if (t >= T) return;
  const uint32_t row_bytes = (uint32_t)((int64_t)d * sizeof(TY));
  int cnt;
#ifndef NIMG_CB_NO_PREFETCH
  // whole-row L2 prefetches (one bulk instruction per row) as soon as the
  // row list is known: the column loop's loads then hit L2
  if (lane == 0 && row_bytes % 16 == 0) bulk_prefetch_l2(ys + t * d, row_bytes);
#endif
  if (gf.tokmask != nullptr) {
    // the gates of router.py:137-143 formed here (gate_tile_kernel's arithmetic):
    // the token's selecting experts in ascending order are its mask's set bits
    const unsigned long long m = gf.tokmask[t];
    cnt = __popcll(m);
    const uint32_t mlo = (uint32_t)m, mhi = (uint32_t)(m >> 32);
    const int nlo = __popc(mlo);
    for (int k = lane; k < cnt; k += 32) {
      const int e = k < nlo ? (int)__fns(mlo, 0, k + 1) : 32 + (int)__fns(mhi, 0, k - nlo + 1);
      const int2 te = gf.tokent[t * E + e];
      rows[k] = te.x;
#ifndef NIMG_CB_NO_PREFETCH
      if (row_bytes % 16 == 0) bulk_prefetch_l2(yr + (int64_t)te.x * d, row_bytes);
#endif
      gl[k] = __int_as_float(te.y);
    }
    // (the gate chain itself runs once the first row loads are in flight, below)
  } else {
    cnt = comb_cnt[t];
    // tok_off: the token's rows are consecutive in the token-ordered yr (and
    // `gates` is indexed the same way); else the expert-major row list
    const int32_t rbase = tok_off != nullptr ? tok_off[t] : 0;
    for (int k = lane; k < cnt; k += 32) {
      const int32_t r = tok_off != nullptr ? rbase + k : comb_rows[t * E + k];
      rows[k] = r;
#ifndef NIMG_CB_NO_PREFETCH
      if (row_bytes % 16 == 0) bulk_prefetch_l2(yr + (int64_t)r * d, row_bytes);
#endif
      gl[k] = gates != nullptr ? gates[r] : 1.0f;   // null: unit gates (gather pullback)
    }
  }
  __syncwarp();
  // GateFuse: gl[] holds raw scores until the first rows are in flight; then
  // gl[k] = gate (router.py:137-143, gate_tile_kernel's arithmetic)
  bool gates_ready = gf.tokmask == nullptr;
  auto form_gates = [&]() {
    float den = 0.f;
    if (lane == 0) {   // fp32(sequential f64 sum in expert order): the np.add.at order
      double tot = 0.0;
      for (int k = 0; k < cnt; ++k) tot += (double)gl[k];
      den = (float)((double)(float)tot + (double)gf.eps32);
    }
    den = __shfl_sync(0xffffffffu, den, 0);
    for (int k = lane; k < cnt; k += 32) {
      const float q = (float)((double)gl[k] / (double)den);
      const float g = (float)((double)q * (double)gf.alpha32);
      gl[k] = g;
      gf.gates_out[rows[k]] = g;
    }
    __syncwarp();
    gates_ready = true;
  };
  constexpr int STEP = 32 * VEC;
  // the in-loop call needs every lane to reach it: only when all lanes run the
  // same number of column steps
  if (!gates_ready && d % (STEP * UNR) != 0) form_gates();
  for (int c0 = lane * VEC; c0 < d; c0 += STEP * UNR) {
    VecIO<TY, VEC> sh[UNR];
    ACC acc[UNR][VEC];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      sh[u].load(ys + t * d + c0 + u * STEP);
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[u][v] = ACC(0);
    }
    constexpr int NB = CB_BATCH / UNR;   // rows in flight per batch (registers: NB*UNR vectors)
    for (int kb = 0; kb < cnt; kb += NB) {
      VecIO<TY, VEC> y[NB][UNR];
#pragma unroll
      for (int q = 0; q < NB; ++q)
        if (kb + q < cnt) {
          const TY* src = yr + (int64_t)rows[kb + q] * d + c0;
#pragma unroll
          for (int u = 0; u < UNR; ++u) y[q][u].load(src + u * STEP);
        }
      if (!gates_ready) form_gates();
#pragma unroll
      for (int q = 0; q < NB; ++q) {
        if (kb + q < cnt) {
          const float g = gl[kb + q];
#pragma unroll
          for (int u = 0; u < UNR; ++u)
#pragma unroll
            for (int v = 0; v < VEC; ++v) acc[u][v] += (ACC)(y[q][u].at(v) * g);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      TO res[VEC];
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const float comb = (float)acc[u][v];
        res[v] = from_f32<TO>((float)((ACC)comb + (ACC)sh[u].at(v)));
      }
      if constexpr (RESID) {
        const int64_t base = t * d + c0 + u * STEP;
        const ACC* tg = thg + (t / S) * d + c0 + u * STEP;
        VecIO<TO, VEC> hv;
        hv.load(hres + base);
        VecIO<ACC, VEC> gv;   // the per-sample gate, vector loads
        gv.load(tg);
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          if constexpr (sizeof(ACC) == 8)   // reference chain: product and sum rounded apart
            res[v] = from_f32<TO>((float)__dadd_rn((double)hv.at(v),
                                                   __dmul_rn(reinterpret_cast<const ACC*>(gv.v)[v],
                                                             (double)to_f32(res[v]))));
          else
            res[v] = from_f32<TO>(__fadd_rn(hv.at(v), __fmul_rn(reinterpret_cast<const ACC*>(gv.v)[v],
                                                                to_f32(res[v]))));
        }
      }
      TO* o = out + t * d + c0 + u * STEP;
      if constexpr (VEC * sizeof(TO) % 16 == 0) {
#pragma unroll
        for (int i = 0; i < VEC * (int)sizeof(TO) / 16; ++i)
          reinterpret_cast<uint4*>(o)[i] = reinterpret_cast<const uint4*>(res)[i];
      } else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) o[v] = res[v];
      }
    }
  }
}

// ------------------------------------------------------------------ launchers
cudaError_t launch_router(bool x_bf16, const void* x_norm, const float* t_emb, const float* w_r,
                          double* tb, double* part, unsigned* counter, double* wd, float* logits,
                          float* scores_bes, int B, int S, int d, int E, cudaStream_t s) {
  const bool dmma = router_uses_dmma(E);
  const int EP = dmma ? DM_EP : router_geom(E).EP;
  const int nkc = (d + RP_KCH - 1) / RP_KCH;
  // the first kernel of the chain: an ordinary launch (full stream order)
  if (dmma) router_prep_dmma_kernel<<<B * rp2_ks(d) + RP2_CONV, 256, 0, s>>>(t_emb, w_r, part, wd,
                                                                          B, d, E);
  else router_prep_kernel<<<dim3(nkc + RP_CONV_BLOCKS, B), 64, 0, s>>>(t_emb, w_r, tb, part, wd,
                                                                       counter, B, d, E, EP);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return err;
  const int64_t T = (int64_t)B * S;
  const bool vec = (d % 8 == 0) && ((uintptr_t)x_norm % 16 == 0);
  if (dmma) {
    // 8-row fragments, ~2 CTAs per SM, at most 8 fragments (64 rows) per CTA
    int sms = 148;
    {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    // k CTAs per SM (fewest rounds that keep <= 8 fragments per CTA, >= 2),
    // fragments spread evenly over them
    const int64_t nfrag = (T + 7) / 8;
    int64_t k = (nfrag + 8LL * sms - 1) / (8LL * sms);
    if (k < 2) k = 2;
    int64_t fpc = (nfrag + k * sms - 1) / (k * sms);
    if (fpc < 1) fpc = 1;
    if (fpc > 8) fpc = 8;
    const int grid = (int)((nfrag + fpc - 1) / fpc);
    const size_t smem = dmma_router_smem(E);
#define NIMG_DMMA_LAUNCH(TX, V)                                                               \
  do {                                                                                         \
    err = cudaFuncSetAttribute(router_scores_dmma_kernel<TX, V>,                               \
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);        \
    if (err != cudaSuccess) return err;                                                        \
    err = launch_pdl(router_scores_dmma_kernel<TX, V>, dim3(grid), dim3(128), smem, s,        \
                     reinterpret_cast<const TX*>(x_norm), wd, part, logits, scores_bes, B, S, d, \
                     E, (int)fpc);                                                              \
    if (err != cudaSuccess) return err;                                                        \
  } while (0)
    if (x_bf16) {
      if (vec) NIMG_DMMA_LAUNCH(bf16, true); else NIMG_DMMA_LAUNCH(bf16, false);
    } else {
      if (vec) NIMG_DMMA_LAUNCH(float, true); else NIMG_DMMA_LAUNCH(float, false);
    }
#undef NIMG_DMMA_LAUNCH
    return cudaGetLastError();
  }
  const RouterGeom g = router_geom(E);
  const int grid = (int)((T + g.TM - 1) / g.TM);
  const size_t smem = router_smem(E);
#define NIMG_ROUTER_LAUNCH(TX, V)                                                              \
  do {                                                                                         \
    err = cudaFuncSetAttribute(router_scores_kernel<TX, V>,                                    \
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);        \
    if (err != cudaSuccess) return err;                                                        \
    err = launch_pdl(router_scores_kernel<TX, V>, dim3(grid), dim3(RT_THREADS), smem, s,       \
                     reinterpret_cast<const TX*>(x_norm), wd, tb, logits, scores_bes, B, S, d, E); \
    if (err != cudaSuccess) return err;                                                        \
  } while (0)
  if (x_bf16) {
    if (vec) NIMG_ROUTER_LAUNCH(bf16, true); else NIMG_ROUTER_LAUNCH(bf16, false);
  } else {
    if (vec) NIMG_ROUTER_LAUNCH(float, true); else NIMG_ROUTER_LAUNCH(float, false);
  }
#undef NIMG_ROUTER_LAUNCH
  return cudaGetLastError();
}

bool router_uses_dmma(int E) { return E <= DM_EP; }
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("NIMG_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

size_t router_part_bytes(int B, int d, int E) {
  return (size_t)((d + RP_KCH - 1) / RP_KCH) * B * E * 8;
}
size_t router_wd_bytes(int d, int E) { return (size_t)d * (E <= DM_EP ? DM_EP : router_geom(E).EP) * 8; }

// NIMG_SELECT=cta: the block-per-column radix-select kernel for every S
static bool select_warp_enabled();
bool gate_tok_supported() { return select_warp_enabled(); }
static bool select_warp_enabled() {
  static const bool on = [] {
    const char* e = getenv("NIMG_SELECT");
    return !(e && strcmp(e, "cta") == 0);
  }();
  return on;
}

bool select_blk_path(int S) { return select_warp_enabled() && S <= 4096; }

cudaError_t launch_ec_select(const float* scores_bes, int32_t* token_flat, float* gate_raw,
                             int16_t* slot_of, int B, int S, int E, int cap, cudaStream_t s,
                             int* cursor, unsigned long long* tokmask, int2* tokent) {
  if (tokmask && (!select_blk_path(S) || E > 64)) return cudaErrorInvalidValue;
  if (select_blk_path(S)) {
    const int P = next_pow2(cap);
    const size_t wsmem = (size_t)P * 8;
    const dim3 grid((unsigned)(B * E));
#define NIMG_BSEL(K)                                                                            \
    do {                                                                                        \
      cudaError_t e2 = set_max_dyn_smem(ec_select_blk_kernel<K>, (int)wsmem);                   \
      if (e2 != cudaSuccess) return e2;                                                         \
      return launch_pdl(ec_select_blk_kernel<K>, grid, dim3(SB_WARPS * 32), wsmem, s,           \
                        scores_bes, token_flat, gate_raw, slot_of, B, S, E, cap, P, cursor,    \
                        tokmask, tokent);                                                       \
    } while (0)
    if (S <= 256) NIMG_BSEL(2);
    if (S <= 512) NIMG_BSEL(4);
    if (S <= 1024) NIMG_BSEL(8);
    if (S <= 2048) NIMG_BSEL(16);
    NIMG_BSEL(32);
#undef NIMG_BSEL
  }
  const size_t smem = select_smem(S, cap);
  cudaError_t err = cudaFuncSetAttribute(ec_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  dim3 grid(B, E);
  return launch_pdl(ec_select_kernel, grid, dim3(SEL_THREADS), smem, s, scores_bes, token_flat,
                    gate_raw, slot_of, B, S, E, cap, cursor);
}

cudaError_t launch_gate_norm(const float* scores_bes, const int16_t* slot_of, float* gates,
                             int32_t* comb_rows, int32_t* comb_cnt, int B, int S, int E, int cap,
                             float gate_eps, float gate_scale, cudaStream_t s, int* bg_flags,
                             int n_bg_flags, TokOrder tko) {
  const int64_t T = (int64_t)B * S;
  if (select_warp_enabled()) {
    const size_t smem = (((size_t)E * GT_TOK * 2 + 15) & ~size_t(15)) + (size_t)E * GT_TOK * 4 +
                        (size_t)(GT_THREADS / 32) * E * 8;
    cudaError_t err = set_max_dyn_smem(gate_tile_kernel, (int)smem);
    if (err != cudaSuccess) return err;
    const int grid = B * ((S + GT_TOK - 1) / GT_TOK);
    return launch_pdl(gate_tile_kernel, dim3(grid), dim3(GT_THREADS), smem, s, scores_bes, slot_of,
                      gates, comb_rows, comb_cnt, B, S, E, cap, gate_eps, gate_scale, bg_flags,
                      n_bg_flags, tko);
  }
  const int grid = (int)((T + GN_WARPS - 1) / GN_WARPS);
  const size_t smem = (size_t)GN_WARPS * E * 8;
  return launch_pdl(gate_norm_kernel, dim3(grid), dim3(GN_WARPS * 32), smem, s, scores_bes, slot_of,
                    gates, comb_rows, comb_cnt, B, S, E, cap, gate_eps, gate_scale, bg_flags,
                    n_bg_flags);
}

__global__ void bg_count_kernel(int rows, int chunk_rows, unsigned* __restrict__ chunk_done) {
  pdl_trigger();
  pdl_wait();
  const int nsub = (rows + 31) / 32;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nsub; j += gridDim.x * blockDim.x) {
    const int r0 = 32 * j, r1 = min(rows, r0 + 32) - 1;
    for (int c = r0 / chunk_rows; c <= r1 / chunk_rows; ++c) atomicAdd(chunk_done + c, 1u);
  }
}
cudaError_t launch_bg_count(int rows, int chunk_rows, unsigned* chunk_done, cudaStream_t s) {
  if (rows <= 0 || chunk_rows <= 0) return cudaSuccess;
  return launch_pdl(bg_count_kernel, dim3(((rows + 31) / 32 + 255) / 256), dim3(256), 0, s, rows,
                    chunk_rows, chunk_done);
}

cudaError_t launch_gather_rows(const void* src, int64_t row_bytes, const int32_t* idx,
                               int64_t n_idx, void* dst, cudaStream_t s) {
  if (n_idx <= 0) return cudaSuccess;
  const bool vec = (row_bytes % 16 == 0) && ((uintptr_t)src % 16 == 0) && ((uintptr_t)dst % 16 == 0);
  if (vec) {
    const int rows_per_cta = 8;
    const int64_t grid = (n_idx + rows_per_cta - 1) / rows_per_cta;
    return launch_pdl(gather_rows_vec_kernel, dim3((unsigned)grid), dim3(32 * rows_per_cta), 0, s,
                      reinterpret_cast<const int4*>(src), row_bytes / 16, idx, n_idx,
                      reinterpret_cast<int4*>(dst));
  }
  return launch_pdl(gather_rows_byte_kernel, dim3((unsigned)n_idx), dim3(128), 0, s,
                    reinterpret_cast<const uint8_t*>(src), row_bytes, idx, n_idx,
                    reinterpret_cast<uint8_t*>(dst));
}

template <typename TY, typename TO, bool RESID>
static cudaError_t combine_dispatch(const void* yr, const void* ys, const float* gates,
                             const int32_t* rows, const int32_t* cnt, void* out, int64_t T, int d,
                             int E, const void* hres, const void* thg, int S, cudaStream_t s,
                             const int32_t* tok_off, const GateFuse& gf) {
  const unsigned grid = (unsigned)((T + CB_WARPS - 1) / CB_WARPS);
  const size_t smem = (size_t)CB_WARPS * E * 8;
  using ACC = typename std::conditional<sizeof(TO) == 2, float, double>::type;
#define NIMG_COMBINE(V, U)                                                                      \
  launch_pdl(combine_kernel<TY, TO, V, ACC, U, RESID>, dim3(grid), dim3(CB_WARPS * 32), smem, s, \
             (const TY*)yr, (const TY*)ys, gates, rows, cnt, (TO*)out, T, d, E, (const TO*)hres, \
             (const ACC*)thg, S, tok_off, gf)
  if (d % 512 == 0) return NIMG_COMBINE(8, 2);
  if (d % 8 == 0) return NIMG_COMBINE(8, 1);
  return NIMG_COMBINE(1, 1);
#undef NIMG_COMBINE
}

cudaError_t launch_combine(bool y_bf16, bool out_bf16, const void* y_routed, const void* y_shared,
                           const float* gates, const int32_t* comb_rows, const int32_t* comb_cnt,
                           void* out, int64_t T, int d, int E, cudaStream_t s, const void* hres,
                           const void* th_gate, int S, const int32_t* tok_off, const GateFuse* gfp) {
  if (T <= 0) return cudaSuccess;
  const bool r = hres != nullptr;
  GateFuse gf{};
  if (gfp) gf = *gfp;
#define NIMG_CD(TY, TO)                                                                              \
  (r ? combine_dispatch<TY, TO, true>(y_routed, y_shared, gates, comb_rows, comb_cnt, out, T, d, E, \
                                      hres, th_gate, S, s, tok_off, gf)                             \
     : combine_dispatch<TY, TO, false>(y_routed, y_shared, gates, comb_rows, comb_cnt, out, T, d, E, \
                                       hres, th_gate, S, s, tok_off, gf))
  cudaError_t err;
  if (y_bf16 && out_bf16) err = NIMG_CD(bf16, bf16);
  else if (y_bf16) err = NIMG_CD(bf16, float);
  else if (out_bf16) err = NIMG_CD(float, bf16);
  else err = NIMG_CD(float, float);
#undef NIMG_CD
  return err;
}

}  // namespace nimg
