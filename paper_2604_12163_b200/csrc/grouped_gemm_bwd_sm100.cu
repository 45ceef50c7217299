// Backward grouped GEMMs of the SwiGLU experts on tcgen05 (TMEM accumulators,
// TMA operands): the swiglu pullback of moe.py:53-62 per expert segment.
//
//   BWD_D2  dH = SwiGLU'(dY W2_e)    A = dY rows (K-major), B = W2_e read
//           MN-major ([d][h] storage is N-contiguous); the epilogue applies the
//           SwiGLU derivative with h1 | h3 saved by the forward and writes
//           dH1 | dH3 (bf16).
//   BWD_D1  dX = dH [W1_e; W3_e]      A = dH rows (K-major, K = 2h), B = W1_e /
//           W3_e MN-major (the K loop switches tensor map at k = h).
//   BWD_W2  dW2_e = dY^T pre          A = dY, B = pre, both MN-major: the
//           reduction runs over the segment's rows, which are the *outer*
//           (strided) dimension of both stored operands.
//   BWD_W1  [dW1_e; dW3_e] = dH^T X   A = dH (M = 2h), B = X, both MN-major.
//
// No transposed copy of any operand is made: TMA lands MN-major boxes {64, 64}
// with 128-B swizzle and the UMMA descriptors say MN-major (idesc bits 15/16,
// LBO = MN-chunk stride). Weight-gradient tiles accumulate a whole segment in
// TMEM and store fp32 once (deterministic: no split-K, no atomics).
//
// Same warp roles as the forward kernel: warp 0 TMA producer, warp 1 TMEM
// allocator + single-thread MMA issuer, warps 2..5 epilogue; 4-stage smem ring,
// 2-deep TMEM accumulator ring; persistent grid of #SMs CTAs.
#include "common.cuh"
#include "nimg_internal.h"

namespace nimg {
namespace tcb {

constexpr int BM = 128, BK = 64, kThreads = 192;
constexpr int kChunk = 64 * BK * 2;            // one {64 MN, 64 K} box = 8 KB

template <int MODE> struct Cfg;
template <> struct Cfg<BWD_D2> { static constexpr int BN = 192, STAGES = 5; };
template <> struct Cfg<BWD_D1> { static constexpr int BN = 256, STAGES = 4; };
template <> struct Cfg<BWD_W2> { static constexpr int BN = 192, STAGES = 5; };
template <> struct Cfg<BWD_W1> { static constexpr int BN = 256, STAGES = 4; };

template <int MODE> constexpr bool a_mn() { return MODE == BWD_W2 || MODE == BWD_W1; }
template <int MODE> constexpr int stage_bytes() { return BM * BK * 2 + Cfg<MODE>::BN * BK * 2; }
template <int MODE> constexpr int smem_bytes() { return Cfg<MODE>::STAGES * stage_bytes<MODE>() + 1024 + 256; }

struct Tile {
  int bank, expert, row0, rows_valid, m0, n0, nk, nk1;
};

template <int MODE>
NIMG_DEV void decode(const BwdParams& p, int t, Tile& ti) {
  int lo = 0, hi = p.nseg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (p.seg_tile0[mid] <= t) lo = mid; else hi = mid - 1;
  }
  const int bank = p.seg_bank[lo];
  const BwdBank& bk = p.bank[bank];
  const int local = t - p.seg_tile0[lo];
  const int m_blk = local / bk.ntn, n_blk = local - (local / bk.ntn) * bk.ntn;
  ti.bank = bank;
  ti.expert = p.seg_expert[lo];
  ti.n0 = n_blk * Cfg<MODE>::BN;
  if (a_mn<MODE>()) {           // weight gradient: M = bk.M, K = segment rows
    ti.row0 = p.seg_row0[lo];
    ti.m0 = m_blk * BM;
    ti.rows_valid = min(BM, bk.M - ti.m0);
    ti.nk = (p.seg_rows[lo] + BK - 1) / BK;
    ti.nk1 = ti.nk;
  } else {                      // data gradient: M = segment rows, K = bk.K
    ti.row0 = p.seg_row0[lo] + m_blk * BM;
    ti.m0 = 0;
    ti.rows_valid = min(BM, p.seg_rows[lo] - m_blk * BM);
    if (MODE == BWD_D1) { ti.nk1 = (bk.h + BK - 1) / BK; ti.nk = 2 * ti.nk1; }
    else { ti.nk = (bk.K + BK - 1) / BK; ti.nk1 = ti.nk; }
  }
}

NIMG_DEV void unpack16(const uint4 (&v)[2], float (&f)[16]) {
  const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(v);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float2 q = __bfloat1622float2(p[i]);
    f[2 * i] = q.x;
    f[2 * i + 1] = q.y;
  }
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1)
grouped_gemm_bwd_sm100(const __grid_constant__ TmapSet tm, const __grid_constant__ BwdParams p) {
  constexpr int BN = Cfg<MODE>::BN, STAGES = Cfg<MODE>::STAGES, SB = stage_bytes<MODE>();
  constexpr bool AMN = a_mn<MODE>();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * SB);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_trigger();

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 4); }
    fence_barrier_init();
    for (int b = 0; b < 2; ++b) {
      tma_prefetch_desc(&tm.a[b]);
      tma_prefetch_desc(&tm.b[b]);
      if (MODE == BWD_D1) tma_prefetch_desc(&tm.b3[b]);
    }
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------- TMA producer
      int stage = 0; uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
        Tile ti; decode<MODE>(p, t, ti);
        for (int kb = 0; kb < ti.nk; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * SB;
          uint8_t* sb = sa + BM * BK * 2;
          mbar_arrive_expect_tx(&full[stage], SB);
          if (AMN) {   // A^T tile: 2 boxes of 64 M-columns x 64 K-rows (3-D map [E][rows][M])
            const int z = ti.bank ? 0 : ti.expert;
            tma_load_3d(sa, &tm.a[ti.bank], &full[stage], ti.m0, kb * BK, z);
            tma_load_3d(sa + kChunk, &tm.a[ti.bank], &full[stage], ti.m0 + 64, kb * BK, z);
          } else {     // A rows: one box {64 K, 128 rows}
            tma_load_2d(sa, &tm.a[ti.bank], &full[stage], kb * BK, ti.row0);
          }
          // B: BN/64 MN-major boxes {64 N, 64 K}
          const void* bm = &tm.b[ti.bank];
          int kc = kb * BK, z = ti.expert;
          if (MODE == BWD_D1 && kb >= ti.nk1) { bm = &tm.b3[ti.bank]; kc = (kb - ti.nk1) * BK; }
          if (AMN) z = ti.bank ? 0 : ti.expert;
#pragma unroll
          for (int j = 0; j < BN / 64; ++j)
            tma_load_3d(sb + j * kChunk, bm, &full[stage], ti.n0 + 64 * j, kc, z);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------------------------------------- MMA issuer
      constexpr uint32_t idesc = make_idesc_bf16_major(BM, BN, AMN, true);
      int stage = 0; uint32_t phase = 0;
      int acc = 0; uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
        Tile ti; decode<MODE>(p, t, ti);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        for (int kb = 0; kb < ti.nk; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * SB);
          const uint32_t sb = sa + BM * BK * 2;
          const uint64_t adesc = AMN ? make_sdesc_mn128(sa, kChunk) : make_sdesc_k128(sa);
          const uint64_t bdesc = make_sdesc_mn128(sb, kChunk);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // K step of 16: K-major +32 B inside the swizzle row; MN-major +16 rows = 2048 B
            const uint64_t ao = AMN ? (uint64_t)(k * 2048 >> 4) : (uint64_t)(2 * k);
            umma_bf16(d_tmem, adesc + ao, bdesc + (uint64_t)(k * 2048 >> 4), idesc, (kb | k) != 0);
          }
          umma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ------------------------------------------------ epilogue (warps 2..5)
    const int q = warp & 3;
    const int r = q * 32 + lane;
    int acc = 0; uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
      Tile ti; decode<MODE>(p, t, ti);
      const BwdBank& bk = p.bank[ti.bank];
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tb = tmem_base + acc * 256 + ((uint32_t)(q * 32) << 16);
      const bool rv = r < ti.rows_valid;
      const int N = bk.N, h = bk.h;
#pragma unroll 1
      for (int c = 0; c < BN / 16; ++c) {
        uint32_t a[16];
        tmem_ld16(tb + c * 16, a);
        tmem_ld_wait();
        const int n = ti.n0 + c * 16;
        if (!rv || n >= N) continue;
        if (MODE == BWD_D2) {
          const int64_t row = ti.row0 + r;
          const bf16* hr = reinterpret_cast<const bf16*>(bk.aux) + row * (int64_t)(2 * h);
          uint4 h1v[2], h3v[2];
          h1v[0] = __ldg(reinterpret_cast<const uint4*>(hr + n));
          h1v[1] = __ldg(reinterpret_cast<const uint4*>(hr + n) + 1);
          h3v[0] = __ldg(reinterpret_cast<const uint4*>(hr + h + n));
          h3v[1] = __ldg(reinterpret_cast<const uint4*>(hr + h + n) + 1);
          float h1[16], h3[16];
          unpack16(h1v, h1);
          unpack16(h3v, h3);
          uint32_t p1[8], p3[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float g1[2], g3[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int i = 2 * j + u;
              const float v = __uint_as_float(a[i]);
              const float sig = 1.0f / (1.0f + __expf(-h1[i]));
              g1[u] = v * h3[i] * sig * (1.0f + h1[i] * (1.0f - sig));
              g3[u] = v * h1[i] * sig;
            }
            p1[j] = pack_bf16x2(g1[0], g1[1]);
            p3[j] = pack_bf16x2(g3[0], g3[1]);
          }
          bf16* o = reinterpret_cast<bf16*>(bk.out) + row * (int64_t)(2 * h);
          uint4* d1 = reinterpret_cast<uint4*>(o + n);
          uint4* d3 = reinterpret_cast<uint4*>(o + h + n);
          d1[0] = make_uint4(p1[0], p1[1], p1[2], p1[3]);
          d1[1] = make_uint4(p1[4], p1[5], p1[6], p1[7]);
          d3[0] = make_uint4(p3[0], p3[1], p3[2], p3[3]);
          d3[1] = make_uint4(p3[4], p3[5], p3[6], p3[7]);
        } else if (MODE == BWD_D1) {
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) pk[j] = pack_bf16x2(__uint_as_float(a[2 * j]), __uint_as_float(a[2 * j + 1]));
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<bf16*>(bk.out) + (ti.row0 + r) * bk.out_ld + n);
          dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        } else {
          const int m = ti.m0 + r;
          const int64_t e = ti.expert;
          float* o;
          if (MODE == BWD_W2) o = reinterpret_cast<float*>(bk.out) + e * (int64_t)bk.M * N + (int64_t)m * N + n;
          else o = m < h ? reinterpret_cast<float*>(bk.out) + e * (int64_t)h * N + (int64_t)m * N + n
                         : reinterpret_cast<float*>(bk.out3) + e * (int64_t)h * N + (int64_t)(m - h) * N + n;
          float4* dst = reinterpret_cast<float4*>(o);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            dst[j] = make_float4(__uint_as_float(a[4 * j]), __uint_as_float(a[4 * j + 1]),
                                 __uint_as_float(a[4 * j + 2]), __uint_as_float(a[4 * j + 3]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

}  // namespace tcb

int tc_bwd_bn(int mode) {
  switch (mode) {
    case BWD_D2: return tcb::Cfg<BWD_D2>::BN;
    case BWD_D1: return tcb::Cfg<BWD_D1>::BN;
    case BWD_W2: return tcb::Cfg<BWD_W2>::BN;
    default: return tcb::Cfg<BWD_W1>::BN;
  }
}

template <int MODE>
static cudaError_t launch_bwd(const TmapSet& tm, const BwdParams& p, int grid, cudaStream_t s) {
  constexpr int smem = tcb::smem_bytes<MODE>();
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tcb::grouped_gemm_bwd_sm100<MODE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return launch_pdl(tcb::grouped_gemm_bwd_sm100<MODE>, dim3(grid), dim3(tcb::kThreads), (size_t)smem, s,
                    tm, p);
}

cudaError_t launch_grouped_tc_bwd(int mode, const TmapSet& tm, const BwdParams& p, int num_sms,
                                  cudaStream_t s) {
  if (p.total_tiles <= 0) return cudaSuccess;
  const int grid = p.total_tiles < num_sms ? p.total_tiles : num_sms;
  switch (mode) {
    case BWD_D2: return launch_bwd<BWD_D2>(tm, p, grid, s);
    case BWD_D1: return launch_bwd<BWD_D1>(tm, p, grid, s);
    case BWD_W2: return launch_bwd<BWD_W2>(tm, p, grid, s);
    default: return launch_bwd<BWD_W1>(tm, p, grid, s);
  }
}

}  // namespace nimg
