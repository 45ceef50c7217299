// Grouped SwiGLU expert GEMMs on 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// Replaces the per-expert loop of grouped_forward / swiglu
// (reference moe.py:115-135, moe.py:31-51): every routed expert segment (and
// the shared expert, moe.py:160, as a second weight "bank") is one row group
// of a persistent, warp-specialised kernel.
//
//   MODE 0 (GEMM1): pre[r, n] = SiLU(x W1^T) * (x W3^T)   -- dual-B tile: the
//       W1 and W3 slices of one N block sit back to back in shared memory and
//       one UMMA (M=128, N=2*112) accumulates both halves into TMEM; the
//       epilogue applies SiLU*mul and writes bf16 `pre`.
//   MODE 1 (GEMM2): y[r, n] = pre W2^T                     -- UMMA M=128, N=256.
//
// Roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM allocator + MMA
// issuer (one thread), warps 2..5 = epilogue (TMEM -> registers -> global).
// Pipelines: STAGES-deep smem ring (full/empty mbarriers) and a 2-deep TMEM
// accumulator ring (tmem_full/tmem_empty), so the epilogue of tile i overlaps
// the MMAs of tile i+1.
#include <cstdlib>

#include "common.cuh"
#include "nimg_internal.h"

namespace nimg {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;                    // 64 bf16 = one 128-B swizzle row
constexpr int kThreads = 192;
constexpr int kATileBytes = BM * BK * 2;  // 16 KB

template <int MODE> struct Cfg;
// GEMM1 output columns per tile: 128 (UMMA N = 256; at h = 1344 = 10 x 128 +
// 64 the last tile of a row block runs N = 128 in the pair kernel), or 112
// (h = 12 x 112, N = 224). 128 measured ~1% faster at cfg2 (GEMM1 652 vs 659 us,
// two runs each, profiles/r02_g1_variants.txt): 7% fewer operand bytes per MMA.
#ifndef NIMG_G1_BN
#define NIMG_G1_BN 128
#endif
template <> struct Cfg<0> {
  static constexpr int BN_OUT = NIMG_G1_BN;          // output columns per tile
  static constexpr int BN_MMA = 2 * NIMG_G1_BN;      // W1 half + W3 half
  static constexpr int B_BOX = NIMG_G1_BN;           // rows per TMA box (each of W1, W3)
  static constexpr int STAGES = 4;
  static constexpr int kBTileBytes = BN_MMA * BK * 2;  // 28 KB
};
template <> struct Cfg<1> {
  static constexpr int BN_OUT = 256;
  static constexpr int BN_MMA = 256;
  static constexpr int B_BOX = 256;
  static constexpr int STAGES = 4;
  static constexpr int kBTileBytes = BN_MMA * BK * 2;  // 32 KB
};

template <int MODE>
constexpr int stage_bytes() { return kATileBytes + Cfg<MODE>::kBTileBytes; }
template <int MODE>
constexpr int smem_bytes() { return Cfg<MODE>::STAGES * stage_bytes<MODE>() + 1024 + 256; }

struct TileInfo {
  int bank, expert, a_row, rows_valid, n0, nk;
};

template <int MODE>
NIMG_DEV void decode_tile(const GroupedParams& p, int t, TileInfo& ti) {
  int lo = 0, hi = p.nseg - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (p.seg_tile0[mid] <= t) lo = mid; else hi = mid - 1;
  }
  const int bank = lo >= p.nseg0 ? 1 : 0;
  const int ntn = p.bank[bank].ntn;
  const int local = t - p.seg_tile0[lo];
  const int m_blk = local / ntn;
  const int n_blk = local - m_blk * ntn;
  ti.bank = bank;
  ti.expert = p.seg_expert[lo];
  ti.a_row = p.seg_row0[lo] + m_blk * BM;
  ti.rows_valid = min(BM, p.seg_rows[lo] - m_blk * BM);
  ti.n0 = n_blk * Cfg<MODE>::BN_OUT;
  ti.nk = (p.bank[bank].K + BK - 1) / BK;
}

NIMG_DEV float silu_mul(float a, float g) { return a / (1.0f + __expf(-a)) * g; }

// Training forward: h1 (16 columns at n) and h3 of one row -> the row-blocked
// h1 | h3 buffer (hblk_off, common.cuh).
NIMG_DEV void store_h1h3(void* h_out, int N, int64_t row, int n, const uint32_t (&a)[16],
                         const uint32_t (&g)[16]) {
  uint32_t p1[8], p3[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    p1[j] = pack_bf16x2(__uint_as_float(a[2 * j]), __uint_as_float(a[2 * j + 1]));
    p3[j] = pack_bf16x2(__uint_as_float(g[2 * j]), __uint_as_float(g[2 * j + 1]));
  }
  const int nch = N >> 4;
  bf16* hb = reinterpret_cast<bf16*>(h_out);
  uint4* d1 = reinterpret_cast<uint4*>(hb + hblk_off(row, n >> 4, nch));
  uint4* d3 = reinterpret_cast<uint4*>(hb + hblk_off(row, nch + (n >> 4), nch));
  st_global_32(d1, make_uint4(p1[0], p1[1], p1[2], p1[3]), make_uint4(p1[4], p1[5], p1[6], p1[7]));
  st_global_32(d3, make_uint4(p3[0], p3[1], p3[2], p3[3]), make_uint4(p3[4], p3[5], p3[6], p3[7]));
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1)
grouped_gemm_sm100(const __grid_constant__ TmapSet tm, const __grid_constant__ GroupedParams p) {
  using C = Cfg<MODE>;
  constexpr int STAGES = C::STAGES;
  constexpr int SB = stage_bytes<MODE>();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * SB);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  pdl_trigger();

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 4); }
    fence_barrier_init();
    for (int b = 0; b < 2; ++b) {
      tma_prefetch_desc(&tm.a[b]);
      tma_prefetch_desc(&tm.b[b]);
      if (MODE == 0) tma_prefetch_desc(&tm.b3[b]);
    }
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();   // setup above overlapped the previous kernel; inputs are ready now

  if (warp == 0) {
    // ------------------------------------------------ TMA producer (whole warp)
    // Contiguous banks: lane 0 issues one 2-D box per k-block. Gather banks
    // (a_idx != null, the routed rows of the 1-GPU layer): the A tile is 32
    // TMA gather4 loads of 4 rows each, one per lane, straight from x_mod by
    // token_flat -- no gathered copy in HBM (moe.py:152-153 fused).
    int stage = 0; uint32_t phase = 0;
    for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
      TileInfo ti; decode_tile<MODE>(p, t, ti);
      const int32_t* idx = p.bank[ti.bank].a_idx;
      int r0 = 0, r1 = 0, r2 = 0, r3 = 0;
      if (idx != nullptr) {
        const int base = ti.a_row + 4 * lane;
        const int fallback = __ldg(idx + ti.a_row);
        r0 = 4 * lane + 0 < ti.rows_valid ? __ldg(idx + base + 0) : fallback;
        r1 = 4 * lane + 1 < ti.rows_valid ? __ldg(idx + base + 1) : fallback;
        r2 = 4 * lane + 2 < ti.rows_valid ? __ldg(idx + base + 2) : fallback;
        r3 = 4 * lane + 3 < ti.rows_valid ? __ldg(idx + base + 3) : fallback;
      }
      for (int kb = 0; kb < ti.nk; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sa = smem + stage * SB;
        uint8_t* sb = sa + kATileBytes;
        if (lane == 0) mbar_arrive_expect_tx(&full[stage], SB);
        __syncwarp();
        if (idx != nullptr) {
          tma_gather4(sa + lane * 4 * BK * 2, &tm.a[ti.bank], &full[stage], kb * BK, r0, r1, r2, r3);
        } else if (lane == 0) {
          tma_load_2d(sa, &tm.a[ti.bank], &full[stage], kb * BK, ti.a_row);
        }
        if (lane == 0) {
          tma_load_3d(sb, &tm.b[ti.bank], &full[stage], kb * BK, ti.n0, ti.expert);
          if (MODE == 0)
            tma_load_3d(sb + C::B_BOX * BK * 2, &tm.b3[ti.bank], &full[stage], kb * BK, ti.n0,
                        ti.expert);
        }
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------ MMA issuer
      constexpr uint32_t idesc = make_idesc_bf16(BM, C::BN_MMA);
      int stage = 0; uint32_t phase = 0;
      int acc = 0; uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
        TileInfo ti; decode_tile<MODE>(p, t, ti);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        for (int kb = 0; kb < ti.nk; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * SB);
          const uint32_t sb = sa + kATileBytes;
          const uint64_t adesc = make_sdesc_k128(sa);
          const uint64_t bdesc = make_sdesc_k128(sb);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // +32 B per K=16 step inside the 128-B swizzle atom (>>4 => +2)
            umma_bf16(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
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
    const int q = warp & 3;            // TMEM lane quadrant this warp may access
    const int r = q * 32 + lane;       // tile row == TMEM lane
    int acc = 0; uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
      TileInfo ti; decode_tile<MODE>(p, t, ti);
      // bank fields into registers once per tile (a runtime-indexed parameter
      // read inside the chunk loop is an LDC on the critical path)
      const GBank& bk = p.bank[ti.bank];
      const int Nb = ti.bank ? p.bank[1].N : p.bank[0].N;   // immediate-offset constant reads
      void* const h_out = ti.bank ? p.bank[1].h_out : p.bank[0].h_out;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tb = tmem_base + acc * 256 + ((uint32_t)(q * 32) << 16);
      const bool rv = r < ti.rows_valid;
      bf16* orow = reinterpret_cast<bf16*>(bk.out) + (int64_t)(ti.a_row + r) * bk.out_ld + ti.n0;
      if (MODE == 0) {
#pragma unroll 1
        for (int c = 0; c < C::BN_OUT / 16; ++c) {
          uint32_t a[16], g[16];
          tmem_ld16(tb + c * 16, a);
          tmem_ld16(tb + C::B_BOX + c * 16, g);
          tmem_ld_wait();
          if (rv && ti.n0 + c * 16 < Nb) {
            uint32_t pk[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
              pk[j] = pack_bf16x2(silu_mul(__uint_as_float(a[2 * j]), __uint_as_float(g[2 * j])),
                                  silu_mul(__uint_as_float(a[2 * j + 1]), __uint_as_float(g[2 * j + 1])));
            uint4* dst = reinterpret_cast<uint4*>(orow + c * 16);
            st_global_32(dst, make_uint4(pk[0], pk[1], pk[2], pk[3]), make_uint4(pk[4], pk[5], pk[6], pk[7]));
            if (h_out != nullptr) store_h1h3(h_out, Nb, ti.a_row + r, ti.n0 + c * 16, a, g);
          }
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < C::BN_OUT / 16; ++c) {
          uint32_t a[16];
          tmem_ld16(tb + c * 16, a);
          tmem_ld_wait();
          if (rv && ti.n0 + c * 16 < Nb) {
            uint32_t pk[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
              pk[j] = pack_bf16x2(__uint_as_float(a[2 * j]), __uint_as_float(a[2 * j + 1]));
            uint4* dst = reinterpret_cast<uint4*>(orow + c * 16);
            st_global_32(dst, make_uint4(pk[0], pk[1], pk[2], pk[3]), make_uint4(pk[4], pk[5], pk[6], pk[7]));
          }
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

// ============================================================================
// CTA-pair variant (cta_group::2). A cluster of 2 CTAs owns a 256-row tile:
// each CTA stages its own 128 A rows and HALF of B (GEMM1: the leader holds
// the W1 slice, the peer the W3 slice; GEMM2: 128 of the 256 W2 rows each),
// so per-SM shared-memory traffic per MMA drops by ~1/3 versus the 1-CTA
// kernel. The leader's single thread issues UMMA M=256; both CTAs' TMA loads
// complete on the leader's full barrier; MMA commits multicast to both CTAs'
// empty / tmem_full barriers; both CTAs' epilogues arrive on the leader's
// tmem_empty barrier. Each CTA's epilogue drains its own TMEM (its 128 rows).
template <int MODE> struct PairCfg;
template <> struct PairCfg<0> {
  static constexpr int BN_OUT = NIMG_G1_BN, BN_MMA = 2 * NIMG_G1_BN, B_ROWS = NIMG_G1_BN, STAGES = 6;
};
template <> struct PairCfg<1> {
  static constexpr int BN_OUT = 256, BN_MMA = 256, B_ROWS = 128, STAGES = 6;
};
template <int MODE> constexpr int pair_stage_bytes() { return kATileBytes + PairCfg<MODE>::B_ROWS * BK * 2; }
template <int MODE, int STAGES = PairCfg<MODE>::STAGES>
constexpr int pair_smem_bytes() { return STAGES * pair_stage_bytes<MODE>() + 1024 + 256; }

constexpr int PBM = 256;  // rows per pair tile

// GEMM1 with 128-column tiles: a row block's last tile holding <= 64 valid
// columns runs at half width
template <int MODE>
NIMG_DEV bool pair_tail_tile(const GroupedParams& p, const TileInfo& ti) {
  if (MODE != 0 || PairCfg<MODE>::BN_OUT != 128) return false;
  return (ti.bank ? p.bank[1].N : p.bank[0].N) - ti.n0 <= PairCfg<MODE>::BN_OUT / 2;
}

template <int MODE>
NIMG_DEV void decode_pair_tile(const GroupedParams& p, int t, TileInfo& ti) {
  int lo = 0, hi = p.nseg - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (p.seg_tile0[mid] <= t) lo = mid; else hi = mid - 1;
  }
  const int bank = lo >= p.nseg0 ? 1 : 0;
  const int ntn = p.bank[bank].ntn;
  const int local = t - p.seg_tile0[lo];
  const int m_blk = local / ntn;
  const int n_blk = local - m_blk * ntn;
  ti.bank = bank;
  ti.expert = p.seg_expert[lo];
  ti.a_row = p.seg_row0[lo] + m_blk * PBM;            // pair tile start
  ti.rows_valid = min(PBM, p.seg_rows[lo] - m_blk * PBM);
  ti.n0 = n_blk * PairCfg<MODE>::BN_OUT;
  ti.nk = (p.bank[bank].K + BK - 1) / BK;
}

// GATHER (GEMM1 only): banks with a_idx != null take their A rows from
// a_idx-indexed source rows. Two extra warps (6, 7) per CTA copy them with
// cp.async (16 B, 128-B swizzle applied by hand) -- the routed-row gather of
// moe.py:152-153 fused into the operand load. Each gather thread arrives
// asynchronously (cp.async.mbarrier.arrive.noinc) on a CTA-local gfull[s]; a
// relay warp (8), which has no copies in flight, waits gfull[s] and forwards
// one cluster-scope arrive to the leader's full[s]. (Waiting / releasing in
// the gather threads themselves would fence on their newer in-flight copies
// and serialise the pipeline -- measured 3.5x slower.) For contiguous (TMA)
// tiles the gather threads arrive without copying.
constexpr int kGatherWarps = 2;

// BG (GEMM1, 1-GPU layer): kBgWarps (2: measured best of 2/4/8 -- more copy
// warps slow the power-capped GEMM more than they gain) extra warps (6..) per CTA run the routed-
// row gather (moe.py:152-153) in the background: global -> global copies of
// 32-row sub-blocks, each published with a release flag. The tile order is
// rotated so the shared expert's tiles (no gathered operand) run first; the
// TMA producer of a routed tile acquires the flags of its rows and fences the
// async proxy before loading them. The gather's HBM traffic overlaps the
// shared tiles' tensor work.
// Forward progress does not assume co-residency of the grid (a concurrent
// kernel, a second layer in flight or an SM-limited context can leave CTAs
// unscheduled): sub-blocks are CLAIMED from a global counter (flags[nsub],
// zeroed with the flags) by whichever copy warps are running, never assigned
// to a CTA. A flag a producer waits on is therefore either claimed -- by a
// warp that is running and finishes the copy -- or unclaimed, and then the
// copy warps of the waiting CTA itself are still claiming and will take it.
#ifndef NIMG_BG_WARPS
#define NIMG_BG_WARPS 2
#endif
constexpr int kBgWarps = NIMG_BG_WARPS;
constexpr int kBgRows = 32;

NIMG_DEV int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
NIMG_DEV void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
NIMG_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

template <int MODE, bool GATHER, int STAGES, bool BG = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads + (GATHER ? 32 * (kGatherWarps + 1) : 0) + (BG ? 32 * kBgWarps : 0), 1)
grouped_gemm_sm100_pair(const __grid_constant__ TmapSet tm, const __grid_constant__ GroupedParams p) {
  using C = PairCfg<MODE>;
  constexpr int SB = pair_stage_bytes<MODE>();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * SB);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* gfull = tempty + 2;                      // GATHER: CTA-local gather completion
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gfull + STAGES);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const bool leader = crank == 0;
  const int cluster_id = blockIdx.x >> 1;
  const int n_clusters = gridDim.x >> 1;
  pdl_trigger();

  if (threadIdx.x == 0) {
    const uint32_t full_count = 1 + (GATHER ? 2 : 0);   // producer + one relay per CTA
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], full_count);
      mbar_init(&empty[s], 1);
      if (GATHER) mbar_init(&gfull[s], 32 * kGatherWarps);
    }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 8); }
    fence_barrier_init();
    for (int b = 0; b < 2; ++b) {
      tma_prefetch_desc(&tm.a[b]);
      tma_prefetch_desc(&tm.b[b]);
      if (MODE == 0) tma_prefetch_desc(&tm.b3[b]);
    }
  }
  if (warp == 1) tmem_alloc_cg2(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();   // setup above overlapped the previous kernel; inputs are ready now
  // BG: visit the shared bank's tiles (the tail of the tile list) first
  const int rot = BG ? p.seg_tile0[p.nseg0] : 0;
  auto tile_at = [&](int t) { return BG ? (t + rot < p.total_tiles ? t + rot : t + rot - p.total_tiles) : t; };

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer (both CTAs)
      int stage = 0; uint32_t phase = 0;
      for (int t = cluster_id; t < p.total_tiles; t += n_clusters) {
        TileInfo ti; decode_pair_tile<MODE>(p, tile_at(t), ti);
        const int a_row = ti.a_row + (int)crank * BM;
        if (BG && ti.bank == 0) {
          // acquire the background-gathered rows of this CTA's half tile
          const int r1 = min(ti.rows_valid, ((int)crank + 1) * BM) - (int)crank * BM;
          if (r1 > 0) {
            const int g0 = p.bg.row_off + a_row;
            for (int j = g0 / kBgRows; j <= (g0 + r1 - 1) / kBgRows; ++j) {
              // bounded: a protocol bug traps (a launch error) instead of hanging the GPU
              uint32_t spins = 0;
              while (ld_acquire_gpu(p.bg.flags + j) == 0)
                if (++spins == (1u << 26)) __trap();
            }
            fence_proxy_async_global();
          }
        }
        for (int kb = 0; kb < ti.nk; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * SB;
          uint8_t* sb = sa + kATileBytes;
          const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
          const bool gathered = GATHER && p.bank[ti.bank].a_idx != nullptr;
          if (leader) mbar_arrive_expect_tx(&full[stage], gathered ? 2 * (SB - kATileBytes) : 2 * SB);
          if (!gathered) tma_load_2d_cg2(sa, &tm.a[ti.bank], fb, kb * BK, a_row);
          if (MODE == 0) {  // leader: W1 slice, peer: W3 slice
            tma_load_3d_cg2(sb, crank ? (const void*)&tm.b3[ti.bank] : (const void*)&tm.b[ti.bank],
                            fb, kb * BK, ti.n0, ti.expert);
          } else {          // W2 rows n0 + 128*crank
            tma_load_3d_cg2(sb, &tm.b[ti.bank], fb, kb * BK, ti.n0 + (int)crank * C::B_ROWS, ti.expert);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      // ------------------------------------------------ MMA issuer (leader only)
      constexpr uint32_t idesc = make_idesc_bf16(PBM, C::BN_MMA);
      // GEMM1 tail tile (<= BN_OUT / 2 valid columns): N = BN_MMA / 2 reads the
      // first BN_OUT / 2 rows of each CTA's B slice (W1 | W3), so h3 lands at
      // accumulator column BN_OUT / 2 (tail_tile(), epilogue)
      constexpr uint32_t idesc_tail = make_idesc_bf16(PBM, C::BN_MMA / 2);
      int stage = 0; uint32_t phase = 0;
      int acc = 0; uint32_t acc_phase = 0;
      for (int t = cluster_id; t < p.total_tiles; t += n_clusters) {
        TileInfo ti; decode_pair_tile<MODE>(p, tile_at(t), ti);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        const uint32_t id = pair_tail_tile<MODE>(p, ti) ? idesc_tail : idesc;
        for (int kb = 0; kb < ti.nk; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * SB);
          const uint32_t sb = sa + kATileBytes;
          const uint64_t adesc = make_sdesc_k128(sa);
          const uint64_t bdesc = make_sdesc_k128(sb);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16_cg2(d_tmem, adesc + 2 * k, bdesc + 2 * k, id, (kb | k) != 0);
          umma_commit_cg2(&empty[stage], 0x3);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit_cg2(&tfull[acc], 0x3);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (GATHER && warp >= 6 && warp < 6 + kGatherWarps) {
    // ------------------------------------------------ A-row gather (warps 6, 7, both CTAs)
    const int gl = (warp - 6) * 32 + lane;                 // 0..63
    const uint32_t sbase = smem_u32(smem);
    int stage = 0; uint32_t phase = 0;
    for (int t = cluster_id; t < p.total_tiles; t += n_clusters) {
      TileInfo ti; decode_pair_tile<MODE>(p, tile_at(t), ti);
      const GBank& bk = p.bank[ti.bank];
      const int32_t* idx = bk.a_idx;
      // this lane's 16 rows of the CTA's 128 (row = gl/8 + 8j) and its 16-B column chunk
      const int row0 = (int)crank * BM;
      const int chunk = gl & 7;
      int64_t src_off[16];
      uint32_t dst_off[16];
      uint32_t valid = 0;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int r = (gl >> 3) + 8 * j;
        const bool v = idx != nullptr && row0 + r < ti.rows_valid;
        const int src_row = v ? __ldg(idx + ti.a_row + row0 + r) : 0;
        src_off[j] = (int64_t)src_row * bk.K + chunk * 8;   // elements (bf16)
        dst_off[j] = (uint32_t)(r * 128 + ((chunk ^ (r & 7)) << 4));
        valid |= (v ? 1u : 0u) << j;
      }
      const bf16* src = reinterpret_cast<const bf16*>(bk.a_src);
      for (int kb = 0; kb < ti.nk; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (idx != nullptr) {
          const uint32_t sa = sbase + stage * SB;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (valid >> j & 1u) cp_async_16(sa + dst_off[j], src + src_off[j] + kb * BK);
        }
        cp_async_mbar_arrive_noinc(&gfull[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (GATHER && warp == 6 + kGatherWarps) {
    // ------------------------------------------------ relay: gfull[s] -> leader's full[s]
    if (lane == 0) {
      int stage = 0; uint32_t phase = 0;
      for (int t = cluster_id; t < p.total_tiles; t += n_clusters) {
        TileInfo ti; decode_pair_tile<MODE>(p, tile_at(t), ti);
        for (int kb = 0; kb < ti.nk; ++kb) {
          mbar_wait(&gfull[stage], phase);
          mbar_arrive_cluster(mapa_shared(smem_u32(&full[stage]), 0));
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (BG && warp >= 6) {
    // ------------------------------------------------ background gather (warps 6.., both CTAs)
    const int nsub = (p.bg.rows + kBgRows - 1) / kBgRows;
    const int nv = p.bg.row_bytes >> 4;   // 16-B vectors per row
    const uint4* src = reinterpret_cast<const uint4*>(p.bg.src);
    uint4* dst = reinterpret_cast<uint4*>(p.bg.dst);
    int* claim = p.bg.flags + nsub;
    for (;;) {
      int j = 0;
      if (lane == 0) j = atomicAdd(claim, 1);
      j = __shfl_sync(0xffffffffu, j, 0);
      if (j >= nsub) break;
      const int r0 = j * kBgRows;
      const int nr = min(kBgRows, p.bg.rows - r0);
      const int my_src = lane < nr ? __ldg(p.bg.idx + r0 + lane) : 0;
#pragma unroll 1
      for (int r = 0; r < nr; r += 2) {   // two rows (16 x 16 B per lane) in flight
        const int s0 = __shfl_sync(0xffffffffu, my_src, r);
        const int s1 = __shfl_sync(0xffffffffu, my_src, min(r + 1, nr - 1));
        const uint4* a0 = src + (int64_t)s0 * nv;
        const uint4* a1 = src + (int64_t)s1 * nv;
        uint4* d0 = dst + (int64_t)(r0 + r) * nv;
#pragma unroll 1
        for (int cb = 0; cb < nv; cb += 256) {
          uint4 v0[8], v1[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int c = cb + lane + 32 * i;
            if (c < nv) { v0[i] = __ldg(a0 + c); v1[i] = __ldg(a1 + c); }
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int c = cb + lane + 32 * i;
            if (c < nv) {
              d0[c] = v0[i];
              if (r + 1 < nr) d0[nv + c] = v1[i];
            }
          }
        }
      }
      __threadfence();
      __syncwarp();
      if (lane == 0) {
        st_release_gpu(p.bg.flags + j, 1);
        if (p.bg.chunk_rows > 0) {   // expert parallel: the copy engines wait on these
          __threadfence_system();
          for (int c = r0 / p.bg.chunk_rows; c <= (r0 + nr - 1) / p.bg.chunk_rows; ++c)
            atomicAdd(p.bg.chunk_done + c, 1u);
        }
      }
    }
  } else if (warp >= 2 && warp < 6) {
    // ------------------------------------------------ epilogue (warps 2..5, both CTAs)
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty[0]), 0);
    const uint32_t tempty_leader1 = mapa_shared(smem_u32(&tempty[1]), 0);
    int acc = 0; uint32_t acc_phase = 0;
    for (int t = cluster_id; t < p.total_tiles; t += n_clusters) {
      TileInfo ti; decode_pair_tile<MODE>(p, tile_at(t), ti);
      const GBank& bk = p.bank[ti.bank];
      const int Nb = ti.bank ? p.bank[1].N : p.bank[0].N;   // immediate-offset constant reads
      void* const h_out = ti.bank ? p.bank[1].h_out : p.bank[0].h_out;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tb = tmem_base + acc * 256 + ((uint32_t)(q * 32) << 16);
      const int row = (int)crank * BM + r;                 // row within the pair tile
      const bool rv = row < ti.rows_valid;
      // GEMM2 with a row map (1-GPU layer): routed row r lands at row a_idx[r]
      // (token order, the combine then reads each token's rows contiguously)
      const int64_t orow_i = (MODE == 1 && bk.a_idx != nullptr && rv) ? (int64_t)__ldg(bk.a_idx + ti.a_row + row)
                                                                      : (int64_t)(ti.a_row + row);
      bf16* orow = reinterpret_cast<bf16*>(bk.out) + orow_i * bk.out_ld + ti.n0;
      const int oflags = ti.bank ? p.bank[1].flags : p.bank[0].flags;
      const bool tail = pair_tail_tile<MODE>(p, ti);
      const uint32_t hoff = tail ? C::B_ROWS / 2 : C::B_ROWS;   // h3's first accumulator column
#pragma unroll 1
      for (int c = 0; c < (tail ? C::BN_OUT / 32 : C::BN_OUT / 16); ++c) {
        uint32_t a[16], g[16];
        tmem_ld16(tb + c * 16, a);
        float v[16];
        if (MODE == 0) {
          tmem_ld16(tb + hoff + c * 16, g);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = silu_mul(__uint_as_float(a[j]), __uint_as_float(g[j]));
        } else {
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(a[j]);
        }
        uint32_t pk[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) pk[j] = pack_bf16x2(v[2 * j], v[2 * j + 1]);
        if (rv && ti.n0 + c * 16 < Nb) {
          if (MODE == 1 && (oflags & kF32Out)) {   // fp32 mode: fp32 rows
            float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(bk.out) +
                                                    orow_i * bk.out_ld + ti.n0 + c * 16);
#pragma unroll
            for (int j = 0; j < 2; ++j)
              st_global_32(dst + 2 * j,
                           make_uint4(__float_as_uint(v[8 * j]), __float_as_uint(v[8 * j + 1]),
                                      __float_as_uint(v[8 * j + 2]), __float_as_uint(v[8 * j + 3])),
                           make_uint4(__float_as_uint(v[8 * j + 4]), __float_as_uint(v[8 * j + 5]),
                                      __float_as_uint(v[8 * j + 6]), __float_as_uint(v[8 * j + 7])));
          } else {
            uint4* dst = reinterpret_cast<uint4*>(orow + c * 16);
            st_global_32(dst, make_uint4(pk[0], pk[1], pk[2], pk[3]), make_uint4(pk[4], pk[5], pk[6], pk[7]));
            if (MODE == 0 && (oflags & kSplit3Out)) {   // fp32 mode: pre as [hi | hi | lo]
              uint32_t lo[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const __nv_bfloat162 hv = *reinterpret_cast<const __nv_bfloat162*>(&pk[j]);
                lo[j] = pack_bf16x2(v[2 * j] - __low2float(hv), v[2 * j + 1] - __high2float(hv));
              }
              uint4* d2 = reinterpret_cast<uint4*>(orow + Nb + c * 16);
              uint4* d3 = reinterpret_cast<uint4*>(orow + 2 * Nb + c * 16);
              st_global_32(d2, make_uint4(pk[0], pk[1], pk[2], pk[3]), make_uint4(pk[4], pk[5], pk[6], pk[7]));
              st_global_32(d3, make_uint4(lo[0], lo[1], lo[2], lo[3]), make_uint4(lo[4], lo[5], lo[6], lo[7]));
            }
            if (MODE == 0 && h_out != nullptr)   // training forward: keep h1 | h3
              store_h1h3(h_out, Nb, ti.a_row + row, ti.n0 + c * 16, a, g);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(acc ? tempty_leader1 : tempty_leader0);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_cg2(tmem_base, 512);
  }
}

}  // namespace tc

// ------------------------------------------------------------------ host side
int tc_bn_out(int mode) { return mode == 0 ? tc::Cfg<0>::BN_OUT : tc::Cfg<1>::BN_OUT; }
int tc_pair_rows() { return tc::PBM; }

template <int MODE, bool GATHER, int STAGES, bool BG = false>
static cudaError_t launch_pair(const TmapSet& tm, const GroupedParams& p, int grid, cudaStream_t stream) {
  constexpr int smem = tc::pair_smem_bytes<MODE, STAGES>();
  constexpr int threads = tc::kThreads + (GATHER ? 32 * (tc::kGatherWarps + 1) : 0) + (BG ? 32 * tc::kBgWarps : 0);
  cudaError_t e = set_max_dyn_smem(tc::grouped_gemm_sm100_pair<MODE, GATHER, STAGES, BG>, smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(tc::grouped_gemm_sm100_pair<MODE, GATHER, STAGES, BG>, dim3(grid), dim3(threads),
                    (size_t)smem, stream, tm, p);
}

// Shallow-pipeline variant (4 stages, ~122-130 KB smem) leaves room on each
// SM for a co-resident router CTA; NIMG_GEMM_STAGES=4 selects it globally.
static int pair_stages() {
  static const int st = [] {
    const char* e = getenv("NIMG_GEMM_STAGES");
    return (e && atoi(e) == 4) ? 4 : 6;
  }();
  return st;
}

cudaError_t launch_grouped_tc_pair(int mode, const TmapSet& tm, const GroupedParams& p, int num_sms,
                                   cudaStream_t stream) {
  if (p.total_tiles <= 0) return cudaSuccess;
  const int clusters = p.total_tiles < num_sms / 2 ? p.total_tiles : num_sms / 2;
  const int grid = 2 * clusters;
  const bool gather = p.bank[0].a_idx != nullptr || p.bank[1].a_idx != nullptr;
  const bool shallow = pair_stages() == 4;
  if (mode == 0) {
    if (gather) return launch_pair<0, true, 6>(tm, p, grid, stream);
    if (p.bg.src != nullptr) return launch_pair<0, false, 6, true>(tm, p, grid, stream);
    return shallow ? launch_pair<0, false, 4>(tm, p, grid, stream) : launch_pair<0, false, 6>(tm, p, grid, stream);
  }
  return shallow ? launch_pair<1, false, 4>(tm, p, grid, stream) : launch_pair<1, false, 6>(tm, p, grid, stream);
}
int tc_b_box(int mode) { return mode == 0 ? tc::Cfg<0>::B_BOX : tc::Cfg<1>::B_BOX; }

cudaError_t launch_grouped_tc(int mode, const TmapSet& tm, const GroupedParams& p, int num_sms,
                              cudaStream_t stream) {
  if (p.total_tiles <= 0) return cudaSuccess;
  const int grid = p.total_tiles < num_sms ? p.total_tiles : num_sms;
  if (mode == 0) {
    constexpr int smem = tc::smem_bytes<0>();
    cudaError_t e = set_max_dyn_smem(tc::grouped_gemm_sm100<0>, smem);
    if (e != cudaSuccess) return e;
    return launch_pdl(tc::grouped_gemm_sm100<0>, dim3(grid), dim3(tc::kThreads), (size_t)smem,
                      stream, tm, p);
  } else {
    constexpr int smem = tc::smem_bytes<1>();
    cudaError_t e = set_max_dyn_smem(tc::grouped_gemm_sm100<1>, smem);
    if (e != cudaSuccess) return e;
    return launch_pdl(tc::grouped_gemm_sm100<1>, dim3(grid), dim3(tc::kThreads), (size_t)smem,
                      stream, tm, p);
  }
}

}  // namespace nimg
