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
#include <cstdlib>

#include "common.cuh"
#include "nimg_internal.h"

namespace nimg {
namespace tcb {

constexpr int BM = 128, BK = 64;
constexpr int kChunk = 64 * BK * 2;            // one {64 MN, 64 K} box = 8 KB

// PAIR = cta_group::2: a cluster of 2 CTAs owns a 256-row (D modes) or
// 256-M (W modes) tile; each CTA stages its own 128 A rows / M-columns and
// half of the N columns of B, the leader issues UMMA M=256 (as the forward
// pair kernel). Per-SM operand traffic per MMA drops by ~1/3.
// D2: one more warp streams the tile's saved h1 | h3 into shared memory with
// bulk copies (NIMG_D2_HSTAGE=0: the epilogue loads them from global itself)
#ifndef NIMG_D2_HSTAGE
#define NIMG_D2_HSTAGE 1
#endif
template <int MODE, bool PAIR> struct Cfg;
template <> struct Cfg<BWD_D2, false> { static constexpr int BN = 192, STAGES = NIMG_D2_HSTAGE ? 4 : 5; };
template <> struct Cfg<BWD_D1, false> { static constexpr int BN = 256, STAGES = 4; };
template <> struct Cfg<BWD_W2, false> { static constexpr int BN = 192, STAGES = 4; };
template <> struct Cfg<BWD_W1, false> { static constexpr int BN = 256, STAGES = 4; };
// router weight gradient dW_r[:d] = x_norm^T dlogits per sample (N = E = 64)
template <> struct Cfg<BWD_WR, false> { static constexpr int BN = 64, STAGES = 8; };
// h = 6 x 224. 256-wide tiles (h = 5 x 256 + 64, the last tile of a row block
// at N = 128, see the MMA issuer) measured 1-3% slower for both dgrad2 and dW2.
#ifndef NIMG_D2_BN
#define NIMG_D2_BN 224
#endif
#ifndef NIMG_W2_BN
#define NIMG_W2_BN 224
#endif
template <> struct Cfg<BWD_D2, true> { static constexpr int BN = NIMG_D2_BN, STAGES = 6; };
template <> struct Cfg<BWD_D1, true> { static constexpr int BN = 256, STAGES = 6; };
template <> struct Cfg<BWD_W2, true> { static constexpr int BN = NIMG_W2_BN, STAGES = 6; };
template <> struct Cfg<BWD_W1, true> { static constexpr int BN = 256, STAGES = 6; };

// epilogue warps: 8 for the SwiGLU-derivative epilogue (two warps per TMEM
// lane quadrant split the column groups), 4 elsewhere
template <int MODE> constexpr int epi_warps() { return MODE == BWD_D2 ? 8 : 4; }
template <int MODE> constexpr bool h_staged() { return MODE == BWD_D2 && NIMG_D2_HSTAGE; }
template <int MODE> constexpr int threads() { return 64 + 32 * epi_warps<MODE>() + (h_staged<MODE>() ? 32 : 0); }
// D2 h1 | h3 staging: a slot holds 2 column chunks of 16 (h1 and h3) for the
// CTA's 128 rows, [chunk][h1|h3][128 rows][16 bf16] = 16 KB; 2 slots
constexpr int kHChunkBytes = 128 * 16 * 2;
constexpr int kHSlotBytes = 4 * kHChunkBytes;
constexpr int kHSlots = 2;
template <int MODE> constexpr int h_bytes() { return h_staged<MODE>() ? kHSlots * kHSlotBytes : 0; }
template <int MODE> constexpr bool a_mn() { return MODE == BWD_W2 || MODE == BWD_W1 || MODE == BWD_WR; }
// per-CTA B columns and their 64-wide TMA boxes (pair: the last box may be
// partly outside this CTA's half; UMMA reads only BN/2 columns of it)
template <int MODE, bool PAIR> constexpr int bn_cta() { return PAIR ? Cfg<MODE, PAIR>::BN / 2 : Cfg<MODE, PAIR>::BN; }
template <int MODE, bool PAIR> constexpr int b_boxes() { return (bn_cta<MODE, PAIR>() + 63) / 64; }
template <int MODE, bool PAIR> constexpr int stage_bytes() { return BM * BK * 2 + b_boxes<MODE, PAIR>() * kChunk; }
// W modes: per epilogue warp two 4-KB staging tiles (32 rows x 32 fp32, 128-B swizzle) for TMA stores
constexpr int kStageOut = 4096;
// (Stored from registers one row per thread, 8 x 16 B per 32 columns -- 32
// partial sectors per warp store: dW2 395 -> 486 us, dW1 728 -> 858 us.)
// timing probes for A/B builds only (wrong results): 1 = W epilogues skip the
// staging and stores, 2 = the dgrad2 epilogue skips h1 | h3 and its stores
#ifndef NIMG_BWD_PROBE
#define NIMG_BWD_PROBE 0
#endif
// W epilogues: whole 32-B sectors stored from registers (16x256b TMEM loads,
// the default: dW1 766 vs 804 us, dW2 equal), or (0) fp32 tiles staged in smem
// for TMA stores (profiles/r02_bwd_epilogue_probe.txt)
#ifndef NIMG_W_SECTOR
#define NIMG_W_SECTOR 1
#endif
template <int MODE> constexpr int out_bytes() { return (a_mn<MODE>() && !NIMG_W_SECTOR) ? 4 * 2 * kStageOut : 0; }
template <int MODE, bool PAIR> constexpr int smem_bytes() {
  return Cfg<MODE, PAIR>::STAGES * stage_bytes<MODE, PAIR>() + out_bytes<MODE>() + h_bytes<MODE>() +
         1024 + 256;
}

struct Tile {
  int bank, expert, row0, rows_valid, m0, n0, nk, nk1;
};

// row0 / m0 / rows_valid are for the whole (pair) tile of TM rows
template <int MODE, bool PAIR>
NIMG_DEV void decode(const BwdParams& p, int t, Tile& ti) {
  constexpr int TM = PAIR ? 2 * BM : BM;
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
  ti.n0 = n_blk * Cfg<MODE, PAIR>::BN;
  if (a_mn<MODE>()) {           // weight gradient: M = bk.M, K = segment rows
    ti.row0 = p.seg_row0[lo];
    ti.m0 = m_blk * TM;
    ti.rows_valid = min(TM, bk.M - ti.m0);
    ti.nk = (p.seg_rows[lo] + BK - 1) / BK;
    ti.nk1 = ti.nk;
  } else {                      // data gradient: M = segment rows, K = bk.K
    ti.row0 = p.seg_row0[lo] + m_blk * TM;
    ti.m0 = 0;
    ti.rows_valid = min(TM, p.seg_rows[lo] - m_blk * TM);
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

template <bool PAIR> NIMG_DEV void load_2d(void* dst, const void* map, uint64_t* bar, int c0, int c1) {
  if (PAIR) tma_load_2d_cg2(dst, map, mapa_shared(smem_u32(bar), 0), c0, c1);
  else tma_load_2d(dst, map, bar, c0, c1);
}
template <bool PAIR> NIMG_DEV void load_3d(void* dst, const void* map, uint64_t* bar, int c0, int c1, int c2) {
  if (PAIR) tma_load_3d_cg2(dst, map, mapa_shared(smem_u32(bar), 0), c0, c1, c2);
  else tma_load_3d(dst, map, bar, c0, c1, c2);
}

template <int MODE, bool PAIR>
__global__ void __launch_bounds__(threads<MODE>(), 1)
grouped_gemm_bwd_sm100(const __grid_constant__ TmapSetBwd tm, const __grid_constant__ BwdParams p) {
  using C = Cfg<MODE, PAIR>;
  constexpr int BN = C::BN, STAGES = C::STAGES, SB = stage_bytes<MODE, PAIR>();
  constexpr int BNC = bn_cta<MODE, PAIR>(), NBOX = b_boxes<MODE, PAIR>();
  constexpr int EPI = epi_warps<MODE>();
  constexpr bool AMN = a_mn<MODE>();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage_out = smem + STAGES * SB;                  // W modes: TMA-store staging
  uint8_t* hbuf = stage_out + out_bytes<MODE>();             // D2: staged h1 | h3 slots
  uint64_t* full = reinterpret_cast<uint64_t*>(hbuf + h_bytes<MODE>());
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* hfull = tempty + 2;                             // D2 staging slots
  uint64_t* hempty = hfull + kHSlots;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hempty + kHSlots);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = PAIR ? cluster_ctarank() : 0;
  const bool leader = crank == 0;
  const int unit = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;      // tile-scheduling unit
  const int n_units = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  pdl_trigger();

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], (PAIR ? 2 : 1) * EPI); }
    if (h_staged<MODE>())
      for (int sl = 0; sl < kHSlots; ++sl) { mbar_init(&hfull[sl], 1); mbar_init(&hempty[sl], EPI); }
    fence_barrier_init();
    for (int b = 0; b < 2; ++b) {
      tma_prefetch_desc(&tm.a[b]);
      tma_prefetch_desc(&tm.b[b]);
      if (MODE == BWD_D1) tma_prefetch_desc(&tm.b3[b]);
      if (AMN) { tma_prefetch_desc(&tm.o[b]); tma_prefetch_desc(&tm.o3[b]); }
    }
  }
  if (warp == 1) { if (PAIR) tmem_alloc_cg2(tmem_slot, 512); else tmem_alloc(tmem_slot, 512); }
  tc_fence_before();
  if (PAIR) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------- TMA producer (both CTAs of a pair)
      int stage = 0; uint32_t phase = 0;
      for (int t = unit; t < p.total_tiles; t += n_units) {
        Tile ti; decode<MODE, PAIR>(p, t, ti);
        for (int kb = 0; kb < ti.nk; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * SB;
          uint8_t* sb = sa + BM * BK * 2;
          if (leader) mbar_arrive_expect_tx(&full[stage], (PAIR ? 2 : 1) * SB);
          // W modes: routed segment e reads rows of z = e of the 3-D [E][rows_e][.]
          // views; the shared bank (z = 0, all T rows) may be split into row
          // chunks (segments with their own partial output z = chunk)
          const int krow = kb * BK + (AMN && ti.bank ? ti.row0 : 0);
          if (AMN) {   // A^T: 2 boxes of 64 M-columns x 64 K-rows (3-D map [E][rows][M])
            const int z = ti.bank ? 0 : ti.expert;
            const int m = ti.m0 + (int)crank * BM;
            load_3d<PAIR>(sa, &tm.a[ti.bank], &full[stage], m, krow, z);
            load_3d<PAIR>(sa + kChunk, &tm.a[ti.bank], &full[stage], m + 64, krow, z);
          } else {     // A rows: one box {64 K, 128 rows}
            load_2d<PAIR>(sa, &tm.a[ti.bank], &full[stage], kb * BK, ti.row0 + (int)crank * BM);
          }
          // B: this CTA's columns, MN-major boxes {64 N, 64 K}
          const void* bm = &tm.b[ti.bank];
          int kc = AMN ? krow : kb * BK, z = ti.expert;
          if (MODE == BWD_D1 && kb >= ti.nk1) { bm = &tm.b3[ti.bank]; kc = (kb - ti.nk1) * BK; }
          if (AMN) z = ti.bank ? 0 : ti.expert;
          const int nb = ti.n0 + (int)crank * BNC;
#pragma unroll
          for (int j = 0; j < NBOX; ++j) load_3d<PAIR>(sb + j * kChunk, bm, &full[stage], nb + 64 * j, kc, z);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      // ---------------------------------------------- MMA issuer (leader)
      constexpr uint32_t idesc = make_idesc_bf16_major(PAIR ? 2 * BM : BM, BN, AMN, true);
      // narrow last tile of a 256-wide pair row: N = 128 reads each CTA's first
      // 64 B columns, which hold all nval <= 64 valid ones (the epilogue reads
      // accumulator columns < nval only)
      constexpr uint32_t idesc_tail = make_idesc_bf16_major(PAIR ? 2 * BM : BM, BN / 2, AMN, true);
      int stage = 0; uint32_t phase = 0;
      int acc = 0; uint32_t acc_phase = 0;
      for (int t = unit; t < p.total_tiles; t += n_units) {
        Tile ti; decode<MODE, PAIR>(p, t, ti);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        const int nval = (ti.bank ? p.bank[1].N : p.bank[0].N) - ti.n0;
        const uint32_t id = (PAIR && BN == 256 && nval <= BN / 4) ? idesc_tail : idesc;
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
            const uint64_t bo = (uint64_t)(k * 2048 >> 4);
            if (PAIR) umma_bf16_cg2(d_tmem, adesc + ao, bdesc + bo, id, (kb | k) != 0);
            else umma_bf16(d_tmem, adesc + ao, bdesc + bo, id, (kb | k) != 0);
          }
          if (PAIR) umma_commit_cg2(&empty[stage], 0x3); else umma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (PAIR) umma_commit_cg2(&tfull[acc], 0x3); else umma_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (h_staged<MODE>() && warp == 2 + EPI) {
    // ------------------------------------------------ D2: h1 | h3 stager (both CTAs, own 128 rows)
    // The row-blocked h1 | h3 layout (hblk_off) keeps 128 rows x 16 columns of a
    // chunk contiguous (4 KB), so a CTA's rows of one chunk are 1 bulk copy (2
    // when they straddle a 128-row block).
    if (lane == 0) {
      constexpr int NCH = BN / 16, NG2 = (NCH + 1) / 2;
      const int rc = (int)crank * BM;
      int hs = 0; uint32_t hph = 0;
      for (int t = unit; t < p.total_tiles; t += n_units) {
        Tile ti; decode<MODE, PAIR>(p, t, ti);
        const BwdBank& bk = p.bank[ti.bank];
        const int N = ti.bank ? p.bank[1].N : p.bank[0].N;
        const int h = ti.bank ? p.bank[1].h : p.bank[0].h;
        const int nch = h >> 4;
        const bf16* hb = reinterpret_cast<const bf16*>(bk.aux);
        const int rv = min(BM, ti.rows_valid - rc);
        const int64_t R0 = ti.row0 + rc;
        const int n1 = rv > 0 ? min(rv, 128 - (int)(R0 & 127)) : 0;   // rows in R0's 128-row block
        for (int g = 0; g < NG2; ++g) {
          mbar_wait(&hempty[hs], hph ^ 1);
          uint32_t bytes = 0;
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const int c = 2 * g + cc;
            if (rv > 0 && c < NCH && ti.n0 + 16 * c < N) bytes += 2u * (uint32_t)rv * 32u;
          }
          mbar_arrive_expect_tx(&hfull[hs], bytes);
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const int c = 2 * g + cc;
            if (!(rv > 0 && c < NCH && ti.n0 + 16 * c < N)) continue;
#pragma unroll
            for (int part = 0; part < 2; ++part) {   // h1, h3
              const int chunk = (ti.n0 >> 4) + c + (part ? nch : 0);
              uint8_t* dst = hbuf + hs * kHSlotBytes + (cc * 2 + part) * kHChunkBytes;
              bulk_load(dst, hb + hblk_off(R0, chunk, nch), (uint32_t)n1 * 32u, &hfull[hs]);
              if (rv > n1)
                bulk_load(dst + n1 * 32, hb + hblk_off(R0 + n1, chunk, nch), (uint32_t)(rv - n1) * 32u,
                          &hfull[hs]);
            }
          }
          if (++hs == kHSlots) { hs = 0; hph ^= 1; }
        }
      }
    }
  } else {
    // ------------------------------------------------ epilogue (warps 2..2+EPI, each CTA its 128 rows)
    const int q = warp & 3;                 // TMEM lane quadrant this warp may access
    const int half = (warp - 2) >> 2;       // D2: which column groups of the quadrant
    const int r = q * 32 + lane;
    const int rc = (int)crank * BM;         // this CTA's first row of the (pair) tile
    const uint32_t te0 = PAIR ? mapa_shared(smem_u32(&tempty[0]), 0) : 0;
    const uint32_t te1 = PAIR ? mapa_shared(smem_u32(&tempty[1]), 0) : 0;
    int acc = 0; uint32_t acc_phase = 0;
    int obuf = 0;   // W modes: staging tile of this warp in use next
    int hslot = 0; uint32_t hphase = 0;   // D2: staged h1 | h3 slot
    for (int t = unit; t < p.total_tiles; t += n_units) {
      Tile ti; decode<MODE, PAIR>(p, t, ti);
      const BwdBank& bk = p.bank[ti.bank];
      const int N = ti.bank ? p.bank[1].N : p.bank[0].N;   // immediate-offset constant reads
      const int h = ti.bank ? p.bank[1].h : p.bank[0].h;
      if (MODE == BWD_D2 && !h_staged<MODE>() && t + n_units < p.total_tiles) {
        // warm L2 with the next tile's h1 | h3 (row-blocked: one 128-B line per
        // 4 rows and chunk; lanes 0, 4, .. cover this warp's 32 rows)
        Tile nx; decode<MODE, PAIR>(p, t + n_units, nx);
        if ((lane & 3) == 0 && rc + r < nx.rows_valid) {
          const BwdBank& nb = p.bank[nx.bank];
          const int nch = nb.h >> 4;
          const bf16* hb = reinterpret_cast<const bf16*>(nb.aux);
          const int64_t row = nx.row0 + rc + r;
          for (int c = half; c < BN / 16 && nx.n0 + 16 * c < nb.N; c += 2) {
            prefetch_l2(hb + hblk_off(row, (nx.n0 >> 4) + c, nch));
            prefetch_l2(hb + hblk_off(row, nch + (nx.n0 >> 4) + c, nch));
          }
        }
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tb = tmem_base + acc * 256 + ((uint32_t)(q * 32) << 16);
      const bool rv = rc + r < ti.rows_valid;
      if constexpr (h_staged<MODE>()) {
        // chunk pairs staged in shared memory by the stager warp: half h of
        // the quadrant's two warps takes chunk 2g + h of pair g
        constexpr int NCH = BN / 16, NG2 = (NCH + 1) / 2;
        const int64_t row = ti.row0 + rc + r;
        bf16* o = reinterpret_cast<bf16*>(bk.out) + row * (int64_t)(2 * h);
#pragma unroll 1
        for (int g = 0; g < NG2; ++g) {
          const int c = 2 * g + half;
          mbar_wait(&hfull[hslot], hphase);
          if (c < NCH && NIMG_BWD_PROBE == 2) {
            uint32_t a[16];
            tmem_ld16(tb + c * 16, a);
            tmem_ld_wait();
          } else if (c < NCH) {
            uint32_t a[16];
            tmem_ld16(tb + c * 16, a);
            tmem_ld_wait();
            const int n = ti.n0 + c * 16;
            if (rv && n < N) {
              const uint8_t* sl = hbuf + hslot * kHSlotBytes + (half * 2) * kHChunkBytes + r * 32;
              const uint4 v1[2] = {reinterpret_cast<const uint4*>(sl)[0], reinterpret_cast<const uint4*>(sl)[1]};
              const uint4 v3[2] = {reinterpret_cast<const uint4*>(sl + kHChunkBytes)[0],
                                   reinterpret_cast<const uint4*>(sl + kHChunkBytes)[1]};
              float h1[16], h3[16];
              unpack16(v1, h1);
              unpack16(v3, h3);
              uint32_t p1[8], p3[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                float g1[2], g3[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                  const int i = 2 * j + u;
                  const float v = __uint_as_float(a[i]);
                  const float sig = __fdividef(1.0f, 1.0f + __expf(-h1[i]));
                  g1[u] = v * h3[i] * sig * (1.0f + h1[i] * (1.0f - sig));
                  g3[u] = v * h1[i] * sig;
                }
                p1[j] = pack_bf16x2(g1[0], g1[1]);
                p3[j] = pack_bf16x2(g3[0], g3[1]);
              }
              uint4* d1 = reinterpret_cast<uint4*>(o + n);
              uint4* d3 = reinterpret_cast<uint4*>(o + h + n);
              st_global_32(d1, make_uint4(p1[0], p1[1], p1[2], p1[3]), make_uint4(p1[4], p1[5], p1[6], p1[7]));
              st_global_32(d3, make_uint4(p3[0], p3[1], p3[2], p3[3]), make_uint4(p3[4], p3[5], p3[6], p3[7]));
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&hempty[hslot]);
          if (++hslot == kHSlots) { hslot = 0; hphase ^= 1; }
        }
      } else if constexpr (MODE == BWD_D2) {
        // groups of G 16-column chunks: every h1 / h3 load of the group is in
        // flight before the first use (the rows are strided: latency-bound otherwise)
        constexpr int G = 3, NCH = BN / 16;
        const int64_t row = ti.row0 + rc + r;
        const int nch = h >> 4;
        const bf16* hb = reinterpret_cast<const bf16*>(bk.aux);
        bf16* o = reinterpret_cast<bf16*>(bk.out) + row * (int64_t)(2 * h);
#pragma unroll 1
        for (int c0 = half * G; c0 < NCH; c0 += 2 * G) {
          uint4 hv[G][4];
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const int n = ti.n0 + (c0 + g) * 16;
            if (rv && c0 + g < NCH && n < N) {
              const uint4* s1 = reinterpret_cast<const uint4*>(hb + hblk_off(row, n >> 4, nch));
              const uint4* s3 = reinterpret_cast<const uint4*>(hb + hblk_off(row, nch + (n >> 4), nch));
              hv[g][0] = __ldg(s1);
              hv[g][1] = __ldg(s1 + 1);
              hv[g][2] = __ldg(s3);
              hv[g][3] = __ldg(s3 + 1);
            }
          }
          uint32_t a[G][16];
#pragma unroll
          for (int g = 0; g < G; ++g)
            if (c0 + g < NCH) tmem_ld16(tb + (c0 + g) * 16, a[g]);
          tmem_ld_wait();
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const int n = ti.n0 + (c0 + g) * 16;
            if (!rv || c0 + g >= NCH || n >= N) continue;
            float h1[16], h3[16];
            const uint4 v1[2] = {hv[g][0], hv[g][1]}, v3[2] = {hv[g][2], hv[g][3]};
            unpack16(v1, h1);
            unpack16(v3, h3);
            uint32_t p1[8], p3[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float g1[2], g3[2];
#pragma unroll
              for (int u = 0; u < 2; ++u) {
                const int i = 2 * j + u;
                const float v = __uint_as_float(a[g][i]);
                const float sig = __fdividef(1.0f, 1.0f + __expf(-h1[i]));
                g1[u] = v * h3[i] * sig * (1.0f + h1[i] * (1.0f - sig));
                g3[u] = v * h1[i] * sig;
              }
              p1[j] = pack_bf16x2(g1[0], g1[1]);
              p3[j] = pack_bf16x2(g3[0], g3[1]);
            }
            uint4* d1 = reinterpret_cast<uint4*>(o + n);
            uint4* d3 = reinterpret_cast<uint4*>(o + h + n);
            st_global_32(d1, make_uint4(p1[0], p1[1], p1[2], p1[3]), make_uint4(p1[4], p1[5], p1[6], p1[7]));
            st_global_32(d3, make_uint4(p3[0], p3[1], p3[2], p3[3]), make_uint4(p3[4], p3[5], p3[6], p3[7]));
          }
        }
      } else if constexpr (MODE == BWD_D1) {
        bf16* const orow = reinterpret_cast<bf16*>(bk.out) + (ti.row0 + rc + r) * bk.out_ld;
#pragma unroll 1
        for (int c = 0; c < BN / 16; ++c) {
          uint32_t a[16];
          tmem_ld16(tb + c * 16, a);
          tmem_ld_wait();
          const int n = ti.n0 + c * 16;
          if (!rv || n >= N) continue;
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) pk[j] = pack_bf16x2(__uint_as_float(a[2 * j]), __uint_as_float(a[2 * j + 1]));
          uint4* dst = reinterpret_cast<uint4*>(orow + n);
          st_global_32(dst, make_uint4(pk[0], pk[1], pk[2], pk[3]), make_uint4(pk[4], pk[5], pk[6], pk[7]));
        }
      } else if constexpr (NIMG_W_SECTOR) {
        // weight gradient stored from registers in whole 32-B sectors: the
        // 16x256b TMEM load gives four lanes 8 contiguous fp32 of one row, so
        // each warp store writes 8 rows x 32 B (no shared-memory staging, no
        // partial-sector writes). W1: rows [0, h) -> dW1, [h, 2h) -> dW3.
        const int m_w = ti.m0 + rc + q * 32;                  // this warp's first row
        const bool to3 = MODE == BWD_W1 && m_w >= h;
        const int mrows = MODE == BWD_W1 ? h : bk.M;          // rows of one output slice
        float* ob = reinterpret_cast<float*>(to3 ? bk.out3 : bk.out) +
                    ((int64_t)ti.expert * mrows + (to3 ? m_w - h : m_w)) * (int64_t)N;
        const int lr = lane >> 2, lc = 2 * (lane & 3);
#pragma unroll 1
        for (int cc = 0; cc < BN / 32; ++cc) {
          uint32_t a0[16], a1[16];
          tmem_ld16x256(tb + cc * 32, a0);                          // rows 0-15 of the warp
          tmem_ld16x256(tb + ((uint32_t)16 << 16) + cc * 32, a1);   // rows 16-31
          tmem_ld_wait();
          const int n = ti.n0 + cc * 32;
          if (n >= N) continue;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const uint32_t* a = hh ? a1 : a0;
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
              const int row = 16 * hh + 8 * rr + lr;
              if (m_w + row >= bk.M) continue;
              float* o = ob + (int64_t)row * N + n + lc;
#pragma unroll
              for (int i = 0; i < 4; ++i)
                if (n + 8 * i + lc < N)
                  *reinterpret_cast<float2*>(o + 8 * i) =
                      make_float2(__uint_as_float(a[4 * i + 2 * rr]), __uint_as_float(a[4 * i + 2 * rr + 1]));
            }
          }
        }
      } else {
        // weight gradient: 32 rows x 32 fp32 per warp per step, staged in a
        // 128-B-swizzled smem tile and written by one TMA store (coalesced,
        // edge-clipped by the tensor map). W1: rows [0, h) -> dW1, [h, 2h) -> dW3
        // (h % 32 == 0, so a warp's 32 rows never straddle).
        const int m_w = ti.m0 + rc + q * 32;                  // this warp's first row
        const bool to3 = MODE == BWD_W1 && m_w >= h;
        const void* omap = to3 ? (const void*)&tm.o3[ti.bank] : (const void*)&tm.o[ti.bank];
        const int orow = to3 ? m_w - h : m_w;
        const bool any = m_w < bk.M;
#pragma unroll 1
        for (int cc = 0; cc < BN / 32; ++cc) {
          uint32_t a[32];
          tmem_ld16(tb + cc * 32, *reinterpret_cast<uint32_t(*)[16]>(&a[0]));
          tmem_ld16(tb + cc * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(&a[16]));
          tmem_ld_wait();
          const int n = ti.n0 + cc * 32;
          if (!any || n >= N || NIMG_BWD_PROBE == 1) continue;
          uint8_t* sbuf = stage_out + (q * 2 + obuf) * kStageOut;
          if (lane == 0) bulk_wait_read<1>();                 // the store that used this tile is done
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<uint4*>(sbuf + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                make_uint4(a[4 * j], a[4 * j + 1], a[4 * j + 2], a[4 * j + 3]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(omap, sbuf, n, orow, ti.expert);
            bulk_commit();
          }
          obuf ^= 1;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR) mbar_arrive_remote(acc ? te1 : te0);
        else mbar_arrive(&tempty[acc]);
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (AMN && !NIMG_W_SECTOR && lane == 0) bulk_wait<0>();
  }

  tc_fence_before();
  if (PAIR) cluster_sync(); else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (PAIR) tmem_dealloc_cg2(tmem_base, 512); else tmem_dealloc(tmem_base, 512);
  }
}

}  // namespace tcb

// CTA-pair backward kernels (default); NIMG_PAIR=0 selects the 1-CTA ones.
static bool bwd_pair() {
  static const bool on = [] {
    const char* e = getenv("NIMG_PAIR");
    return !(e && e[0] == '0');
  }();
  return on;
}
bool tc_bwd_pair(int mode) { return mode != BWD_WR && bwd_pair(); }

int tc_bwd_bn(int mode) {
  const bool pr = tc_bwd_pair(mode);
  switch (mode) {
    case BWD_D2: return pr ? tcb::Cfg<BWD_D2, true>::BN : tcb::Cfg<BWD_D2, false>::BN;
    case BWD_D1: return pr ? tcb::Cfg<BWD_D1, true>::BN : tcb::Cfg<BWD_D1, false>::BN;
    case BWD_W2: return pr ? tcb::Cfg<BWD_W2, true>::BN : tcb::Cfg<BWD_W2, false>::BN;
    case BWD_WR: return tcb::Cfg<BWD_WR, false>::BN;
    default: return pr ? tcb::Cfg<BWD_W1, true>::BN : tcb::Cfg<BWD_W1, false>::BN;
  }
}
int tc_bwd_tile_rows(int mode) { return tc_bwd_pair(mode) ? 2 * tcb::BM : tcb::BM; }

template <int MODE, bool PAIR>
static cudaError_t launch_bwd(const TmapSetBwd& tm, const BwdParams& p, int num_sms, cudaStream_t s) {
  constexpr int smem = tcb::smem_bytes<MODE, PAIR>();
  cudaError_t e = set_max_dyn_smem(tcb::grouped_gemm_bwd_sm100<MODE, PAIR>, smem);
  if (e != cudaSuccess) return e;
  const int units = PAIR ? num_sms / 2 : num_sms;
  const int grid = (p.total_tiles < units ? p.total_tiles : units) * (PAIR ? 2 : 1);
  if (!PAIR)
    return launch_pdl(tcb::grouped_gemm_bwd_sm100<MODE, PAIR>, dim3(grid), dim3(tcb::threads<MODE>()),
                      (size_t)smem, s, tm, p);
  // cluster of 2 along x (the forward pair kernel declares it statically; here
  // one template serves both, so the launch attribute sets it)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(tcb::threads<MODE>());
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr2[2];
  attr2[0].id = cudaLaunchAttributeClusterDimension;
  attr2[0].val.clusterDim.x = 2;
  attr2[0].val.clusterDim.y = 1;
  attr2[0].val.clusterDim.z = 1;
  attr2[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr2[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr2;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, tcb::grouped_gemm_bwd_sm100<MODE, PAIR>, tm, p);
}

cudaError_t launch_grouped_tc_bwd(int mode, const TmapSetBwd& tm, const BwdParams& p, int num_sms,
                                  cudaStream_t s) {
  if (p.total_tiles <= 0) return cudaSuccess;
  const bool pr = tc_bwd_pair(mode);
  switch (mode) {
    case BWD_D2: return pr ? launch_bwd<BWD_D2, true>(tm, p, num_sms, s) : launch_bwd<BWD_D2, false>(tm, p, num_sms, s);
    case BWD_D1: return pr ? launch_bwd<BWD_D1, true>(tm, p, num_sms, s) : launch_bwd<BWD_D1, false>(tm, p, num_sms, s);
    case BWD_W2: return pr ? launch_bwd<BWD_W2, true>(tm, p, num_sms, s) : launch_bwd<BWD_W2, false>(tm, p, num_sms, s);
    case BWD_WR: return launch_bwd<BWD_WR, false>(tm, p, num_sms, s);
    default: return pr ? launch_bwd<BWD_W1, true>(tm, p, num_sms, s) : launch_bwd<BWD_W1, false>(tm, p, num_sms, s);
  }
}

}  // namespace nimg
