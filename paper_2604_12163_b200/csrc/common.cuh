// Shared device helpers for the sm_100a expert-choice MoE kernels:
// mbarrier / TMA / tcgen05 inline PTX, bf16 packing, and numpy-order sums.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define NIMG_DEV __device__ __forceinline__

namespace nimg {

typedef __nv_bfloat16 bf16;

// ---------------------------------------------------------------- basics
// Programmatic dependent launch. Every kernel of the layer triggers its
// dependents on entry and waits for its predecessor before its first global
// access, so a kernel's launch and prologue overlap the previous kernel's tail
// while all memory effects stay in stream order (each wait covers the whole
// chain transitively). Both are no-ops for a launch without the attribute.
NIMG_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
NIMG_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

NIMG_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

NIMG_DEV float to_f32(float v) { return v; }
NIMG_DEV float to_f32(bf16 v) { return __bfloat162float(v); }
template <typename T> NIMG_DEV T from_f32(float v);
template <> NIMG_DEV float from_f32<float>(float v) { return v; }
template <> NIMG_DEV bf16 from_f32<bf16>(float v) { return __float2bfloat16_rn(v); }

NIMG_DEV uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// ---------------------------------------------------------------- mbarrier
NIMG_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
NIMG_DEV void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
NIMG_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
NIMG_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
NIMG_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ---------------------------------------------------------------- TMA
NIMG_DEV void tma_prefetch_desc(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}
NIMG_DEV void tma_load_2d(void* smem_dst, const void* tmap, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
NIMG_DEV void tma_load_3d(void* smem_dst, const void* tmap, uint64_t* bar, int c0, int c1,
                          int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// 4 arbitrary rows (r0..r3) x one box of columns from a 2-D map whose box is
// {cols, 1}; lands as 4 consecutive (swizzled) rows at smem_dst.
NIMG_DEV void tma_gather4(void* smem_dst, const void* tmap, uint64_t* bar, int col, int r0, int r1,
                          int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(col), "r"(r0), "r"(r1),
      "r"(r2), "r"(r3)
      : "memory");
}

// TMA tensor store (smem -> global, bulk-group completion) and its fences.
NIMG_DEV void tma_store_3d(const void* tmap, const void* smem_src, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(tmap)),
      "r"(smem_u32(smem_src)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
NIMG_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> NIMG_DEV void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N> NIMG_DEV void bulk_wait() { asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory"); }
NIMG_DEV void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
// Bulk L2 prefetch of `bytes` (multiple of 16) starting at a 16-B aligned address.
NIMG_DEV void bulk_prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// ---------------------------------------------------------------- clusters
NIMG_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
NIMG_DEV void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cta address -> shared::cluster address of the same offset in CTA `rank`
NIMG_DEV uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// Remote arrive with the default (CTA-scope release) semantics: for the
// TMEM-buffer-free signal of the pair epilogues, which only orders the
// preceding tcgen05 loads (tcgen05.fence::before_thread_sync) -- a
// cluster-scope release would also wait for every outstanding global store
// of the arriving thread (MEMBAR.ALL.GPU).
NIMG_DEV void mbar_arrive_remote(uint32_t cluster_addr) {
#if defined(NIMG_ARRIVE_CLUSTER_RELEASE)
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
#else
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
#endif
}
NIMG_DEV void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// 2-CTA TMA: data lands in this CTA's smem, completion is signalled on an
// mbarrier that may live in the peer CTA of the pair (the MMA leader).
NIMG_DEV void tma_load_2d_cg2(void* smem_dst, const void* tmap, uint32_t bar_cluster, int c0,
                              int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}
NIMG_DEV void tma_load_3d_cg2(void* smem_dst, const void* tmap, uint32_t bar_cluster, int c0,
                              int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// ---------------------------------------------------------------- cp.async (LDGSTS)
NIMG_DEV void cp_async_16(uint32_t smem_addr, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr), "l"(gmem) : "memory");
}
NIMG_DEV void cp_async_commit_group() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> NIMG_DEV void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// arrive on `bar` once all of this thread's prior cp.async have landed
// (.noinc: the barrier's init count includes these arrivals)
NIMG_DEV void cp_async_mbar_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// generic-proxy shared-memory writes -> visible to the async proxy (UMMA reads)
NIMG_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ---------------------------------------------------------------- tcgen05
NIMG_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
NIMG_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Whole warp: allocate `ncols` TMEM columns, base address written to smem.
NIMG_DEV void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
NIMG_DEV void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}

NIMG_DEV void tmem_alloc_cg2(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
NIMG_DEV void tmem_dealloc_cg2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
// Pair MMA (leader CTA issues): A rows 0..127 from this CTA's smem and
// 128..255 from the peer's (same offsets); B rows split N/2 per CTA.
NIMG_DEV void umma_bf16_cg2(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive (once the pair's prior MMAs complete) on the barrier at this smem
// offset in every CTA of `mask`.
NIMG_DEV void umma_commit_cg2(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, bf16 inputs, fp32 accumulate; one thread issues.
NIMG_DEV void umma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on an mbarrier once all previously issued tcgen05.mma of this thread complete.
NIMG_DEV void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns -> 16 registers per thread.
NIMG_DEV void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
// 16 TMEM lanes x 32 fp32 columns (4 repeats of 256 bits): thread t holds row
// t/4 (regs 4i, 4i+1) and row t/4 + 8 (regs 4i+2, 4i+3) at columns
// 8i + 2(t%4) + {0, 1} -- four lanes cover 32 contiguous bytes of a row.
NIMG_DEV void tmem_ld16x256(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
// 32 contiguous bytes from one thread: one 256-bit store (STG.256, a whole L2
// sector) when 32-B aligned, else two 16-B stores. NIMG_ST256=0: always two.
#ifndef NIMG_ST256
#define NIMG_ST256 1
#endif
NIMG_DEV void st_global_32(void* p, uint4 lo, uint4 hi) {
  if (NIMG_ST256 && (reinterpret_cast<uintptr_t>(p) & 31u) == 0u) {
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(lo.x), "r"(lo.y),
                 "r"(lo.z), "r"(lo.w), "r"(hi.x), "r"(hi.y), "r"(hi.z), "r"(hi.w)
                 : "memory");
  } else {
    reinterpret_cast<uint4*>(p)[0] = lo;
    reinterpret_cast<uint4*>(p)[1] = hi;
  }
}
NIMG_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor, K-major operand, 128B swizzle: 8-row atoms of
// 128 B rows, atoms 1024 B apart (SBO), LBO unused (=1), version 1 (sm_100).
NIMG_DEV uint64_t make_sdesc_k128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;             // LBO (16 B units)
  d |= (uint64_t)(1024 >> 4) << 32;   // SBO
  d |= (uint64_t)1 << 46;             // descriptor version
  d |= (uint64_t)2 << 61;             // SWIZZLE_128B
  return d;
}

// UMMA shared-memory descriptor, MN-major operand, 128B swizzle (canonical
// ((8,n),(8,k)):((1,LBO),(8,SBO)) in 16-B units): each k row holds 64
// MN-contiguous bf16 (128 B), 8 k rows form a 1024-B swizzle atom (SBO apart),
// and successive 64-wide MN chunks sit `lbo_bytes` apart. This is exactly
// what a TMA box {64 (MN), k rows} with SWIZZLE_128B lands.
NIMG_DEV uint64_t make_sdesc_mn128(uint32_t smem_addr, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;   // LBO: MN-chunk stride
  d |= (uint64_t)(1024 >> 4) << 32;                    // SBO: 8-k-row group stride
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor: kind::f16, A/B bf16, D fp32, K-major A and B.
__host__ __device__ constexpr uint32_t make_idesc_bf16(int M, int N) {
  return (1u << 4)                       // D format f32
         | (1u << 7)                     // A bf16
         | (1u << 10)                    // B bf16
         | ((uint32_t)(N >> 3) << 17)    // N
         | ((uint32_t)(M >> 4) << 24);   // M
}
// Same with per-operand major-ness (bit 15: A MN-major, bit 16: B MN-major).
__host__ __device__ constexpr uint32_t make_idesc_bf16_major(int M, int N, bool a_mn, bool b_mn) {
  return make_idesc_bf16(M, N) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16);
}

// ---------------------------------------------------------------- saved h1 | h3 layout
// The tcgen05 training forward keeps h1 = x W1^T and h3 = x W3^T for the
// SwiGLU pullback in a row-blocked layout matched to the epilogues that write
// (GEMM1) and read (dgrad of GEMM2) it: both hold one row per thread and 16
// columns per step, so each (128-row block, 16-column chunk) is one contiguous
// 4-KB block with a row's 16 values at row%128 * 32 B -- a warp's 32 rows are
// 1 KB contiguous (coalesced), where a row-major [rows][2h] layout would be 32
// separate lines. Chunks [0, nch) are h1, [nch, 2 nch) are h3 (nch = h / 16).
NIMG_DEV int64_t hblk_off(int64_t row, int chunk, int nch) {
  return (((row >> 7) * (2 * nch) + chunk) << 11) + ((row & 127) << 4);
}

// ---------------------------------------------------------------- int8 tcgen05 / bulk copy
// D[tmem] (+)= A[smem] * B[smem]^T, signed int8 inputs, exact int32 accumulate.
NIMG_DEV void umma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                      uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Instruction descriptor: kind::i8, A/B signed int8, D s32, K-major A and B.
__host__ __device__ constexpr uint32_t make_idesc_s8(int M, int N) {
  return (2u << 4)                       // D format s32
         | (1u << 7)                     // A signed 8-bit
         | (1u << 10)                    // B signed 8-bit
         | ((uint32_t)(N >> 3) << 17)
         | ((uint32_t)(M >> 4) << 24);
}
// 32 lanes x 32 bit, 8 consecutive columns -> 8 registers per thread.
NIMG_DEV void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
}
NIMG_DEV void tmem_ld4(uint32_t taddr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}
// Plain (non-tensor) bulk copy global -> shared, completion on an mbarrier.
NIMG_DEV void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------- router t half
// The t half of the router product [x_norm || t_emb] . W_r (router.py:120-122)
// is per sample: part[b, ks, e] = sum over the ks-th k-range of t_emb[b, k] *
// W_r[d + k, e] in f64, computed by a block of 256 threads (thread (e, q) sums
// one of 4 sub-slices, folded in a fixed order), and folded per sample in ks
// order by router_tbias (deterministic). Shared by the DMMA and int8 routers so
// both add the identical f64 t-bias.
__host__ __device__ inline int router_tpart_ks(int d) {
  const int nkc = (d + 63) / 64;   // <= router_part_bytes' chunk count: the partials fit
  return nkc < 8 ? nkc : 8;
}
NIMG_DEV void router_tpart_block(const float* __restrict__ t_emb, const float* __restrict__ w_r,
                                 double* __restrict__ part, int b, int ks, int d, int E) {
  __shared__ double sp[4][64];
  const int KS = router_tpart_ks(d);
  const int e = threadIdx.x & 63, q = threadIdx.x >> 6;
  const int nsl = 4 * KS, sl = ks * 4 + q;
  const int klen = (d + nsl - 1) / nsl, k0 = sl * klen, k1 = min(d, k0 + klen);
  double acc = 0.0;
  if (e < E) {
    const float* t = t_emb + (int64_t)b * d;
    const float* w = w_r + (int64_t)d * E + e;
    int k = k0;
    for (; k + 16 <= k1; k += 16) {   // loads batched ahead of the (sequential) f64 chain
      float tv[16], wv[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        tv[i] = __ldg(t + k + i);
        wv[i] = __ldg(w + (int64_t)(k + i) * E);
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) acc = fma((double)tv[i], (double)wv[i], acc);
    }
    for (; k < k1; ++k) acc = fma((double)__ldg(t + k), (double)__ldg(w + (int64_t)k * E), acc);
  }
  sp[q][e] = acc;
  __syncthreads();
  if (q == 0 && e < E)
    part[((int64_t)b * KS + ks) * E + e] = ((sp[0][e] + sp[1][e]) + sp[2][e]) + sp[3][e];
}
NIMG_DEV double router_tbias(const double* __restrict__ part, int64_t b, int e, int d, int E) {
  const int KS = router_tpart_ks(d);
  const double* pp = part + (b * KS) * E + e;
  double r = pp[0];
  for (int ks = 1; ks < KS; ++ks) r += pp[(int64_t)ks * E];
  return r;
}

// ---------------------------------------------------------------- numpy sum
// Exact restatement of numpy's pairwise summation (float add.reduce over a
// contiguous axis, e.g. `e.sum(axis=-1)` / `mean` in tensor.py:471, :527):
// < 8 terms sequential from 0.0; <= 128 terms with eight stride-8
// accumulators folded ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a sequential
// tail; larger n split at n/2 rounded down to a multiple of 8.
static __device__ __noinline__ double np_pairwise_sum(const double* a, int n) {
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

}  // namespace nimg
