// Router logits on the INT8 tensor cores, exact: the x half of
// [x_norm || t_emb] . W_r (router.py:120-122, tensor.py:280-296) for bf16
// x_norm and E == 64 experts.
//
// The reference sums the products in f64 and rounds once to fp32. A bf16 x has
// an 8-bit significand and an fp32 W_r a 24-bit one, so the x half is an exact
// sum of integers once both sides are written in fixed point:
//
//   x[t, k] = X[t, k] * 2^(e_t - 134 - XW), |X| < 2^(XW+8) = 2^31  (row scale)
//   w[k, e] = W[k, e] * 2^(ew_e - WEXP),    |W| < 2^39                (column scale)
//
// Both are cut into base-256 digits, two's complement: X = sum_i X_i 256^(3-i)
// and W = sum_j W_j 256^(4-j), the top digit signed and the others unsigned
// bytes. Then sum_k X W = sum_s G_s 256^(7-s), G_s = sum_{i+j=s} sum_k X_i W_j,
// where every G_s is an int8 x int8 GEMM with int32 accumulation: EXACT, in any
// order (tcgen05.mma kind::i8, whose A / B signedness is per instruction: per
// K step, digit i x W_0 (N = 64, B signed) lands on TMEM group i and digit i x
// [W_1|W_2|W_3|W_4] (N = 256, B unsigned) on groups i+1..i+4). (NIMG_I8_B256=0
// builds the round-1/2 scheme: 7-bit balanced / sign-magnitude digits, 28-bit x
// and 35-bit W windows.)
// Elements outside the fixed-point windows are not lost: a W element below
// 2^-15 of its column max becomes an exact f64 correction term (a per-expert
// list of up to CORR_MAX, ascending k), and an x element outside its row's XW-binade window (the
// scale is guessed from the row's first 128 elements, XH binades of headroom)
// becomes an exact f64 term in a per-row list; a row whose list overflows is
// recomputed by the f64 fix-up kernel. The epilogue forms v = H 2^32 + L
// exactly in int64 halves, scales by a power of two, adds the corrections and
// the f64 t-bias, rounds to fp32 and PROVES the rounding: if the f64 value is
// not farther than its error bound from an fp32 rounding boundary, the token is
// recomputed by the fix-up kernel with a plain f64 dot (the DMMA router's
// arithmetic). The fp32 logits therefore equal the correctly rounded f64 ones
// -- the same bits the f64 routers produce -- at int8 tensor-core speed.
//
// Kernels: router_prep_i8 (t-half partials, W digit image in the UMMA smem
// layout, correction lists, counter reset), router_scores_i8 (one CTA per 128
// tokens, 18 warps: 16 converter warps write the x digits into 128-B swizzled
// smem, a producer warp bulk-copies the W digits, one thread issues the MMAs,
// and the 16 converter warps then run the epilogue and the numpy-order f64
// softmax), router_fix_i8 (flagged tokens, f64). At cfg2 (T = 16384): 8.8 +
// 68 + 3.5 us against 174 us for the FP64 DMMA router (profiles/r01b_*).
#include <cstdio>
#include <cstring>

#include "common.cuh"
#include "nimg_internal.h"

namespace nimg {
namespace ri8 {

constexpr int NE = 64;                       // experts = UMMA N
constexpr int BM = 128;                      // tokens per CTA = UMMA M = TMEM lanes
// k per stage = the int8 row of one swizzle atom: 64 (64-B swizzle, 4 stages of
// 52 KB: the MMAs never wait on a refill) or 128 (128-B swizzle, 2 stages of
// 104 KB: measured MMA-starved, profiles/r02_router_ncu.md)
#ifndef NIMG_I8_KB
#define NIMG_I8_KB 64
#endif
constexpr int KB = NIMG_I8_KB;
static_assert(KB == 64 || KB == 128, "stage k width");
constexpr int CPR = KB / 16;                 // 16-element chunks per row and stage
// byte offset of 16-B chunk c of K-major row r inside a swizzled operand slice
NIMG_DEV int swz_off(int r, int c) {
  return KB == 128 ? r * KB + ((c ^ (r & 7)) << 4) : r * KB + ((c ^ ((r >> 1) & 3)) << 4);
}
NIMG_DEV uint64_t sdesc_k(uint32_t addr) {
  if (KB == 128) return make_sdesc_k128(addr);
  uint64_t dsc = 0;                           // K-major, 64-B swizzle: 8-row atoms of 64 B
  dsc |= (uint64_t)((addr >> 4) & 0x3FFF);
  dsc |= (uint64_t)1 << 16;                   // LBO (unused)
  dsc |= (uint64_t)(512 >> 4) << 32;          // SBO: 8 rows x 64 B
  dsc |= (uint64_t)1 << 46;                   // descriptor version (sm_100)
  dsc |= (uint64_t)4 << 61;                   // SWIZZLE_64B
  return dsc;
}
// x digit planes: 4 (28-bit window, the default) or 3 (21-bit: measured slower,
// its narrower window sends ~1 element per row to the exact f64 list); W_r always 5
#ifndef NIMG_I8_LX
#define NIMG_I8_LX 4
#endif
// Digit base. 256 (default): x and W are two's-complement integers cut into
// bytes -- the top byte signed, the others unsigned (tcgen05 kind::i8 takes the
// signedness of A and B per instruction) -- with a 32-bit x window (24
// binades) and a 40-bit W window. 128: balanced / sign-magnitude 7-bit digits,
// 28-bit x window (19 binades), 35-bit W window (the round-1/2 scheme).
#ifndef NIMG_I8_B256
#define NIMG_I8_B256 1
#endif
constexpr bool B256 = NIMG_I8_B256;
constexpr int LX = NIMG_I8_LX, LW = 5, NG = LX + LW - 1;
// binades of the x window: 12 or 19 (base 128; |X| < 2^(7 LX - 1) keeps every
// balanced digit of the fast path within [-64, 64] and the top digit of the
// slow path's two's-complement split within [-64, 63]), 23 (base 256: |X| <
// 2^31, an int32)
constexpr int XW = B256 ? 8 * LX - 9 : 7 * LX - 9;
constexpr int DB = B256 ? 8 : 7;             // bits per digit
// W column window: the column max's 24-bit significand M lands as M << WSH
// (base 256: |W| < 2^39, a signed 40-bit integer; base 128: 35-bit magnitude)
constexpr int WSH = B256 ? LW * DB - 25 : LW * DB - 24;
constexpr int WEXP = 150 + WSH;              // w = W * 2^(ew - WEXP)
// Fast-path conversion on the FMA pipe (NIMG_I8_FCONV=0: the integer path)
#ifndef NIMG_I8_FCONV
#define NIMG_I8_FCONV 1
#endif
// NIMG_I8_TRACE=1: CTAs 0 and 64 printf a %globaltimer trace (A/B builds only)
#ifndef NIMG_I8_TRACE
#define NIMG_I8_TRACE 0
#endif
NIMG_DEV uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// timing probes for A/B builds only (wrong results): 1 = no conversion,
// 2 = no MMAs, 3 = no epilogue
#ifndef NIMG_I8_PROBE
#define NIMG_I8_PROBE 0
#endif
constexpr int XH = LX == 3 ? 1 : 2;          // headroom over the first-stage max (binades)
static_assert(LX == 3 || LX == 4, "x digit planes");
constexpr int A_SLICE = BM * KB;             // 8 / 16 KB
constexpr int W_SLICE = NE * KB;             // 4 / 8 KB
constexpr int W_STAGE = LW * W_SLICE;        // 20 / 40 KB
constexpr int STAGE = LX * A_SLICE + W_STAGE;   // 52 / 104 KB (LX = 4)
constexpr int NSTAGE = KB == 64 ? 4 : 2;
constexpr int NCONV = 512;                   // converter / epilogue threads (warps 0-15)
constexpr int JOBS = BM * CPR / NCONV;       // 16-element chunks per converter thread and stage
constexpr int XPF = KB == 64 ? 2 : 1;        // x stages prefetched ahead in registers
constexpr int THREADS = NCONV + 64;          // + MMA warp 16 + W producer warp 17
constexpr int CORR_MAX = 256;                // exact W corrections per expert (more: f64 path)
constexpr int CORR_SM = 32;                  // of them staged in smem for the epilogue
constexpr int XC_MAX = 8;                    // exact x terms per row (more: f64 row)
// control block after the stages: barriers, TMEM slot, per-row scale / flag /
// x-term lists
constexpr int C_EMAX = 256, C_RFLAG = C_EMAX + BM * 4, C_XCN = C_RFLAG + BM * 4;
constexpr int C_XCK = C_XCN + BM * 4, C_XCV = C_XCK + BM * XC_MAX * 4;
constexpr int CTRL = C_XCV + BM * XC_MAX * 4;
constexpr size_t EPI_END = 195584;           // end of the epilogue buffers (below)
// the stage ring, reused by the epilogue once the MMAs have drained it
constexpr size_t BUF = (size_t)NSTAGE * STAGE > EPI_END ? (size_t)NSTAGE * STAGE : EPI_END;
constexpr size_t SMEM = BUF + CTRL + 1024;
// epilogue reuse of the (drained) stage buffers
constexpr int LGS = NE + 1;                  // padded row strides (bank spread)
constexpr size_t TBS_OFF = 0;                // folded t-bias, <= 130 samples x 64 f64
constexpr size_t LG_OFF = 67584;             // fp32 logits [128][65]
constexpr size_t EX_OFF = 101376;            // f64 exp [128][65]
constexpr size_t WC_OFF = 167936;            // W corrections staged: k, dw, counts, scales
constexpr size_t PM_OFF = 193536;            // per-row partial maxima [128][4] fp32
static_assert(WC_OFF + (size_t)NE * CORR_SM * 12 + NE * 8 <= PM_OFF, "epilogue smem");
static_assert(PM_OFF + (size_t)BM * 4 * 4 <= EPI_END, "epilogue smem");
static_assert(EX_OFF + (size_t)BM * LGS * 8 <= WC_OFF, "epilogue smem");
static_assert(LG_OFF + (size_t)BM * LGS * 4 <= EX_OFF, "epilogue smem");


struct Ws {
  uint8_t* wimg;      // [d/KB][LW][64 rows x KB B, swizzled]
  int* ew;            // [64] column exponent (biased)
  int* ccnt;          // [64] corrections per expert
  int* ck;            // [64][CORR_MAX] k of each correction (ascending)
  double* cdw;        // [64][CORR_MAX] w - w~ (exact)
  int* bflag;         // [64] column needs the f64 path for every token
  unsigned* counter;  // flagged-token count
  int* list;          // [T] flagged tokens
};
inline size_t al(size_t x) { return (x + 255) & ~size_t(255); }
inline size_t ws_bytes(int64_t T, int d) {
  return al((size_t)(d / KB) * W_STAGE) + al(NE * 4) * 2 + al((size_t)NE * CORR_MAX * 4) +
         al((size_t)NE * CORR_MAX * 8) + al(NE * 4) + al(16) + al((size_t)T * 4);
}
inline Ws carve(void* base, int64_t T, int d) {
  uint8_t* p = static_cast<uint8_t*>(base);
  Ws w;
  w.wimg = p;                                    p += al((size_t)(d / KB) * W_STAGE);
  w.ew = reinterpret_cast<int*>(p);              p += al(NE * 4);
  w.ccnt = reinterpret_cast<int*>(p);            p += al(NE * 4);
  w.ck = reinterpret_cast<int*>(p);              p += al((size_t)NE * CORR_MAX * 4);
  w.cdw = reinterpret_cast<double*>(p);          p += al((size_t)NE * CORR_MAX * 8);
  w.bflag = reinterpret_cast<int*>(p);           p += al(NE * 4);
  w.counter = reinterpret_cast<unsigned*>(p);    p += al(16);
  w.list = reinterpret_cast<int*>(p);
  (void)T;
  return w;
}

NIMG_DEV double pow2(int e) {   // 2^e for -1022 <= e <= 1023
  return __hiloint2double((e + 1023) << 20, 0);
}
// 28-bit magnitude -> four 7-bit digits, byte 3 = most significant
NIMG_DEV uint32_t spread7(uint32_t X) {
  return (X & 0x7Fu) | ((X << 1) & 0x7F00u) | ((X << 2) & 0x7F0000u) | ((X << 3) & 0x7F000000u);
}
// Signed 28-bit X -> its base-128 digits, one per byte: bytes 0-2 unsigned
// 7-bit, byte 3 the signed top digit (X >> 21), so X = sum_i byte_i 128^i with
// every byte a valid int8. Each step doubles the part above a digit boundary
// (inserts the 8th bit), valid for negative X in two's complement too.
NIMG_DEV uint32_t spread_signed(uint32_t X) {
  X += X & ~0x7Fu;
  X += X & ~0x7FFFu;
  if (LX == 4) X += X & ~0x7FFFFFu;
  return X;
}
// X (|X| < 2^(DB LX - 1), two's complement) -> its digits, byte i = digit i
// from the bottom: base 256 is X itself
NIMG_DEV uint32_t spread_digits(uint32_t X) { return B256 ? X : spread_signed(X); }
// per-byte negation of digits in [0, 127]
NIMG_DEV uint32_t neg_bytes(uint32_t Y) { return (0x80808080u - Y) ^ 0x80808080u; }
NIMG_DEV void bar_conv() { asm volatile("bar.sync 1, 512;" ::: "memory"); }

// Fast-path digits on the FMA pipe. For an element inside the row's window,
// X = x * 2^(134 + XW - e_t) is an integer, |X| < 2^(XW+8), and
//   t3 = fl(X + 1.5*2^44)   rounds X to a multiple of 2^21: D3 = the rounded
//                           quotient sits in t3's low mantissa bits
//   r3 = X - (t3 - 1.5*2^44)   exact, |r3| <= 2^20
// and likewise 2^14, 2^7, 1 for D2, D1, D0: balanced digits in [-64, 64]
// with X = sum D_i 128^i, each the low byte (two's complement) of its float's
// bit pattern. Every step is exact (the operands stay inside one binade of
// the magic constant), so the integer MMA sees exactly X. Two FFMA and eight
// FADD per element on the FMA pipe, against ~20 ALU-pipe shift / mask / add
// operations for the integer split (ALU rt = 2/SMSP: that split bounded the
// kernel, ncu profiles/r02_router_ncu.md).
template <int LXD>
NIMG_DEV void digits_fma(float x, float scale, uint32_t (&t)[LXD]) {
  constexpr float M3 = 26388279066624.0f, M2 = 206158430208.0f, M1 = 1610612736.0f,
                  M0 = 12582912.0f;   // 1.5 * 2^{44, 37, 30, 23}
  if (LXD == 4) {
    const float t3 = fmaf(x, scale, M3);
    const float r3 = fmaf(x, scale, -(t3 - M3));
    const float t2 = r3 + M2;
    const float r2 = r3 - (t2 - M2);
    const float t1 = r2 + M1;
    const float r1 = r2 - (t1 - M1);
    t[0] = __float_as_uint(t3);
    t[1] = __float_as_uint(t2);
    t[2] = __float_as_uint(t1);
    t[3] = __float_as_uint(r1 + M0);
  } else {
    const float t2 = fmaf(x, scale, M2);
    const float r2 = fmaf(x, scale, -(t2 - M2));
    const float t1 = r2 + M1;
    const float r1 = r2 - (t1 - M1);
    t[0] = __float_as_uint(t2);
    t[1] = __float_as_uint(t1);
    t[2] = __float_as_uint(r1 + M0);
  }
}

// Base-256 fast path. X = x * 2^(134 + XW - e_t) is an integer, |X| < 2^31:
//   t = RD(X + 1.5*2^39)   (fma.rm) = 1.5*2^39 + q 2^16, q = floor(X / 2^16):
//                          t's low 16 mantissa bits are q (two's complement),
//                          the top digit (signed) and digit 2 (unsigned); with
//                          LX = 3 (|X| < 2^23) q is the top digit itself
//   r = X - q 2^16         exact, 0 <= r < 2^16
//   u = r + 1.5*2^23       u's low 16 bits are r: digits 1 and 0 (unsigned)
// so X = D3 2^24 + D2 2^16 + D1 2^8 + D0 exactly, in 4 FMA-pipe operations
// (LX = 3: X = D2 2^16 + D1 2^8 + D0).
NIMG_DEV void digits_b256(float x, float scale, uint32_t& hi, uint32_t& lo) {
  constexpr float MH = 824633720832.0f, ML = 12582912.0f;   // 1.5 * 2^39, 1.5 * 2^23
  const float t = __fmaf_rd(x, scale, MH);
  const float r = fmaf(x, scale, -(t - MH));
  hi = __float_as_uint(t);
  lo = __float_as_uint(r + ML);
}

// ------------------------------------------------------------------ prep
// blocks [0, B*KS): t-half partials (shared with the DMMA router).
// blocks [B*KS, + 64): block e owns expert column e: the column's max exponent,
// its five W digit planes written straight into the smem image the scores
// kernel bulk-copies (K-major, 128-B swizzle), and the exact corrections of
// the elements below the column window (WSH + 24 bits), in ascending k.
__global__ void __launch_bounds__(256)
router_prep_i8_kernel(const float* __restrict__ t_emb, const float* __restrict__ w_r,
                      double* __restrict__ part, Ws ws, int B, int d, ZeroSpans zs) {
  pdl_trigger();
  // buffers later kernels of the step accumulate into (the layer forward's
  // token masks and GEMM1's gather flags); every earlier use is complete, as
  // this is an ordinary launch
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < zs.n64;
       i += (int64_t)gridDim.x * blockDim.x)
    zs.p64[i] = 0ull;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < zs.n32;
       i += (int64_t)gridDim.x * blockDim.x)
    zs.p32[i] = 0;
  const int KS = router_tpart_ks(d);
  if ((int)blockIdx.x < B * KS) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *ws.counter = 0u;
    router_tpart_block(t_emb, w_r, part, blockIdx.x / KS, blockIdx.x % KS, d, NE);
    return;
  }
  __shared__ uint32_t red[8];
  __shared__ int wsum[8];
  __shared__ int sbad;
  const int e = blockIdx.x - B * KS;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t* wu = reinterpret_cast<const uint32_t*>(w_r);
  uint32_t mx = 0;
  for (int k = tid; k < d; k += 256) mx = max(mx, __ldg(wu + (int64_t)k * NE + e) & 0x7FFFFFFFu);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if (lane == 0) red[warp] = mx;
  if (tid == 0) sbad = 0;
  __syncthreads();
  mx = red[0];
#pragma unroll
  for (int i = 1; i < 8; ++i) mx = max(mx, red[i]);
  const int ew = max((int)(mx >> 23), 1);
  int nc = 0;   // corrections so far (block-uniform)
  for (int k0 = 0; k0 < d; k0 += 1024) {
    const int kq = k0 + 4 * tid;   // this thread's 4 consecutive k
    const bool act = kq < d;
    uint32_t dig[LW] = {0u, 0u, 0u, 0u, 0u};
    double dw[4];
    int has[4] = {0, 0, 0, 0};
    if (act) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t u = __ldg(wu + (int64_t)(kq + q) * NE + e);
        const uint32_t mag = u & 0x7FFFFFFFu;
        const int e8 = (int)(mag >> 23);
        const uint32_t M = (mag & 0x7FFFFFu) | (e8 ? 0x800000u : 0u);
        const int ee = max(e8, 1);
        const int sh = ee - ew + WSH;
        uint64_t Wi;
        uint32_t res = 0;
        if (sh >= 0) {
          Wi = (uint64_t)M << sh;
        } else {
          const int r = min(-sh, 25);
          Wi = r >= 25 ? 0 : (uint64_t)(M >> r);
          res = M - (uint32_t)(Wi << r);
        }
        has[q] = res != 0u;
        // w - w~ = sign * res * 2^(ee - 150): exact in f64
        dw[q] = ((u >> 31) ? -1.0 : 1.0) * (double)res * pow2(ee - 150);
        if (B256) {   // two's complement, byte j from the top (byte 0 signed)
          const int64_t Ws = (u >> 31) ? -(int64_t)Wi : (int64_t)Wi;
#pragma unroll
          for (int j = 0; j < LW; ++j) dig[j] |= ((uint32_t)(Ws >> (8 * (LW - 1 - j))) & 0xFFu) << (8 * q);
        } else {      // sign-magnitude 7-bit digits
#pragma unroll
          for (int j = 0; j < LW; ++j) {
            uint32_t dj = (uint32_t)(Wi >> (7 * (LW - 1 - j))) & 0x7Fu;
            if (u >> 31) dj = (0x80u - dj) ^ 0x80u;
            dig[j] |= (dj & 0xFFu) << (8 * q);
          }
        }
      }
      const int kb = kq / KB, kin = kq % KB;
      const int off = swz_off(e, kin >> 4) | (kin & 15);
#pragma unroll
      for (int j = 0; j < LW; ++j)
        *reinterpret_cast<uint32_t*>(ws.wimg + (size_t)kb * W_STAGE + j * W_SLICE + off) = dig[j];
    }
    // block-ordered compaction of the corrections (k ascending)
    const int cnt = has[0] + has[1] + has[2] + has[3];
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int before = nc, total = nc;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      if (w < warp) before += wsum[w];
      total += wsum[w];
    }
    int pos = before + incl - cnt;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (has[q]) {
        if (pos < CORR_MAX) {
          ws.ck[e * CORR_MAX + pos] = kq + q;
          ws.cdw[e * CORR_MAX + pos] = dw[q];
        }
        ++pos;
      }
    }
    nc = total;
    __syncthreads();   // wsum reuse
  }
  if (tid == 0) {
    ws.ew[e] = ew;
    ws.ccnt[e] = min(nc, CORR_MAX);
    // inf / nan in the column, or too many corrections: f64 path for every token
    ws.bflag[e] = (mx >= 0x7F800000u || nc > CORR_MAX) ? 1 : 0;
  }
}

// ------------------------------------------------------------------ scores
// One CTA per 128 tokens. Warps 0-15 convert x to digit planes (2 jobs of 16
// elements per thread per stage) and run the epilogue; warp 16 issues the
// MMAs; warp 17 bulk-copies the W digit planes.
//
// The row scale is guessed from the row's first 128 elements (two binades of
// headroom above their max): any element outside the 21-binade window [emax-20,
// emax] -- and any zero-exponent or non-finite one -- is left out of the
// integer sum and added back exactly in f64 from a short per-row list.
__global__ void __launch_bounds__(THREADS, 1)
router_scores_i8_kernel(const bf16* __restrict__ x, const float* __restrict__ w_r, int tpc,
                        const double* __restrict__ part, Ws ws, float* __restrict__ logits,
                        float* __restrict__ scores_bes, int B, int S, int d) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ctrl = sm + BUF;
  uint64_t* full = reinterpret_cast<uint64_t*>(ctrl);
  uint64_t* empty = full + NSTAGE;
  uint64_t* tfull = empty + NSTAGE;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ctrl + 64);
  int* emax_s = reinterpret_cast<int*>(ctrl + C_EMAX);
  int* rflag_s = reinterpret_cast<int*>(ctrl + C_RFLAG);
  int* xcn = reinterpret_cast<int*>(ctrl + C_XCN);
  int* xck = reinterpret_cast<int*>(ctrl + C_XCK);
  float* xcv = reinterpret_cast<float*>(ctrl + C_XCV);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t T = (int64_t)B * S;
  // tpc <= BM tokens per CTA (the MMA tile stays M = 128; rows past tpc are
  // zero digits): sized on the host so the grid fills whole waves of SMs
  const int64_t t0 = (int64_t)blockIdx.x * tpc;
  const int rows = (int)(T - t0 < tpc ? T - t0 : tpc);
  const int nkb = d / KB;
  pdl_trigger();
  const bool trace = NIMG_I8_TRACE && (blockIdx.x == 0 || blockIdx.x == 64);
  __shared__ uint64_t trs[48];   // trace: 0 start, 1 W past pdl, 2+kb full[kb] (kb < 32), 40.. epilogue
  if (trace && tid == 0) trs[0] = gtimer();

  if (tid == 0) {
    for (int s = 0; s < NSTAGE; ++s) { mbar_init(&full[s], NCONV + 1); mbar_init(&empty[s], 1); }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (tid < BM) { rflag_s[tid] = 0; xcn[tid] = 0; }
  if (warp == NCONV / 32) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp < NCONV / 32) {
    // ---------------------------------------------- converters
    // job = tid + 512 jj: tile row job / CPR, 16-element chunk job % CPR of the stage
    const bf16* src[JOBS];
    bool rv[JOBS];
#pragma unroll
    for (int jj = 0; jj < JOBS; ++jj) {
      const int job = tid + NCONV * jj, r = job / CPR, c = job % CPR;
      rv[jj] = r < rows;
      src[jj] = x + (t0 + (rv[jj] ? r : 0)) * d + c * 16;
    }
    // x ring in registers: stage kb sits in xr[kb % (XPF + 1)]
    uint4 xr[XPF + 1][2 * JOBS];
    auto load = [&](int kb, uint4 (&buf)[2 * JOBS]) {
#pragma unroll
      for (int jj = 0; jj < JOBS; ++jj) {
        if (rv[jj]) {
          const uint4* p = reinterpret_cast<const uint4*>(src[jj] + kb * KB);
          buf[2 * jj] = __ldg(p);
          buf[2 * jj + 1] = __ldg(p + 1);
        } else {
          buf[2 * jj] = buf[2 * jj + 1] = make_uint4(0u, 0u, 0u, 0u);
        }
      }
    };
#pragma unroll
    for (int i = 0; i < XPF; ++i)
      if (i < nkb) load(i, xr[i]);
    // row scale guess from the first stage: the CPR lanes of a row share it
    int base[JOBS];
    uint32_t lo7[JOBS], hi7[JOBS];
    float xscale[JOBS];   // 2^(134 + XW - e_t): x -> X on the fast path
    bool sok[JOBS];       // the scale is a normal float (else: integer path)
#pragma unroll
    for (int jj = 0; jj < JOBS; ++jj) {
      const uint4 a = xr[0][2 * jj], b = xr[0][2 * jj + 1];
      uint32_t m = __vmaxu2(__vmaxu2(__vmaxu2(a.x & 0x7FFF7FFFu, a.y & 0x7FFF7FFFu),
                                     __vmaxu2(a.z & 0x7FFF7FFFu, a.w & 0x7FFF7FFFu)),
                            __vmaxu2(__vmaxu2(b.x & 0x7FFF7FFFu, b.y & 0x7FFF7FFFu),
                                     __vmaxu2(b.z & 0x7FFF7FFFu, b.w & 0x7FFF7FFFu)));
      m = max(m & 0xFFFFu, m >> 16);
#pragma unroll
      for (int o = 1; o < CPR; o <<= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
      const int eg = min(max((int)(m >> 7), 1), 254) + XH;
      base[jj] = XW - eg;
      sok[jj] = NIMG_I8_FCONV && eg >= XW + 8 && eg <= XW + 260;
      xscale[jj] = __uint_as_float((uint32_t)(sok[jj] ? 261 + XW - eg : 127) << 23);
      lo7[jj] = (uint32_t)max(eg - XW, 1) << 7;
      hi7[jj] = (uint32_t)min(eg, 254) << 7;
      if ((tid % CPR) == 0) emax_s[(tid + NCONV * jj) / CPR] = eg;
    }
    int stage = 0;
    uint32_t phase = 0;
    // one stage: convert x stage kb (registers `cur`) into the smem digit planes
    auto convert = [&](int kb, const uint4 (&cur)[2 * JOBS]) {
      mbar_wait(&empty[stage], phase ^ 1);
      uint8_t* sa = sm + (size_t)stage * STAGE;
#pragma unroll
      for (int jj = 0; jj < (NIMG_I8_PROBE == 1 ? 0 : JOBS); ++jj) {
        const int job = tid + NCONV * jj, r = job / CPR, c = job % CPR;
        const uint32_t wv[8] = {cur[2 * jj].x,     cur[2 * jj].y,     cur[2 * jj].z,     cur[2 * jj].w,
                                cur[2 * jj + 1].x, cur[2 * jj + 1].y, cur[2 * jj + 1].z, cur[2 * jj + 1].w};
        // all 16 exponents inside [elo, ehi] (no zero / subnormal / inf / nan):
        // the branch-free path; otherwise element by element
        uint32_t mn = 0xFFFFFFFFu, mxe = 0u;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          mn = __vminu2(mn, wv[i] & 0x7F807F80u);
          mxe = __vmaxu2(mxe, wv[i] & 0x7F807F80u);
        }
        const bool fast = min(mn & 0xFFFFu, mn >> 16) >= lo7[jj] && max(mxe & 0xFFFFu, mxe >> 16) <= hi7[jj];
        uint32_t out[LX][4];
        if (B256 && fast && sok[jj]) {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            uint32_t th[4], tl[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint32_t w = wv[2 * g + (q >> 1)];
              const float xv = __uint_as_float((q & 1) ? (w & 0xFFFF0000u) : (w << 16));
              digits_b256(xv, xscale[jj], th[q], tl[q]);
            }
            // LX = 4: bytes 1 / 0 of th are digits 3 (top, signed) / 2; LX = 3:
            // byte 0 of th is digit 2 (top, signed). Bytes 1 / 0 of tl: digits 1 / 0.
            const uint32_t h01 = __byte_perm(th[0], th[1], 0x5140), h23 = __byte_perm(th[2], th[3], 0x5140);
            const uint32_t l01 = __byte_perm(tl[0], tl[1], 0x5140), l23 = __byte_perm(tl[2], tl[3], 0x5140);
            if (LX == 4) out[0][g] = __byte_perm(h01, h23, 0x7632);
            out[LX - 3][g] = __byte_perm(h01, h23, 0x5410);
            out[LX - 2][g] = __byte_perm(l01, l23, 0x7632);
            out[LX - 1][g] = __byte_perm(l01, l23, 0x5410);
          }
        } else if (!B256 && fast && sok[jj]) {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            uint32_t tb[4][LX];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint32_t w = wv[2 * g + (q >> 1)];
              const float xv = __uint_as_float((q & 1) ? (w & 0xFFFF0000u) : (w << 16));
              digits_fma<LX>(xv, xscale[jj], tb[q]);
            }
#pragma unroll
            for (int i = 0; i < LX; ++i)   // plane i: byte 0 of the four elements' digit i
              out[i][g] = __byte_perm(__byte_perm(tb[0][i], tb[1][i], 0x0040),
                                      __byte_perm(tb[2][i], tb[3][i], 0x0040), 0x5410);
          }
        } else {
        uint32_t Y[16];
        if (fast) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t w = wv[i];
            const int ml = (int)(w << 16) >> 31, mh = (int)w >> 31;
            const uint32_t sl = ((((w & 0x7Fu) | 0x80u) ^ (uint32_t)ml) - (uint32_t)ml);
            const uint32_t shv = ((((w >> 16) & 0x7Fu) | 0x80u) ^ (uint32_t)mh) - (uint32_t)mh;
            Y[2 * i] = spread_digits(sl << (((w >> 7) & 0xFFu) + base[jj]));
            Y[2 * i + 1] = spread_digits(shv << (((w >> 23) & 0xFFu) + base[jj]));
          }
        } else {
#pragma unroll
          for (int el = 0; el < 16; ++el) {
            const uint32_t u = (wv[el >> 1] >> (16 * (el & 1))) & 0xFFFFu;
            const int e8 = (int)((u >> 7) & 0xFFu);
            const int sh = e8 + base[jj];
            if (((unsigned)sh > (unsigned)XW) | ((unsigned)(e8 - 1) > 253u)) {
              Y[el] = 0u;
              if (u & 0x7FFFu) {   // exact f64 term in the epilogue
                const int slot = atomicAdd(&xcn[r], 1);
                if (slot < XC_MAX) {
                  xck[r * XC_MAX + slot] = kb * KB + c * 16 + el;
                  xcv[r * XC_MAX + slot] = __uint_as_float(u << 16);
                }
              }
            } else {
              const uint32_t m = (u & 0x8000u) ? 0xFFFFFFFFu : 0u;
              Y[el] = spread_digits(((((u & 0x7Fu) | 0x80u) ^ m) - m) << sh);
            }
          }
        }
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          // 4x4 byte transpose: out[i] = digit i of elements 4g..4g+3 (byte 3 - i)
          const uint32_t a0 = __byte_perm(Y[4 * g], Y[4 * g + 1], 0x5140);
          const uint32_t a1 = __byte_perm(Y[4 * g + 2], Y[4 * g + 3], 0x5140);
          const uint32_t a2 = __byte_perm(Y[4 * g], Y[4 * g + 1], 0x7362);
          const uint32_t a3 = __byte_perm(Y[4 * g + 2], Y[4 * g + 3], 0x7362);
          out[LX - 1][g] = __byte_perm(a0, a1, 0x5410);
          out[LX - 2][g] = __byte_perm(a0, a1, 0x7632);
          out[LX - 3][g] = __byte_perm(a2, a3, 0x5410);
          if (LX == 4) out[0][g] = __byte_perm(a2, a3, 0x7632);
        }
        }
        const int off = swz_off(r, c);
#pragma unroll
        for (int i = 0; i < LX; ++i)
          *reinterpret_cast<uint4*>(sa + i * A_SLICE + off) =
              make_uint4(out[i][0], out[i][1], out[i][2], out[i][3]);
      }
      fence_proxy_async_smem();
      mbar_arrive(&full[stage]);
      if (++stage == NSTAGE) { stage = 0; phase ^= 1; }
    };
    // the loop is unrolled by the ring length so every ring index is static
    // (registers, not local memory)
    for (int kb0 = 0; kb0 < nkb; kb0 += XPF + 1) {
#pragma unroll
      for (int u = 0; u <= XPF; ++u) {
        const int kb = kb0 + u;
        if (kb < nkb) {
          if (kb + XPF < nkb) load(kb + XPF, xr[(u + XPF) % (XPF + 1)]);
          convert(kb, xr[u]);
        }
      }
    }

    // ---------------------------------------------- epilogue
    mbar_wait(tfull, 0);
    if constexpr (NIMG_I8_PROBE != 3) {   // (timing probe 3: no epilogue)
    tc_fence_after();
    if (trace && tid == 0) trs[40] = gtimer();
    pdl_wait();   // prep outputs (t-bias partials, scales, corrections)
    if (trace && tid == 0) trs[41] = gtimer();
    const int64_t b_first = t0 / S;
    const int nb = (int)((t0 + rows - 1) / S - b_first + 1);
    double* tbs = reinterpret_cast<double*>(sm + TBS_OFF);
    float* lgs = reinterpret_cast<float*>(sm + LG_OFF);
    double* exs = reinterpret_cast<double*>(sm + EX_OFF);
    int* wck = reinterpret_cast<int*>(sm + WC_OFF);
    double* wcd = reinterpret_cast<double*>(sm + WC_OFF + NE * CORR_SM * 4);
    int* wcn = reinterpret_cast<int*>(sm + WC_OFF + NE * CORR_SM * 12);
    int* wew = wcn + NE;
    for (int i = tid; i < nb * NE; i += NCONV) tbs[i] = router_tbias(part, b_first + i / NE, i % NE, d, NE);
    for (int i = tid; i < NE * CORR_SM; i += NCONV) {
      const int ee = i / CORR_SM, c = i % CORR_SM;
      if (c < __ldg(ws.ccnt + ee)) {
        wck[i] = __ldg(ws.ck + ee * CORR_MAX + c);
        wcd[i] = __ldg(ws.cdw + ee * CORR_MAX + c);
      }
    }
    if (tid < NE) { wcn[tid] = __ldg(ws.ccnt + tid); wew[tid] = __ldg(ws.ew + tid); }
    bar_conv();
    if (trace && tid == 0) trs[43] = gtimer();

    const int q = warp & 3, p = warp >> 2;   // TMEM lane quadrant, 16-expert quarter
    const int r = q * 32 + lane;
    const bool valid = r < rows;
    const int64_t t = t0 + (valid ? r : 0);
    const int b = (int)t / S, srow = (int)t - b * S;   // T < 2^31 (capi check)
    const double* tbr = tbs + (b - b_first) * NE;
    const int er = emax_s[r];
    const int nx = xcn[r];
    const int nxu = min(nx, XC_MAX);
    const bf16* xrow = x + t * d;
    uint32_t fl = nx > XC_MAX;
    float pm = -INFINITY;   // max of this thread's 16 logits (NaN ignored, as fmax)
    float* pmx = reinterpret_cast<float*>(sm + PM_OFF);
    const uint32_t tl = tmem_base + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
    for (int ec = 0; ec < 4; ++ec) {
      const int e0 = p * 16 + ec * 4;
      uint32_t g[NG][4];
#pragma unroll
      for (int s = 0; s < NG; ++s) tmem_ld4(tl + s * NE + e0, g[s]);
      tmem_ld_wait();
      // the four logits of this column quad side by side (independent chains)
      double v4[4], cs4[4], ca4[4], hl4[4];
      int ncs4[4], cmax = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int e = e0 + j;
        // v = sum_s G_s base^(NG-1-s) = H 2^(4 DB) + L, H and L exact in int64
        int64_t H = 0, L = 0;
#pragma unroll
        for (int s = 0; s < NG - 4; ++s) H = H * (1 << DB) + (int64_t)(int)g[s][j];
#pragma unroll
        for (int s = NG - 4; s < NG; ++s) L = L * (1 << DB) + (int64_t)(int)g[s][j];
        // base 256: H and L may exceed 2^53 (d > 2048), so their conversions
        // are inexact in general; hl4 bounds those roundings for the proof
        const double Hd = (double)H, Ld = (double)L;
        v4[j] = fma(Hd, B256 ? 4294967296.0 : 268435456.0, Ld);
        hl4[j] = B256 ? fabs(Hd) * 4294967296.0 + fabs(Ld) : 0.0;
        const double sc = pow2(er + wew[e] - 134 - WEXP - XW);
        v4[j] *= sc;
        hl4[j] *= sc;
        cs4[j] = 0.0;
        ca4[j] = 0.0;
        ncs4[j] = wcn[e];
        cmax = max(cmax, ncs4[j]);
      }
      // W corrections x~ * (w - w~) (x~ = 0 for the row's listed elements): the
      // four logits' x loads are issued together, then consumed
      for (int c = 0; c < cmax; ++c) {
        uint32_t u4[4];
        double dw4[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          u4[j] = 0u;
          dw4[j] = 0.0;
          if (c < ncs4[j]) {
            const int e = e0 + j;
            const bool in_sm = c < CORR_SM;
            const int kc = in_sm ? wck[e * CORR_SM + c] : __ldg(ws.ck + e * CORR_MAX + c);
            dw4[j] = in_sm ? wcd[e * CORR_SM + c] : __ldg(ws.cdw + e * CORR_MAX + c);
            u4[j] = __bfloat16_as_ushort(xrow[kc]);
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (c < ncs4[j]) {
            const uint32_t u = u4[j];
            const int e8 = (int)((u >> 7) & 0xFFu), sh = e8 + XW - er;
            const bool special = ((unsigned)sh > (unsigned)XW) | ((unsigned)(e8 - 1) > 253u);
            const double pr = special ? 0.0 : (double)__uint_as_float(u << 16) * dw4[j];
            cs4[j] += pr;
            ca4[j] += fabs(pr);
          }
        }
      }
      // (x - x~) * w for the row's listed x elements: the four logits' W values
      // are one 16-B load per element, all of them in flight at once
      double xs4[4] = {0.0, 0.0, 0.0, 0.0}, xa4[4] = {0.0, 0.0, 0.0, 0.0};
      if (nxu > 0) {
        float4 wl[XC_MAX];
#pragma unroll
        for (int c = 0; c < XC_MAX; ++c)
          if (c < nxu) wl[c] = __ldg(reinterpret_cast<const float4*>(w_r + (int64_t)xck[r * XC_MAX + c] * NE + e0));
#pragma unroll
        for (int c = 0; c < XC_MAX; ++c) {
          if (c < nxu) {
            const double xv = (double)xcv[r * XC_MAX + c];
            const double pr[4] = {xv * (double)wl[c].x, xv * (double)wl[c].y, xv * (double)wl[c].z,
                                  xv * (double)wl[c].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              xs4[j] += pr[j];
              xa4[j] += fabs(pr[j]);
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int e = e0 + j;
        const double v = v4[j];
        double cs = cs4[j], ca = ca4[j];
        const int ncw = wcn[e];
        cs += xs4[j];   // (x - x~) * w for the listed elements (below)
        ca += xa4[j];
        const double z = (v + cs) + tbr[e];
        // rounding of v (and of its halves' conversions), of the correction sums
        // and of the two adds
        const double bound = (2.0 * fabs(v) + hl4[j] + (ncw + nxu + 2) * ca + fabs(z)) * 0x1p-52;
        const float rf = __double2float_rn(z);
        // rf is the rounding of every value within `bound` of z iff that band
        // stays strictly inside rf's rounding interval [|rf| - hd, |rf| + hu]
        // (half the spacing above / below; below is halved at a power of two)
        const uint32_t fb = __float_as_uint(rf) & 0x7FFFFFFFu;
        const int ex = (int)(fb >> 23);
        const double hu = pow2(max(ex, 1) - 151);
        const double hd = ((fb & 0x7FFFFFu) == 0u && ex > 1) ? 0.5 * hu : hu;
        const double dd = fabs(z) - (double)__uint_as_float(fb);
        fl |= (ex == 255) | (fb == 0u) | !((dd - bound > -hd) && (dd + bound < hu));
        lgs[r * LGS + e] = rf;
        pm = fmaxf(pm, rf);
      }
    }
    if (trace && tid == 0) trs[45] = gtimer();
    if (fl && valid) atomicOr(&rflag_s[r], 1);
    pmx[r * 4 + p] = pm;
    bar_conv();
    if (trace && tid == 0) trs[42] = gtimer();
    // numpy-order softmax over the 64 experts (tensor.py:467-479): the four
    // threads of a row compute the same max and sum; each writes its 16
    const double mxv = (double)fmaxf(fmaxf(pmx[r * 4], pmx[r * 4 + 1]), fmaxf(pmx[r * 4 + 2], pmx[r * 4 + 3]));
#pragma unroll 4
    for (int e = p * 16; e < p * 16 + 16; ++e) exs[r * LGS + e] = exp((double)lgs[r * LGS + e] - mxv);
    bar_conv();
    double acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = exs[r * LGS + j];
#pragma unroll
    for (int i = 8; i < NE; i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += exs[r * LGS + i + j];
    const double sum = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    if (valid) {
#pragma unroll 4
      for (int e = p * 16; e < p * 16 + 16; ++e)
        scores_bes[((int64_t)b * NE + e) * S + srow] = (float)(exs[r * LGS + e] / sum);
      const float* lr = lgs + r * LGS + p * 16;
#pragma unroll
      for (int i = 0; i < 2; ++i)   // 64 B of this row's logits: two whole sectors
        st_global_32(logits + t * NE + p * 16 + 8 * i,
                     make_uint4(__float_as_uint(lr[8 * i]), __float_as_uint(lr[8 * i + 1]),
                                __float_as_uint(lr[8 * i + 2]), __float_as_uint(lr[8 * i + 3])),
                     make_uint4(__float_as_uint(lr[8 * i + 4]), __float_as_uint(lr[8 * i + 5]),
                                __float_as_uint(lr[8 * i + 6]), __float_as_uint(lr[8 * i + 7])));
      if (p == 0 && rflag_s[r]) ws.list[atomicAdd(ws.counter, 1u)] = (int)t;
    }
    if (trace && tid == 0) trs[44] = gtimer();
    }
  } else if (warp == NCONV / 32) {
    // ---------------------------------------------- MMA issuer
    if (lane == 0) {
      // x digit i times [W_0 | W_1 | W_2 | W_3] (N = 256, the slices are
      // contiguous rows of the stage) lands on the contiguous TMEM groups
      // i..i+3; W_4 (N = 64) on group i+4.
      constexpr uint32_t idesc256 = make_idesc_s8(BM, 4 * NE);
      constexpr uint32_t idesc64 = make_idesc_s8(BM, NE);
      // base 256: A is signed for the top x digit only, B for W_0 only; idesc
      // bit 7 / 10 = A / B signed
      constexpr uint32_t kASigned = 1u << 7, kBSigned = 1u << 10;
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&full[stage], phase);
        if (trace && kb < 38) trs[2 + kb] = gtimer();
        tc_fence_after();
        const uint32_t sa = smem_u32(sm + (size_t)stage * STAGE);
        const uint32_t sw = sa + LX * A_SLICE;
        const uint64_t b03 = sdesc_k(sw);
        const uint64_t b4 = sdesc_k(sw + 4 * W_SLICE);
        const uint64_t b0 = b03, b14 = sdesc_k(sw + W_SLICE);
#pragma unroll
        for (int kk = 0; kk < KB / 32; ++kk) {
          const bool first = kb == 0 && kk == 0;
          if constexpr (B256) {
            // x digit i times W_0 (N = 64, signed B) lands on TMEM group i and
            // times [W_1 | W_2 | W_3 | W_4] (N = 256, unsigned B) on groups
            // i+1..i+4. Digits run top-down from i = 3 so that, in the first K
            // step, every MMA either starts all its groups or accumulates onto
            // groups already started.
#pragma unroll
            for (int i = LX - 1; i >= 0; --i) {
              const uint64_t adesc = sdesc_k(sa + i * A_SLICE) + 2 * kk;
              const uint32_t as = i == 0 ? kASigned : 0u;
              if (NIMG_I8_PROBE != 2) {
                umma_i8(tmem_base + i * NE, adesc, b0 + 2 * kk, (idesc64 & ~(kASigned | kBSigned)) | as | kBSigned,
                        first ? 0u : 1u);
                umma_i8(tmem_base + (i + 1) * NE, adesc, b14 + 2 * kk, (idesc256 & ~(kASigned | kBSigned)) | as,
                        (first && i == LX - 1) ? 0u : 1u);
              }
            }
          } else {
#pragma unroll
          for (int i = 0; i < LX; ++i) {
            const uint64_t adesc = sdesc_k(sa + i * A_SLICE) + 2 * kk;
            if (NIMG_I8_PROBE != 2) {
              umma_i8(tmem_base + i * NE, adesc, b03 + 2 * kk, idesc256, (first && i == 0) ? 0u : 1u);
              umma_i8(tmem_base + (i + 4) * NE, adesc, b4 + 2 * kk, idesc64, first ? 0u : 1u);
            }
          }
          }
        }
        umma_commit(&empty[stage]);
        if (++stage == NSTAGE) { stage = 0; phase ^= 1; }
      }
      umma_commit(tfull);
    }
  } else {
    // ---------------------------------------------- W digit producer
    if (lane == 0) {
      pdl_wait();   // the prep kernel wrote the digit image
      if (trace) trs[1] = gtimer();
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], W_STAGE);
        bulk_load(sm + (size_t)stage * STAGE + LX * A_SLICE, ws.wimg + (size_t)kb * W_STAGE, W_STAGE,
                  &full[stage]);
        if (++stage == NSTAGE) { stage = 0; phase ^= 1; }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == NCONV / 32) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
  if (trace && tid == 0) {
    const double t0s = (double)trs[0];
    printf("ri8 cta %d (us): Wpdl %.1f | full kb0 %.1f kb1 %.1f kb2 %.1f kb3 %.1f kb8 %.1f kb16 %.1f kb24 %.1f kbL %.1f | "
           "tfull %.1f pdl %.1f setup %.1f thr0 %.1f logits %.1f end %.1f\n", (int)blockIdx.x, (trs[1] - t0s) * 1e-3,
           (trs[2] - t0s) * 1e-3, (trs[3] - t0s) * 1e-3, (trs[4] - t0s) * 1e-3, (trs[5] - t0s) * 1e-3,
           (trs[10] - t0s) * 1e-3, (trs[18] - t0s) * 1e-3, (trs[26] - t0s) * 1e-3,
           (trs[1 + nkb] - t0s) * 1e-3, (trs[40] - t0s) * 1e-3, (trs[41] - t0s) * 1e-3,
           (trs[43] - t0s) * 1e-3, (trs[45] - t0s) * 1e-3,
           (trs[42] - t0s) * 1e-3, (trs[44] - t0s) * 1e-3);
  }
}

// ------------------------------------------------------------------ fix-up
// Flagged tokens (or all of them when W_r could not be written in fixed
// point): the f64 dot, the t-bias, fp32 rounding and the softmax again.
// Warp w sums the k-slice [w d/16, (w+1) d/16) for experts 2 lane, 2 lane + 1;
// the 16 slice sums are folded in a fixed order.
constexpr int FIX_THREADS = 512;
__global__ void __launch_bounds__(FIX_THREADS)
router_fix_i8_kernel(const bf16* __restrict__ x, const float* __restrict__ w_r,
                     const double* __restrict__ part, Ws ws, float* __restrict__ logits,
                     float* __restrict__ scores_bes, int B, int S, int d) {
  pdl_trigger();
  pdl_wait();
  __shared__ double red[FIX_THREADS / 32][NE];
  __shared__ double ex[NE];
  __shared__ float lg[NE];
  __shared__ double tot;
  int all = 0;
  for (int i = 0; i < NE; ++i) all |= ws.bflag[i];
  const int64_t T = (int64_t)B * S;
  const int64_t n = all ? T : (int64_t)*ws.counter;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NW = FIX_THREADS / 32;
  const int klen = d / NW, k0 = warp * klen;
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const int64_t t = all ? i : (int64_t)ws.list[i];
    const int64_t b = t / S, srow = t % S;
    const bf16* xr = x + t * d;
    double a0 = 0.0, a1 = 0.0;
#pragma unroll 8
    for (int k = k0; k < k0 + klen; ++k) {
      const double xv = (double)__bfloat162float(xr[k]);
      const float2 w2 = __ldg(reinterpret_cast<const float2*>(w_r + (int64_t)k * NE) + lane);
      a0 = fma(xv, (double)w2.x, a0);
      a1 = fma(xv, (double)w2.y, a1);
    }
    red[warp][2 * lane] = a0;
    red[warp][2 * lane + 1] = a1;
    __syncthreads();
    if (threadIdx.x < NE) {
      const int e = threadIdx.x;
      double z = red[0][e];
      for (int w = 1; w < NW; ++w) z += red[w][e];
      lg[e] = (float)(z + router_tbias(part, b, e, d, NE));
    }
    __syncthreads();
    if (threadIdx.x < NE) {
      const int e = threadIdx.x;
      double mxv = -INFINITY;
      for (int j = 0; j < NE; ++j) mxv = fmax(mxv, (double)lg[j]);
      ex[e] = exp((double)lg[e] - mxv);
    }
    __syncthreads();
    if (threadIdx.x == 0) tot = np_pairwise_sum(ex, NE);
    __syncthreads();
    if (threadIdx.x < NE) {
      const int e = threadIdx.x;
      logits[t * NE + e] = lg[e];
      scores_bes[(b * NE + e) * S + srow] = (float)(ex[e] / tot);
    }
    __syncthreads();
  }
}

}  // namespace ri8

bool router_i8_eligible(bool x_bf16, int d, int E, const void* x_norm, const void* w_r) {
  // read per call (a getenv is ~100 ns) so tests can compare both routers in one process
  const char* v = getenv("NIMG_ROUTER");
  if (v && (!strcmp(v, "dmma") || !strcmp(v, "f64"))) return false;
  // int32 group sums: <= 4 digit pairs x d x 255^2 < 2^31 for d <= 8192 (base 256)
  return x_bf16 && E == ri8::NE && d % ri8::KB == 0 && d <= (ri8::B256 ? 8192 : 32768) &&
         (uintptr_t)x_norm % 16 == 0 && (uintptr_t)w_r % 16 == 0;
}
size_t router_i8_ws_bytes(int64_t T, int d) { return ri8::ws_bytes(T, d); }

cudaError_t launch_router_i8(const void* x_norm, const float* t_emb, const float* w_r, double* part,
                             void* i8ws, float* logits, float* scores_bes, int B, int S, int d,
                             cudaStream_t s, ZeroSpans zs) {
  const int64_t T = (int64_t)B * S;
  ri8::Ws ws = ri8::carve(i8ws, T, d);
  // the first kernel of the chain: an ORDINARY launch (full stream order). The
  // scores kernel's converters read x_norm before any griddepcontrol.wait, so
  // everything that wrote x_norm (e.g. the block prologue) must have completed
  // before this kernel starts and triggers its dependents. (A PDL launch here
  // would let the scores kernel start while the prologue still writes x_norm.)
  ri8::router_prep_i8_kernel<<<B * router_tpart_ks(d) + ri8::NE, 256, 0, s>>>(t_emb, w_r, part, ws, B, d, zs);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return err;
  err = set_max_dyn_smem(ri8::router_scores_i8_kernel, (int)ri8::SMEM);
  if (err != cudaSuccess) return err;
  const bf16* x = reinterpret_cast<const bf16*>(x_norm);
  // tokens per CTA: 128 (the MMA tile). NIMG_I8_BALANCE=1 sizes CTAs to fill
  // whole waves of SMs instead (T = 16384: 147 CTAs of 112 tokens) -- measured
  // slower (78.6 vs 67.6 us in the launch list: every CTA still streams the
  // whole W digit image and runs the full M = 128 MMAs)
  int sms = 148;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  static const bool balance = [] {
    const char* v = getenv("NIMG_I8_BALANCE");
    return v && v[0] == '1';
  }();
  int tpc = ri8::BM;
  if (balance) {
    const int64_t waves = (T + (int64_t)sms * ri8::BM - 1) / ((int64_t)sms * ri8::BM);
    const int64_t per = (T + sms * waves - 1) / (sms * waves);
    tpc = (int)((per + 7) / 8 * 8);
    if (tpc > ri8::BM) tpc = ri8::BM;
    if (tpc < 8) tpc = 8;
  }
  err = launch_pdl(ri8::router_scores_i8_kernel, dim3((unsigned)((T + tpc - 1) / tpc)),
                   dim3(ri8::THREADS), ri8::SMEM, s, x, w_r, tpc, (const double*)part, ws, logits,
                   scores_bes, B, S, d);
  if (err != cudaSuccess) return err;
  static const bool stats = [] {   // debugging only (synchronises)
    const char* v = getenv("NIMG_ROUTER_I8_STATS");
    return v && v[0] == '1';
  }();
  static const bool nofix = [] {   // debugging only: leave flagged tokens as they are
    const char* v = getenv("NIMG_ROUTER_I8_NOFIX");
    return v && v[0] == '1';
  }();
  {
    if (stats) {
      unsigned cnt = 0;
      int bf[ri8::NE];
      cudaMemcpyAsync(&cnt, ws.counter, 4, cudaMemcpyDeviceToHost, s);
      cudaMemcpyAsync(bf, ws.bflag, sizeof(bf), cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      int all = 0;
      for (int i = 0; i < ri8::NE; ++i) all |= bf[i];
      fprintf(stderr, "[router_i8] T=%lld flagged=%u all_fallback=%d\n", (long long)T, cnt, all);
    }
  }
  if (nofix) return cudaSuccess;
  return launch_pdl(ri8::router_fix_i8_kernel, dim3(148), dim3(ri8::FIX_THREADS), 0, s, x, w_r, (const double*)part,
                    ws, logits, scores_bes, B, S, d);
}

}  // namespace nimg
