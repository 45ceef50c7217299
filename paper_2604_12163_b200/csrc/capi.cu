// C-ABI layer (include/nimg_moe.h): validation, workspace carving, TMA
// descriptor encoding and stream-ordered launch sequencing. No allocation and
// no host synchronisation happen here.
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include <cuda_bf16.h>

#include "../../include/nimg_moe.h"
#include "nimg_internal.h"

using namespace nimg;

namespace {

thread_local std::string g_err;
// Optional stage events (nimg_profile_events): recorded on the launch stream
// at the stage boundaries of nimg_moe_forward (0 start, 1 routed, 2 gathered,
// 3 GEMM1 done, 4 GEMM2 done, 5 combined; 6 router scores done). Null = off.
thread_local cudaEvent_t g_events[8];
thread_local int g_nevents = 0;
inline void mark(int i, cudaStream_t st) {
  if (i < g_nevents && g_events[i]) cudaEventRecord(g_events[i], st);
}

}  // namespace

cudaError_t nimg::set_max_dyn_smem(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;   // (kernel, device) -> bytes set
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  int& have = done[{kernel, dev}];
  if (have >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

namespace {

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                     \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      return fail(NIMG_ERR_CUDA, "%s failed: %s", #expr, cudaGetErrorString(_e));         \
  } while (0)

#define NIMG_TRY(expr)        \
  do {                        \
    int _r = (expr);          \
    if (_r != NIMG_OK) return _r; \
  } while (0)

constexpr size_t kAlign = 256;
inline size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }
inline size_t elt(int32_t dt) { return dt == NIMG_BF16 ? 2 : (dt == NIMG_F64 ? 8 : 4); }
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// ------------------------------------------------------------- tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// bf16 [rows, K] row-major, box (64 x box_rows), 128-B swizzle.
int map_2d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t K, uint32_t box_rows) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(NIMG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {K, rows};
  cuuint64_t strides[1] = {K * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(NIMG_ERR_CUDA, "tensor map 2d encode failed (%d)", (int)r);
  return NIMG_OK;
}
// bf16 [E, N, K] row-major, box (64 x box_rows x 1), 128-B swizzle.
int map_3d(CUtensorMap* m, const void* base, uint64_t E, uint64_t N, uint64_t K,
           uint32_t box_rows) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(NIMG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {K, N, E};
  cuuint64_t strides[2] = {K * 2, N * K * 2};
  cuuint32_t box[3] = {64, box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(NIMG_ERR_CUDA, "tensor map 3d encode failed (%d)", (int)r);
  return NIMG_OK;
}

// fp32 [E, M, N] row-major output (weight gradients), box (32 x 32 x 1),
// 128-B swizzle: the TMA-store target of the backward weight-gradient tiles.
int map_3d_f32_out(CUtensorMap* m, void* base, uint64_t E, uint64_t M, uint64_t N) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(NIMG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {N, M, E};
  cuuint64_t strides[2] = {N * 4, M * N * 4};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(NIMG_ERR_CUDA, "tensor map (f32 out) encode failed (%d)", (int)r);
  return NIMG_OK;
}

// SMs the persistent GEMMs size their grid by. NIMG_GEMM_MAX_SMS caps it
// (leaves SMs for concurrently running communication kernels).
int device_sms(int* out) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  static int cache[64] = {0};
  if (dev < 64 && cache[dev]) { *out = cache[dev]; return NIMG_OK; }
  int n = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  const char* cap = getenv("NIMG_GEMM_MAX_SMS");
  if (cap && atoi(cap) > 1 && atoi(cap) < n) n = atoi(cap) & ~1;
  if (dev < 64) cache[dev] = n;
  *out = n;
  return NIMG_OK;
}

// ------------------------------------------------------------- validation
int check_moe_desc(const nimg_moe_desc* d) {
  if (!d) return fail(NIMG_ERR_CONFIG, "null descriptor");
  if (d->act_dtype != NIMG_F32 && d->act_dtype != NIMG_BF16 && d->act_dtype != NIMG_F64)
    return fail(NIMG_ERR_CONFIG, "unsupported act_dtype %d", d->act_dtype);
  if (d->act_dtype == NIMG_F64 ? d->router_dtype != NIMG_F64
                               : (d->router_dtype != NIMG_F32 && d->router_dtype != NIMG_BF16))
    return fail(NIMG_ERR_CONFIG, "router_dtype %d incompatible with act_dtype %d", d->router_dtype,
                d->act_dtype);
  if (d->act_dtype == NIMG_F64 && !(d->gate_eps_f64 > 0.0))
    return fail(NIMG_ERR_CONFIG, "gate_eps must be > 0");
  if (d->B < 1 || d->S < 1 || d->d < 1 || d->h < 1 || d->h_shared < 1)
    return fail(NIMG_ERR_SHAPE, "empty dimension B=%lld S=%lld d=%lld h=%lld hs=%lld",
                (long long)d->B, (long long)d->S, (long long)d->d, (long long)d->h,
                (long long)d->h_shared);
  if (d->E < 1) return fail(NIMG_ERR_CONFIG, "n_experts must be >= 1");     // router.py:45-46
  if (!(d->gate_eps > 0.f)) return fail(NIMG_ERR_CONFIG, "gate_eps must be > 0");  // router.py:49-50
  if (d->cap < 1) return fail(NIMG_ERR_CONFIG, "computed capacity is zero");  // router.py:117-118
  if (d->cap > d->S) return fail(NIMG_ERR_CONFIG, "capacity %lld > S %lld", (long long)d->cap, (long long)d->S);
  if (d->E > 512) return fail(NIMG_ERR_CONFIG, "n_experts %lld > 512 unsupported", (long long)d->E);
  if (d->S > 16384) return fail(NIMG_ERR_CONFIG, "S %lld > 16384 unsupported", (long long)d->S);
  if (d->cap > 4096) return fail(NIMG_ERR_CONFIG, "capacity %lld > 4096 unsupported", (long long)d->cap);
  const int64_t T = d->B * d->S;
  if (d->E * d->B * d->cap >= (int64_t)1 << 31 || T * d->E >= (int64_t)1 << 31)
    return fail(NIMG_ERR_CONFIG, "problem too large for int32 row indices");
  return NIMG_OK;
}

// Route scratch: t-bias, DFMA-router partials / f64 W_r / counters, and the
// slot table slot_of (B, E, S) int16 (slot in the expert's column, -1 = not
// selected), written in full by ec_select.
struct RouteWs {
  double* tb;
  double* part;
  double* wd;
  int16_t* slot_of;
  unsigned* counters;
  void* i8;        // INT8 router scratch (router_i8.cu)
  int* bg_flags;   // GEMM1 background-gather flags, one per 32 routed rows
  // token-ordered expert outputs (1-GPU layer): GEMM2 writes routed row r to
  // row_map[r]; token t's rows are [tok_off[t], tok_off[t] + comb_cnt[t]) in
  // expert-ascending order, their gates gate_tok[..]; cursor: per sample
  int* tok_off;
  int* row_map;
  float* gate_tok;
  int* cursor;
  unsigned long long* tokmask;   // per-token selecting-expert masks (gates formed in the combine)
  int2* tokent;                  // [T][E] (routed row, raw score) of each selecting (token, e)
};
// one flag per 32 routed rows, plus the sub-block claim counter (flags[nsub])
int64_t bg_flag_count(const nimg_moe_desc* d) { return (d->E * d->B * d->cap + 31) / 32 + 1; }
size_t slot_bytes(const nimg_moe_desc* d) { return (size_t)d->E * d->B * d->S * 2; }
size_t route_ws_bytes(const nimg_moe_desc* d) {
  return align_up((size_t)d->B * d->E * 8) +
         align_up(router_part_bytes((int)d->B, (int)d->d, (int)d->E)) +
         align_up(router_wd_bytes((int)d->d, (int)d->E)) + align_up(slot_bytes(d)) +
         align_up((size_t)d->B * 4) + align_up(router_i8_ws_bytes(d->B * d->S, (int)d->d)) +
         align_up((size_t)bg_flag_count(d) * 4) + align_up((size_t)d->B * d->S * 4) +
         2 * align_up((size_t)d->E * d->B * d->cap * 4) + align_up((size_t)d->B * 4) +
         align_up((size_t)d->B * d->S * 8) + align_up((size_t)d->B * d->S * d->E * 8);
}
RouteWs carve_route(const nimg_moe_desc* d, void* ws) {
  uint8_t* p = static_cast<uint8_t*>(ws);
  RouteWs r;
  r.tb = reinterpret_cast<double*>(p);
  p += align_up((size_t)d->B * d->E * 8);
  r.part = reinterpret_cast<double*>(p);
  p += align_up(router_part_bytes((int)d->B, (int)d->d, (int)d->E));
  r.wd = reinterpret_cast<double*>(p);
  p += align_up(router_wd_bytes((int)d->d, (int)d->E));
  r.slot_of = reinterpret_cast<int16_t*>(p);
  p += align_up(slot_bytes(d));
  r.counters = reinterpret_cast<unsigned*>(p);
  p += align_up((size_t)d->B * 4);
  r.i8 = p;
  p += align_up(router_i8_ws_bytes(d->B * d->S, (int)d->d));
  r.bg_flags = reinterpret_cast<int*>(p);
  p += align_up((size_t)bg_flag_count(d) * 4);
  r.tok_off = reinterpret_cast<int*>(p);
  p += align_up((size_t)d->B * d->S * 4);
  r.row_map = reinterpret_cast<int*>(p);
  p += align_up((size_t)d->E * d->B * d->cap * 4);
  r.gate_tok = reinterpret_cast<float*>(p);
  p += align_up((size_t)d->E * d->B * d->cap * 4);
  r.cursor = reinterpret_cast<int*>(p);
  p += align_up((size_t)d->B * 4);
  r.tokmask = reinterpret_cast<unsigned long long*>(p);
  p += align_up((size_t)d->B * d->S * 8);
  r.tokent = reinterpret_cast<int2*>(p);
  return r;
}

bool use_pair_kernels();
bool use_tok_order();
// NIMG_GATES_IN_COMBINE=0: the 1-GPU forward keeps the separate gate kernel
static bool gates_in_combine() {
  static const bool on = [] {
    const char* e = getenv("NIMG_GATES_IN_COMBINE");
    return !(e && e[0] == '0');
  }();
  return on;
}
// fp32 mode on the bf16 tensor cores (split_kernels.cu, "bf16x3"): fp32
// layers whose widths tile the tcgen05 pair kernels; NIMG_FP32_TC=0 keeps the
// CUDA-core fp32 GEMMs
bool ffn_use_x3(const nimg_ffn_desc* f) {
  static const bool on = [] {
    const char* e = getenv("NIMG_FP32_TC");
    return !(e && e[0] == '0');
  }();
  if (!on || f->act_dtype != NIMG_F32 || !use_pair_kernels()) return false;
  if (f->d % 64 || f->h % 64) return false;
  if (f->n_shared_rows > 0 && f->h_shared % 64) return false;
  return true;
}
struct X3Ws {
  void *xr, *xs, *w1, *w3, *w2, *sw1, *sw3, *sw2, *pre_r, *pre_s;
  size_t bytes;
};
X3Ws x3_layout(const nimg_ffn_desc* f, void* base) {
  X3Ws w{};
  uint8_t* p = static_cast<uint8_t*>(base);
  size_t o = 0;
  auto take = [&](size_t elems) { void* q = p ? p + o : nullptr; o += align_up(elems * 2); return q; };
  const size_t d = f->d, h = f->h, hs = f->h_shared, E = f->n_experts;
  const size_t nr = f->n_rows, ns = f->n_shared_rows;
  w.xr = take(nr * 3 * d);
  w.xs = take(ns * 3 * d);
  w.w1 = take(nr ? E * h * 3 * d : 0);
  w.w3 = take(nr ? E * h * 3 * d : 0);
  w.w2 = take(nr ? E * d * 3 * h : 0);
  w.sw1 = take(ns ? hs * 3 * d : 0);
  w.sw3 = take(ns ? hs * 3 * d : 0);
  w.sw2 = take(ns ? d * 3 * hs : 0);
  w.pre_r = take(nr * 3 * h);
  w.pre_s = take(ns * 3 * hs);
  w.bytes = o;
  return w;
}

bool ffn_use_tc(const nimg_ffn_desc* f) {
  if (f->act_dtype != NIMG_BF16) return false;
  if (f->d % 16 || f->h % 16) return false;
  if (f->n_shared_rows > 0 && f->h_shared % 16) return false;
  return true;
}
size_t ffn_ws_bytes(const nimg_ffn_desc* f) {
  if (ffn_use_x3(f)) return x3_layout(f, nullptr).bytes;
  const size_t e = ffn_use_tc(f) ? 2 : (f->act_dtype == NIMG_F64 ? 8 : 4);
  return align_up((size_t)f->n_rows * f->h * e) + align_up((size_t)f->n_shared_rows * f->h_shared * e);
}

template <class P>
int fill_segments(P& p, const nimg_ffn_desc* f, const int64_t* off, const int32_t* ex, int bm,
                  int ntn0, int ntn1) {
  int64_t tiles = 0;
  int n = 0;
  for (int i = 0; i < f->nseg; ++i) {
    const int64_t rows = off[i + 1] - off[i];
    if (ex && ex[i] < 0) continue;   // skip segment: rows not computed, output untouched
    p.seg_row0[n] = (int)off[i];
    p.seg_rows[n] = (int)rows;
    p.seg_expert[n] = ex ? ex[i] : i;
    p.seg_tile0[n] = (int)tiles;
    tiles += (rows + bm - 1) / bm * ntn0;
    ++n;
  }
  p.nseg0 = n;
  if (f->n_shared_rows > 0) {
    p.seg_row0[n] = 0;
    p.seg_rows[n] = (int)f->n_shared_rows;
    p.seg_expert[n] = 0;
    p.seg_tile0[n] = (int)tiles;
    tiles += (f->n_shared_rows + bm - 1) / bm * ntn1;
    ++n;
  }
  p.nseg = n;
  p.seg_tile0[n] = (int)tiles;
  if (tiles >= ((int64_t)1 << 31)) return fail(NIMG_ERR_CONFIG, "too many tiles");
  p.total_tiles = (int)tiles;
  return NIMG_OK;
}

int check_ffn(const nimg_ffn_desc* f, const int64_t* off, const int32_t* ex) {
  if (!f) return fail(NIMG_ERR_CONFIG, "null descriptor");
  if (f->act_dtype != NIMG_F32 && f->act_dtype != NIMG_BF16 && f->act_dtype != NIMG_F64)
    return fail(NIMG_ERR_CONFIG, "unsupported act_dtype %d", f->act_dtype);
  if (f->nseg < 0 || f->nseg > kMaxSeg - 8)
    return fail(NIMG_ERR_CONFIG, "nseg %d outside [0, %d]", f->nseg, kMaxSeg - 8);
  if (f->d < 1 || f->h < 1 || (f->n_shared_rows > 0 && f->h_shared < 1))
    return fail(NIMG_ERR_SHAPE, "empty feature dimension");
  if (f->n_rows < 0 || f->n_shared_rows < 0 || f->n_rows >= ((int64_t)1 << 31) ||
      f->n_shared_rows >= ((int64_t)1 << 31))
    return fail(NIMG_ERR_SHAPE, "row count out of range");
  if (f->nseg > 0) {
    if (!off) return fail(NIMG_ERR_SHAPE, "null offsets");
    // GroupedBatch validation (moe.py:105-112)
    if (off[0] != 0) return fail(NIMG_ERR_SHAPE, "invalid offsets: offsets[0] != 0");
    for (int i = 0; i < f->nseg; ++i)
      if (off[i + 1] < off[i]) return fail(NIMG_ERR_SHAPE, "invalid offsets: decreasing at %d", i);
    if (off[f->nseg] != f->n_rows)
      return fail(NIMG_ERR_SHAPE, "offsets end %lld != token count %lld", (long long)off[f->nseg],
                  (long long)f->n_rows);
    for (int i = 0; i < f->nseg; ++i) {
      const int e = ex ? ex[i] : i;
      if (e < -1 || e >= f->n_experts) return fail(NIMG_ERR_SHAPE, "segment %d expert %d out of range", i, e);
    }
  } else if (f->n_rows != 0) {
    return fail(NIMG_ERR_SHAPE, "rows without segments");
  }
  return NIMG_OK;
}

// CTA-pair tcgen05 kernels (default); NIMG_PAIR=0 selects the 1-CTA kernels.
bool use_pair_kernels() {
  static const bool on = [] {
    const char* e = getenv("NIMG_PAIR");
    return !(e && e[0] == '0');
  }();
  return on;
}

// gather_idx != null (tcgen05 path only): routed row r of GEMM1's A operand is
// row gather_idx[r] of xr, which then has gather_src_rows rows (TMA gather4).
// Training forward: `pre` lands in caller buffers (kept for the weight
// gradient of GEMM2) and GEMM1 also stores h1 | h3 (the SwiGLU pullback's
// inputs); force_simt keeps the whole layer on the CUDA-core path (fp32
// intermediates) when the tcgen05 backward cannot take the shape.
struct FfnTrain {
  bool force_simt;
  void *pre_r, *pre_s, *h_r, *h_s;
};

// fp32 layer on the bf16 tcgen05 pair kernels: split operands (K' = 3K), GEMM1
// writes `pre` split, GEMM2 writes fp32 rows (split_kernels.cu).
int expert_ffn_x3(const nimg_ffn_desc* f, const int64_t* off, const int32_t* ex, const void* xr,
                  const void* w1, const void* w3, const void* w2, void* yr, const void* xs,
                  const void* sw1, const void* sw3, const void* sw2, void* ys, void* ws,
                  cudaStream_t st) {
  const X3Ws L = x3_layout(f, ws);
  const bool has_r = f->n_rows > 0, has_s = f->n_shared_rows > 0;
  const int d = (int)f->d, h = (int)f->h, hs = (int)(has_s ? f->h_shared : f->h);
  const int64_t E = f->n_experts;
  const float* F = nullptr;
  if (has_r) {
    CUDA_TRY(launch_split3_rows(static_cast<const float*>(xr), nullptr, L.xr, f->n_rows, d, 0, st));
    CUDA_TRY(launch_split3_rows(static_cast<const float*>(w1), nullptr, L.w1, E * h, d, 1, st));
    CUDA_TRY(launch_split3_rows(static_cast<const float*>(w3), nullptr, L.w3, E * h, d, 1, st));
    CUDA_TRY(launch_split3_rows(static_cast<const float*>(w2), nullptr, L.w2, E * d, h, 1, st));
  }
  if (has_s) {
    CUDA_TRY(launch_split3_rows(static_cast<const float*>(xs), nullptr, L.xs, f->n_shared_rows, d, 0, st));
    CUDA_TRY(launch_split3_rows(static_cast<const float*>(sw1), nullptr, L.sw1, hs, d, 1, st));
    CUDA_TRY(launch_split3_rows(static_cast<const float*>(sw3), nullptr, L.sw3, hs, d, 1, st));
    CUDA_TRY(launch_split3_rows(static_cast<const float*>(sw2), nullptr, L.sw2, d, hs, 1, st));
  }
  (void)F;
  int sms = 0;
  NIMG_TRY(device_sms(&sms));
  const int tile_rows = tc_pair_rows();
  const int rb = has_r ? 0 : 1;
  {  // GEMM1: pre' = split(SiLU(x' W1'^T) * (x' W3'^T)), K' = 3d
    GroupedParams p;
    memset(&p, 0, sizeof(p));
    const int bn = tc_bn_out(0), box = tc_b_box(0);
    NIMG_TRY(fill_segments(p, f, off, ex, tile_rows, (h + bn - 1) / bn, (hs + bn - 1) / bn));
    TmapSet tm;
    memset(&tm, 0, sizeof(tm));
    if (has_r) {
      NIMG_TRY(map_2d(&tm.a[0], L.xr, f->n_rows, 3 * (uint64_t)d, 128));
      NIMG_TRY(map_3d(&tm.b[0], L.w1, E, h, 3 * (uint64_t)d, box));
      NIMG_TRY(map_3d(&tm.b3[0], L.w3, E, h, 3 * (uint64_t)d, box));
    }
    if (has_s) {
      NIMG_TRY(map_2d(&tm.a[1], L.xs, f->n_shared_rows, 3 * (uint64_t)d, 128));
      NIMG_TRY(map_3d(&tm.b[1], L.sw1, 1, hs, 3 * (uint64_t)d, box));
      NIMG_TRY(map_3d(&tm.b3[1], L.sw3, 1, hs, 3 * (uint64_t)d, box));
    }
    if (!has_r) { tm.a[0] = tm.a[1]; tm.b[0] = tm.b[1]; tm.b3[0] = tm.b3[1]; }
    if (!has_s) { tm.a[1] = tm.a[rb]; tm.b[1] = tm.b[rb]; tm.b3[1] = tm.b3[rb]; }
    p.bank[0] = GBank{L.pre_r, 3 * h, 3 * d, h, (h + bn - 1) / bn, kSplit3Out, nullptr, nullptr, nullptr};
    p.bank[1] = GBank{L.pre_s, 3 * hs, 3 * d, hs, (hs + bn - 1) / bn, kSplit3Out, nullptr, nullptr, nullptr};
    CUDA_TRY(launch_grouped_tc_pair(0, tm, p, sms, st));
    mark(3, st);
  }
  {  // GEMM2: y = pre' W2'^T in fp32, K' = 3h
    GroupedParams p;
    memset(&p, 0, sizeof(p));
    const int bn = tc_bn_out(1), box = tc_b_box(1) / 2;
    NIMG_TRY(fill_segments(p, f, off, ex, tile_rows, (d + bn - 1) / bn, (d + bn - 1) / bn));
    TmapSet tm;
    memset(&tm, 0, sizeof(tm));
    if (has_r) {
      NIMG_TRY(map_2d(&tm.a[0], L.pre_r, f->n_rows, 3 * (uint64_t)h, 128));
      NIMG_TRY(map_3d(&tm.b[0], L.w2, E, d, 3 * (uint64_t)h, box));
    }
    if (has_s) {
      NIMG_TRY(map_2d(&tm.a[1], L.pre_s, f->n_shared_rows, 3 * (uint64_t)hs, 128));
      NIMG_TRY(map_3d(&tm.b[1], L.sw2, 1, d, 3 * (uint64_t)hs, box));
    }
    if (!has_r) { tm.a[0] = tm.a[1]; tm.b[0] = tm.b[1]; }
    if (!has_s) { tm.a[1] = tm.a[0]; tm.b[1] = tm.b[0]; }
    tm.b3[0] = tm.b[0];
    tm.b3[1] = tm.b[1];
    p.bank[0] = GBank{yr, d, 3 * h, d, (d + bn - 1) / bn, kF32Out, nullptr, nullptr, nullptr};
    p.bank[1] = GBank{ys, d, 3 * hs, d, (d + bn - 1) / bn, kF32Out, nullptr, nullptr, nullptr};
    CUDA_TRY(launch_grouped_tc_pair(1, tm, p, sms, st));
  }
  return NIMG_OK;
}

int expert_ffn_impl(const nimg_ffn_desc* f, const int64_t* off, const int32_t* ex,
                    const void* xr, const void* w1, const void* w3, const void* w2, void* yr,
                    const void* xs, const void* sw1, const void* sw3, const void* sw2, void* ys,
                    void* ws, size_t ws_bytes, cudaStream_t st,
                    const int32_t* gather_idx = nullptr, int64_t gather_src_rows = 0,
                    const FfnTrain* tr = nullptr, const BgGather* bg = nullptr,
                    const int32_t* y_row_map = nullptr) {
  NIMG_TRY(check_ffn(f, off, ex));
  if (!tr && ws_bytes < ffn_ws_bytes(f)) return fail(NIMG_ERR_CONFIG, "workspace too small");
  const bool has_r = f->n_rows > 0, has_s = f->n_shared_rows > 0;
  if (!has_r && !has_s) return NIMG_OK;
  if ((has_r && (!xr || !w1 || !w3 || !w2 || !yr)) || (has_s && (!xs || !sw1 || !sw3 || !sw2 || !ys)))
    return fail(NIMG_ERR_SHAPE, "null tensor pointer");
  const bool tc = ffn_use_tc(f) && !(tr && tr->force_simt);
  if (!tc && !tr && !gather_idx && !bg && ffn_use_x3(f)) {
    const void* ptrs[] = {xr, w1, w3, w2, yr, xs, sw1, sw3, sw2, ys};
    for (const void* q : ptrs)
      if (q && !aligned16(q)) return fail(NIMG_ERR_SHAPE, "tensor not 16-byte aligned");
    return expert_ffn_x3(f, off, ex, xr, w1, w3, w2, yr, xs, sw1, sw3, sw2, ys, ws, st);
  }
  const bool f64 = f->act_dtype == NIMG_F64;
  if (f64 && (tr || gather_idx || bg)) return fail(NIMG_ERR_CONFIG, "internal: f64 mode is forward-only");
  const size_t e = tc ? 2 : (f64 ? 8 : 4);
  uint8_t* pre_r = static_cast<uint8_t*>(ws);
  uint8_t* pre_s = pre_r + align_up((size_t)f->n_rows * f->h * e);
  if (tr) {
    pre_r = static_cast<uint8_t*>(tr->pre_r);
    pre_s = static_cast<uint8_t*>(tr->pre_s);
  }
  void* h_r = tr ? tr->h_r : nullptr;
  void* h_s = tr ? tr->h_s : nullptr;
  const int d = (int)f->d, h = (int)f->h, hs = (int)(has_s ? f->h_shared : f->h);

  if (tc) {
    const void* ptrs[] = {xr, w1, w3, w2, yr, xs, sw1, sw3, sw2, ys, pre_r, pre_s};
    for (const void* q : ptrs)
      if (q && !aligned16(q)) return fail(NIMG_ERR_SHAPE, "tensor not 16-byte aligned");
    int sms = 0;
    NIMG_TRY(device_sms(&sms));
    // CTA-pair (cta_group::2) kernels; they gather A rows with cp.async, the
    // 1-CTA kernels with TMA gather4
    const bool pair = use_pair_kernels();
    const int tile_rows = pair ? tc_pair_rows() : 128;
    // GEMM1: pre = SiLU(x W1^T) * (x W3^T)
    {
      GroupedParams p;
      memset(&p, 0, sizeof(p));
      const int bn = tc_bn_out(0), box = tc_b_box(0);
      NIMG_TRY(fill_segments(p, f, off, ex, tile_rows, (h + bn - 1) / bn, (hs + bn - 1) / bn));
      TmapSet tm;
      memset(&tm, 0, sizeof(tm));
      const int rb = has_r ? 0 : 1;  // any valid bank to alias an unused one
      if (has_r) {
        if (gather_idx) NIMG_TRY(map_2d(&tm.a[0], xr, gather_src_rows, d, 1));
        else NIMG_TRY(map_2d(&tm.a[0], xr, f->n_rows, d, 128));
        NIMG_TRY(map_3d(&tm.b[0], w1, f->n_experts, h, d, box));
        NIMG_TRY(map_3d(&tm.b3[0], w3, f->n_experts, h, d, box));
      }
      if (has_s) {
        NIMG_TRY(map_2d(&tm.a[1], xs, f->n_shared_rows, d, 128));
        NIMG_TRY(map_3d(&tm.b[1], sw1, 1, hs, d, box));
        NIMG_TRY(map_3d(&tm.b3[1], sw3, 1, hs, d, box));
      }
      if (!has_r) { tm.a[0] = tm.a[1]; tm.b[0] = tm.b[1]; tm.b3[0] = tm.b3[1]; }
      if (!has_s) { tm.a[1] = tm.a[rb]; tm.b[1] = tm.b[rb]; tm.b3[1] = tm.b3[rb]; }
      p.bank[0] = GBank{pre_r, h, d, h, (h + bn - 1) / bn, 0, gather_idx, gather_idx ? xr : nullptr, h_r};
      p.bank[1] = GBank{pre_s, hs, d, hs, (hs + bn - 1) / bn, 0, nullptr, nullptr, h_s};
      if (bg && pair && has_r && has_s && !gather_idx) p.bg = *bg;
      if (pair) CUDA_TRY(launch_grouped_tc_pair(0, tm, p, sms, st));
      else CUDA_TRY(launch_grouped_tc(0, tm, p, sms, st));
      mark(3, st);
    }
    // GEMM2: y = pre W2^T
    {
      GroupedParams p;
      memset(&p, 0, sizeof(p));
      const int bn = tc_bn_out(1), box = pair ? tc_b_box(1) / 2 : tc_b_box(1);
      NIMG_TRY(fill_segments(p, f, off, ex, tile_rows, (d + bn - 1) / bn, (d + bn - 1) / bn));
      TmapSet tm;
      memset(&tm, 0, sizeof(tm));
      if (has_r) {
        NIMG_TRY(map_2d(&tm.a[0], pre_r, f->n_rows, h, 128));
        NIMG_TRY(map_3d(&tm.b[0], w2, f->n_experts, d, h, box));
      }
      if (has_s) {
        NIMG_TRY(map_2d(&tm.a[1], pre_s, f->n_shared_rows, hs, 128));
        NIMG_TRY(map_3d(&tm.b[1], sw2, 1, d, hs, box));
      }
      if (!has_r) { tm.a[0] = tm.a[1]; tm.b[0] = tm.b[1]; }
      if (!has_s) { tm.a[1] = tm.a[0]; tm.b[1] = tm.b[0]; }
      tm.b3[0] = tm.b[0];
      tm.b3[1] = tm.b[1];
      // y_row_map (pair kernel): routed row r -> row y_row_map[r] of yr
      p.bank[0] = GBank{yr, d, h, d, (d + bn - 1) / bn, 0, pair ? y_row_map : nullptr, nullptr};
      p.bank[1] = GBank{ys, d, hs, d, (d + bn - 1) / bn, 0, nullptr, nullptr};
      if (pair) CUDA_TRY(launch_grouped_tc_pair(1, tm, p, sms, st));
      else CUDA_TRY(launch_grouped_tc(1, tm, p, sms, st));
    }
    return NIMG_OK;
  }

  // SIMT path: fp32 pre / y (f64 in the f64 storage mode)
  if (gather_idx) return fail(NIMG_ERR_CONFIG, "internal: fused gather needs the tcgen05 path");
  const bool bf = f->act_dtype == NIMG_BF16;
  const int bm = simt_bm(), bn = simt_bn();
  {
    SimtParams p;
    memset(&p, 0, sizeof(p));
    NIMG_TRY(fill_segments(p, f, off, ex, bm, (h + bn - 1) / bn, (hs + bn - 1) / bn));
    p.bank[0] = SimtBank{xr, d, w1, w3, pre_r, h, d, h, (h + bn - 1) / bn, 0, static_cast<float*>(h_r)};
    p.bank[1] = SimtBank{xs, d, sw1, sw3, pre_s, hs, d, hs, (hs + bn - 1) / bn, 0, static_cast<float*>(h_s)};
    CUDA_TRY(launch_grouped_simt(0, bf, p, st, f64));
    mark(3, st);
  }
  {
    SimtParams p;
    memset(&p, 0, sizeof(p));
    NIMG_TRY(fill_segments(p, f, off, ex, bm, (d + bn - 1) / bn, (d + bn - 1) / bn));
    p.bank[0] = SimtBank{pre_r, h, w2, nullptr, yr, d, h, d, (d + bn - 1) / bn, 0};
    p.bank[1] = SimtBank{pre_s, hs, sw2, nullptr, ys, d, hs, d, (d + bn - 1) / bn, 0};
    CUDA_TRY(launch_grouped_simt(1, bf, p, st, f64));
  }
  return NIMG_OK;
}

// fuse_gates: the layer forward's combine forms the gates itself (GateFuse):
// select also writes the per-token expert masks, and the gate kernel is skipped
// (comb_rows / comb_cnt are then not written; gates are, by the combine)
int route_impl(const nimg_moe_desc* d, const void* x_norm, const void* t_emb_v, const void* w_r_v,
               const nimg_route_out* o, void* ws, size_t ws_bytes, cudaStream_t st,
               bool fuse_gates = false) {
  NIMG_TRY(check_moe_desc(d));
  if (!o || !o->logits || !o->scores_bes || !o->token_flat || !o->gate_raw || !o->gates ||
      !o->comb_rows || !o->comb_cnt)
    return fail(NIMG_ERR_SHAPE, "null routing output pointer");
  if (!x_norm || !t_emb_v || !w_r_v) return fail(NIMG_ERR_SHAPE, "null input pointer");
  if (!ws || ws_bytes < route_ws_bytes(d)) return fail(NIMG_ERR_CONFIG, "workspace too small");
  const int B = (int)d->B, S = (int)d->S, dd = (int)d->d, E = (int)d->E, cap = (int)d->cap;
  RouteWs w = carve_route(d, ws);
  if (d->act_dtype == NIMG_F64) {   // f64 storage mode: every routing value in f64
    CUDA_TRY(launch_route_f64(static_cast<const double*>(x_norm), static_cast<const double*>(t_emb_v),
                              static_cast<const double*>(w_r_v), static_cast<double*>(o->logits),
                              static_cast<double*>(o->scores_bes), o->token_flat,
                              static_cast<double*>(o->gate_raw), static_cast<double*>(o->gates),
                              o->comb_rows, o->comb_cnt, w.slot_of, B, S, dd, E, cap, d->gate_eps_f64,
                              d->gate_scale_f64, st));
    mark(6, st);
    return NIMG_OK;
  }
  const float* t_emb = static_cast<const float*>(t_emb_v);
  const float* w_r = static_cast<const float*>(w_r_v);
  float* logits = static_cast<float*>(o->logits);
  float* scores_bes = static_cast<float*>(o->scores_bes);
  // the router reads x_norm in its own dtype (router.py:120-122 routes on the
  // caller's x_norm values, whatever x_mod's dtype)
  const bool xn_bf16 = d->router_dtype == NIMG_BF16;
  // ec_select writes the whole slot table; only the DFMA router (E > 64) needs
  // its per-sample completion counters armed (0xFFFFFFFF; the workspace is
  // caller-owned).
  if (!router_uses_dmma(E))
    CUDA_TRY(cudaMemsetAsync(w.counters, 0xFF, (size_t)B * 4, st));
  // fuse_gates: the token masks and what the gate kernel would have zeroed
  // (GEMM1's gather flags) -- by the INT8 router's prep kernel, else memsets
  const bool i8 = router_i8_eligible(xn_bf16, dd, E, x_norm, w_r);
  if (fuse_gates && !i8) {
    CUDA_TRY(cudaMemsetAsync(w.bg_flags, 0, (size_t)bg_flag_count(d) * 4, st));
    CUDA_TRY(cudaMemsetAsync(w.tokmask, 0, (size_t)B * S * 8, st));
  }
  if (i8) {
    ZeroSpans zs;
    if (fuse_gates) zs = ZeroSpans{w.tokmask, (int64_t)B * S, w.bg_flags, bg_flag_count(d)};
    CUDA_TRY(launch_router_i8(x_norm, t_emb, w_r, w.part, w.i8, logits, scores_bes, B, S, dd, st, zs));
  } else
    CUDA_TRY(launch_router(xn_bf16, x_norm, t_emb, w_r, w.tb, w.part, w.counters, w.wd, logits,
                           scores_bes, B, S, dd, E, st));
  mark(6, st);   // router scores done (inside stage 0 -> 1)
  CUDA_TRY(launch_ec_select(scores_bes, o->token_flat, static_cast<float*>(o->gate_raw), w.slot_of, B,
                            S, E, cap, st, w.cursor, fuse_gates ? w.tokmask : nullptr,
                            fuse_gates ? w.tokent : nullptr));
  if (fuse_gates) return NIMG_OK;
  // fp32(eps) / fp32(alpha): as_tensor(scalar, like=fp32 tensor) (tensor.py:183-187)
  CUDA_TRY(launch_gate_norm(scores_bes, w.slot_of, static_cast<float*>(o->gates), o->comb_rows, o->comb_cnt, B, S,
                            E, cap, d->gate_eps, d->gate_scale, st, w.bg_flags,
                            (int)bg_flag_count(d),
                            use_tok_order() ? TokOrder{w.tok_off, w.row_map, w.gate_tok, w.cursor}
                                            : TokOrder{nullptr, nullptr, nullptr, nullptr}));
  return NIMG_OK;
}

// Routed-row gather (moe.py:152-153): a separate HBM-bound kernel by default.
// NIMG_FUSED_GATHER=1 fuses it into GEMM1's operand load instead -- the pair
// kernel copies the token_flat-selected x_mod rows with cp.async (relay-warp
// signalled), the 1-CTA kernel (NIMG_PAIR=0) with TMA tile::gather4. Both are
// correct (bitwise equal, tests/test_gpu_parity.py) but slower on B200:
// LDGSTS sustains ~8 B/cycle/SM and gather4 issues at ~45 cycles per 512 B,
// against the ~36 B/cycle/SM of A operand the UMMA consumes (GEMM1 1.51 ms /
// 1.83 ms fused vs 0.63 ms + 0.064 ms separate gather at cfg2).
bool use_bg_gather() {
  static const bool on = [] {
    const char* e = getenv("NIMG_BG_GATHER");
    return !(e && e[0] == '0');
  }();
  return on;
}
// NIMG_TOK_ORDER=1: GEMM2 writes the routed rows in token order and the
// combine streams each token's rows (bitwise equal). Off by default: measured
// equal at cfg2 (combine 89.2 -> 86.8 us, GEMM2 +1.7 us, gates +3.6 us for the
// row allocation) -- the combine is bound by mixed read/write DRAM
// efficiency, not by its row gather.
bool use_tok_order() {
  static const bool on = [] {
    const char* e = getenv("NIMG_TOK_ORDER");
    return e && e[0] == '1';
  }();
  return on;
}
bool use_fused_gather(int32_t path, int64_t d) {
  static const bool on = [] {
    const char* e = getenv("NIMG_FUSED_GATHER");
    return e && e[0] == '1';
  }();
  return on && path == NIMG_PATH_TCGEN05 && d % 64 == 0;   // (bf16 layers: checked by the caller)
}

// ------------------------------------------------------------- training state
// tcgen05 training path: bf16 layer whose backward GEMMs tile cleanly
// (K = h and 2h split at 64-column boxes); else the CUDA-core path with fp32
// intermediates.
bool train_use_tc(const nimg_moe_desc* d) {
  return d->act_dtype == NIMG_BF16 && d->d % 64 == 0 && d->h % 64 == 0 && d->h_shared % 64 == 0;
}

struct TrainState {
  bool tc;
  void *xg, *h_r, *h_s, *pre_r, *pre_s, *y_r;
  size_t bytes;
};
TrainState train_state_layout(const nimg_moe_desc* d, void* base) {
  TrainState s{};
  s.tc = train_use_tc(d);
  const size_t R = (size_t)d->E * d->B * d->cap, T = (size_t)d->B * d->S;
  const size_t ea = elt(d->act_dtype), ei = s.tc ? 2 : 4;
  uint8_t* p = static_cast<uint8_t*>(base);
  size_t o = 0;
  auto take = [&](size_t bytes) { void* q = p ? p + o : nullptr; o += align_up(bytes); return q; };
  s.xg = take(R * d->d * ea);
  // tcgen05: row-blocked h1 | h3 (hblk_off, 128-row blocks); CUDA cores: row-major fp32
  s.h_r = take(s.tc ? hblk_elems((int64_t)R, d->h) * 2 : R * 2 * d->h * ei);
  s.h_s = take(s.tc ? hblk_elems((int64_t)T, d->h_shared) * 2 : T * 2 * d->h_shared * ei);
  s.pre_r = take(R * d->h * ei);
  s.pre_s = take(T * d->h_shared * ei);
  s.y_r = take(R * d->d * ei);
  s.bytes = o;
  return s;
}

struct BwdWs {
  void *dy_r, *dy_s, *dh_r, *dh_s, *dx_r, *dx_s;
  float *dlogits, *colsum, *part;
  bf16_raw *dl16, *wr16;   // tcgen05 router pullback operands
  float *sp1, *sp2, *sp3;  // shared-bank weight-gradient row-chunk partials
  size_t bytes;
};
// Shared-expert weight gradients reduce over all T rows (16x a routed
// segment at cfg2): on the tcgen05 path they are split into ks row chunks
// (own partial outputs, folded in fixed order) so the persistent grid's
// round-robin stays balanced.
int shared_wgrad_chunks(const nimg_moe_desc* d) {
  if (!train_use_tc(d)) return 1;
  const int64_t T = d->B * d->S, rows_e = d->B * d->cap;
  int ks = (int)(T / (4 * rows_e));
  ks = ks < 1 ? 1 : (ks > 4 ? 4 : ks);
  while (ks > 1 && T % (64 * ks)) --ks;
  return ks;
}
// Router pullback on tcgen05 (bf16 layer, TMA-aligned E)
bool router_bwd_tc(const nimg_moe_desc* d) { return train_use_tc(d) && d->E % 8 == 0; }
BwdWs bwd_ws_layout(const nimg_moe_desc* d, void* base) {
  BwdWs w{};
  const bool tc = train_use_tc(d);
  const size_t R = (size_t)d->E * d->B * d->cap, T = (size_t)d->B * d->S;
  const size_t ei = tc ? 2 : 4;
  uint8_t* p = static_cast<uint8_t*>(base);
  size_t o = 0;
  auto take = [&](size_t bytes) { void* q = p ? p + o : nullptr; o += align_up(bytes); return q; };
  w.dy_r = take(R * d->d * ei);
  w.dy_s = tc ? nullptr : take(T * d->d * ei);   // tcgen05: g_out itself is the shared A operand
  w.dh_r = take(R * 2 * d->h * ei);
  w.dh_s = take(T * 2 * d->h_shared * ei);
  w.dx_r = take(R * d->d * ei);
  w.dx_s = take(T * d->d * ei);
  w.dlogits = static_cast<float*>(take(T * d->E * 4));
  w.colsum = static_cast<float*>(take((size_t)d->B * d->E * 4));
  const size_t part_simt = router_bwd_part_bytes((int64_t)T, (int)d->d, (int)d->E);
  const size_t part_tc = (size_t)d->B * d->d * d->E * 4;   // one partial per sample
  w.part = static_cast<float*>(take(part_simt > part_tc ? part_simt : part_tc));
  const bool rtc = router_bwd_tc(d);
  const int ks = shared_wgrad_chunks(d);
  w.sp2 = ks > 1 ? static_cast<float*>(take((size_t)ks * d->d * d->h_shared * 4)) : nullptr;
  w.sp1 = ks > 1 ? static_cast<float*>(take((size_t)ks * d->h_shared * d->d * 4)) : nullptr;
  w.sp3 = ks > 1 ? static_cast<float*>(take((size_t)ks * d->h_shared * d->d * 4)) : nullptr;
  w.dl16 = rtc ? static_cast<bf16_raw*>(take(T * d->E * 2)) : nullptr;
  w.wr16 = rtc ? static_cast<bf16_raw*>(take((size_t)d->d * d->E * 2)) : nullptr;
  w.bytes = o;
  return w;
}

// Segment table of one backward grouped launch. W modes put the shared bank
// first (its tiles reduce over all T rows: longest first).
int fill_bwd_segments(BwdParams& p, int mode, const nimg_moe_desc* d, int bm, int bn,
                      int ks_shared = 1) {
  const bool wm = mode == BWD_W2 || mode == BWD_W1;
  const int64_t rows_e = d->B * d->cap, T = d->B * d->S;
  int n = 0;
  int64_t tiles = 0;
  auto add = [&](int bank, int64_t row0, int64_t rows, int expert) {
    BwdBank& bk = p.bank[bank];
    p.seg_row0[n] = (int)row0;
    p.seg_rows[n] = (int)rows;
    p.seg_expert[n] = expert;
    p.seg_bank[n] = bank;
    p.seg_tile0[n] = (int)tiles;
    bk.ntn = (bk.N + bn - 1) / bn;
    bk.ntm = wm ? (bk.M + bm - 1) / bm : 0;
    tiles += wm ? (int64_t)bk.ntm * bk.ntn : (rows + bm - 1) / bm * bk.ntn;
    ++n;
  };
  if (wm) {
    const int ks = ks_shared;
    for (int c = 0; c < ks; ++c) add(1, c * (T / ks), T / ks, c);
  }
  for (int e = 0; e < d->E; ++e) add(0, e * rows_e, rows_e, e);
  if (!wm) add(1, 0, T, 0);
  p.nseg = n;
  p.seg_tile0[n] = (int)tiles;
  if (tiles >= ((int64_t)1 << 31)) return fail(NIMG_ERR_CONFIG, "too many tiles");
  p.total_tiles = (int)tiles;
  return NIMG_OK;
}

nimg_ffn_desc layer_ffn_desc(const nimg_moe_desc* d) {
  nimg_ffn_desc f;
  memset(&f, 0, sizeof(f));
  f.n_rows = d->E * d->B * d->cap;
  f.n_shared_rows = d->B * d->S;
  f.d = d->d;
  f.h = d->h;
  f.h_shared = d->h_shared;
  f.n_experts = d->E;
  f.act_dtype = d->act_dtype;
  f.nseg = (int32_t)d->E;
  return f;
}

}  // namespace

// ================================================================== C ABI
extern "C" {

const char* nimg_last_error(void) { return g_err.c_str(); }
int nimg_abi_version(void) { return 2; }
int nimg_device_sms(int* sms) {
  if (!sms) return fail(NIMG_ERR_CONFIG, "null output");
  return device_sms(sms);
}

int nimg_capacity_for(int64_t S, int64_t E, double C, int64_t* cap) {
  if (!cap) return fail(NIMG_ERR_CONFIG, "null output");
  if (S < 1 || E < 1 || !(C > 0))
    return fail(NIMG_ERR_CONFIG, "invalid capacity arguments S=%lld E=%lld C=%g", (long long)S,
                (long long)E, C);
  const int64_t c = (int64_t)std::ceil(C * (double)S / (double)E);  // router.py:74 order
  *cap = c < S ? c : S;
  return NIMG_OK;
}

int nimg_route_workspace_bytes(const nimg_moe_desc* d, size_t* bytes) {
  NIMG_TRY(check_moe_desc(d));
  if (!bytes) return fail(NIMG_ERR_CONFIG, "null output");
  *bytes = route_ws_bytes(d);
  return NIMG_OK;
}

int nimg_route(const nimg_moe_desc* d, const void* x_norm, const void* t_emb, const void* w_r,
               const nimg_route_out* out, void* ws, size_t ws_bytes, void* stream) {
  return route_impl(d, x_norm, t_emb, w_r, out, ws, ws_bytes, (cudaStream_t)stream);
}

// The fused routing form (gates formed in the combine): E <= 64, the block
// select path, fp32 / bf16 values.
static bool route_fusable(const nimg_moe_desc* d) {
  return d && d->act_dtype != NIMG_F64 && d->E <= 64 && select_blk_path((int)d->S);
}
int nimg_route_fusable(const nimg_moe_desc* d) {
  NIMG_TRY(check_moe_desc(d));
  return route_fusable(d) ? 1 : 0;
}
int nimg_route_for_combine(const nimg_moe_desc* d, const void* x_norm, const void* t_emb,
                           const void* w_r, const nimg_route_out* out, void* ws, size_t ws_bytes,
                           void* stream) {
  NIMG_TRY(check_moe_desc(d));
  if (!route_fusable(d)) return fail(NIMG_ERR_CONFIG, "routing not fusable with the combine (E %lld, S %lld)",
                                     (long long)d->E, (long long)d->S);
  return route_impl(d, x_norm, t_emb, w_r, out, ws, ws_bytes, (cudaStream_t)stream, true);
}
int nimg_combine_routed(const nimg_moe_desc* d, const void* route_ws, int32_t y_dtype,
                        int32_t out_dtype, const void* y_routed, const void* y_shared, void* gates,
                        const void* hres, const void* th_ff, void* out, void* stream) {
  NIMG_TRY(check_moe_desc(d));
  if (!route_fusable(d)) return fail(NIMG_ERR_CONFIG, "routing not fusable with the combine");
  if (!route_ws || !y_shared || !out || !gates || (d->cap > 0 && !y_routed))
    return fail(NIMG_ERR_SHAPE, "null pointer");
  if (y_dtype == NIMG_F64 || out_dtype == NIMG_F64) return fail(NIMG_ERR_CONFIG, "f64 combine is not fused");
  const RouteWs rw = carve_route(d, const_cast<void*>(route_ws));
  const GateFuse gf{rw.tokmask, rw.tokent, static_cast<float*>(gates), d->gate_eps, d->gate_scale};
  const int64_t T = d->B * d->S;
  CUDA_TRY(launch_combine(y_dtype == NIMG_BF16, out_dtype == NIMG_BF16, y_routed, y_shared, nullptr,
                          nullptr, nullptr, out, T, (int)d->d, (int)d->E, (cudaStream_t)stream, hres,
                          th_ff, (int)d->S, nullptr, &gf));
  return NIMG_OK;
}

int nimg_gather_rows(const void* src, int64_t n_src_rows, int64_t row_bytes, const int32_t* idx,
                     int64_t n_idx, void* dst, void* stream) {
  if (n_idx < 0 || row_bytes < 0 || n_src_rows < 0) return fail(NIMG_ERR_SHAPE, "negative size");
  if (n_idx == 0 || row_bytes == 0) return NIMG_OK;
  if (!src || !idx || !dst) return fail(NIMG_ERR_SHAPE, "null pointer");
  CUDA_TRY(launch_gather_rows(src, row_bytes, idx, n_idx, dst, (cudaStream_t)stream));
  return NIMG_OK;
}

int nimg_ffn_path(const nimg_ffn_desc* f, int32_t* path, int32_t* y_dtype) {
  if (!f || !path || !y_dtype) return fail(NIMG_ERR_CONFIG, "null argument");
  const bool tc = ffn_use_tc(f);
  *path = tc || ffn_use_x3(f) ? NIMG_PATH_TCGEN05 : NIMG_PATH_SIMT;
  *y_dtype = tc ? NIMG_BF16 : (f->act_dtype == NIMG_F64 ? NIMG_F64 : NIMG_F32);
  return NIMG_OK;
}

int nimg_ffn_workspace_bytes(const nimg_ffn_desc* f, size_t* bytes) {
  if (!f || !bytes) return fail(NIMG_ERR_CONFIG, "null argument");
  *bytes = ffn_ws_bytes(f);
  return NIMG_OK;
}

int nimg_expert_ffn(const nimg_ffn_desc* f, const int64_t* off, const int32_t* ex, const void* xr,
                    const void* w1, const void* w3, const void* w2, void* yr, const void* xs,
                    const void* sw1, const void* sw3, const void* sw2, void* ys, void* ws,
                    size_t ws_bytes, void* stream) {
  return expert_ffn_impl(f, off, ex, xr, w1, w3, w2, yr, xs, sw1, sw3, sw2, ys, ws, ws_bytes,
                         (cudaStream_t)stream);
}

int nimg_route_bg_flags(const nimg_moe_desc* d, void* route_ws, int32_t** flags) {
  NIMG_TRY(check_moe_desc(d));
  if (!route_ws || !flags) return fail(NIMG_ERR_CONFIG, "null argument");
  *flags = carve_route(d, route_ws).bg_flags;
  return NIMG_OK;
}

int nimg_expert_ffn_gather(const nimg_ffn_desc* f, const int64_t* off, const int32_t* ex,
                           const void* xr, const void* w1, const void* w3, const void* w2, void* yr,
                           const void* xs, const void* sw1, const void* sw3, const void* sw2,
                           void* ys, void* ws, size_t ws_bytes, const nimg_bg_gather* g,
                           void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  NIMG_TRY(check_ffn(f, off, ex));
  if (!g || !g->src || !g->idx || !g->dst || !g->flags || g->rows < 0 || g->row_bytes <= 0 ||
      g->row_off < 0 || g->row_off + f->n_rows > g->rows || (g->chunk_rows > 0 && !g->chunk_done))
    return fail(NIMG_ERR_SHAPE, "bad gather descriptor");
  if (f->n_rows > 0 && xr != static_cast<const uint8_t*>(g->dst) + (size_t)g->row_off * g->row_bytes)
    return fail(NIMG_ERR_SHAPE, "x_routed must be dst + row_off rows");
  const bool fuse = ffn_use_tc(f) && use_pair_kernels() && f->n_rows > 0 && f->n_shared_rows > 0 &&
                    g->row_bytes % 16 == 0;
  BgGather bg{g->src, g->idx, g->dst, g->flags, g->rows, g->row_bytes, g->row_off, g->chunk_rows,
              g->chunk_done};
  if (!fuse) {   // the separate gather kernel, then the same chunk counts
    CUDA_TRY(launch_gather_rows(g->src, g->row_bytes, g->idx, g->rows, g->dst, st));
    if (g->chunk_rows > 0) CUDA_TRY(launch_bg_count(g->rows, g->chunk_rows, g->chunk_done, st));
  }
  return expert_ffn_impl(f, off, ex, xr, w1, w3, w2, yr, xs, sw1, sw3, sw2, ys, ws, ws_bytes, st,
                         nullptr, 0, nullptr, fuse ? &bg : nullptr);
}

int nimg_combine(int64_t T, int64_t d, int64_t E, int32_t y_dtype, int32_t out_dtype,
                 const void* y_routed, const void* y_shared, const void* gates_v,
                 const int32_t* comb_rows, const int32_t* comb_cnt, void* out, void* stream) {
  if (T < 0 || d < 1 || E < 1) return fail(NIMG_ERR_SHAPE, "bad combine shape");
  if (T == 0) return NIMG_OK;
  if (!y_shared || !comb_cnt || !comb_rows || !out || !gates_v)
    return fail(NIMG_ERR_SHAPE, "null pointer");
  if ((y_dtype == NIMG_F64) != (out_dtype == NIMG_F64))
    return fail(NIMG_ERR_CONFIG, "f64 combine needs f64 y and out");
  if (y_dtype == NIMG_F64) {
    CUDA_TRY(launch_combine_f64(static_cast<const double*>(y_routed), static_cast<const double*>(y_shared),
                                static_cast<const double*>(gates_v), comb_rows, comb_cnt,
                                static_cast<double*>(out), T, (int)d, (int)E, (cudaStream_t)stream));
    return NIMG_OK;
  }
  const float* gates = static_cast<const float*>(gates_v);
  CUDA_TRY(launch_combine(y_dtype == NIMG_BF16, out_dtype == NIMG_BF16, y_routed, y_shared, gates,
                          comb_rows, comb_cnt, out, T, (int)d, (int)E, (cudaStream_t)stream));
  return NIMG_OK;
}

// ---------------------------------------------------------------- stack helpers
static int check_rows(int64_t rows, int64_t S, int64_t d, int32_t dt, const void* const* ptrs, int n) {
  if (rows < 0 || S < 1 || d < 1 || rows % S) return fail(NIMG_ERR_SHAPE, "bad row geometry");
  if (dt != NIMG_BF16 && dt != NIMG_F32) return fail(NIMG_ERR_CONFIG, "unsupported dtype %d", dt);
  if (d % (dt == NIMG_BF16 ? 8 : 4)) return fail(NIMG_ERR_SHAPE, "d %lld not a multiple of 16 bytes", (long long)d);
  for (int i = 0; i < n; ++i)
    if (!ptrs[i] || !aligned16(ptrs[i])) return fail(NIMG_ERR_SHAPE, "null or misaligned pointer");
  return NIMG_OK;
}

int nimg_ln_modulate(int64_t rows, int64_t S, int64_t d, int32_t dtype, const void* x,
                     const float* scale, const float* shift, void* out, float eps, void* stream) {
  const void* p[] = {x, scale, out};
  NIMG_TRY(check_rows(rows, S, d, dtype, p, 3));
  CUDA_TRY(launch_row_modulate(0, dtype == NIMG_BF16, x, nullptr, nullptr, scale, shift, nullptr,
                               out, rows, (int)S, (int)d, eps, (cudaStream_t)stream));
  return NIMG_OK;
}

int nimg_gate_res_ln_modulate(int64_t rows, int64_t S, int64_t d, int32_t dtype, const void* x,
                              const void* r, const float* th, const float* scale, void* h_out,
                              void* m_out, float eps, void* stream) {
  const void* p[] = {x, r, th, scale, h_out, m_out};
  NIMG_TRY(check_rows(rows, S, d, dtype, p, 6));
  CUDA_TRY(launch_row_modulate(1, dtype == NIMG_BF16, x, r, th, scale, nullptr, h_out, m_out, rows,
                               (int)S, (int)d, eps, (cudaStream_t)stream));
  return NIMG_OK;
}

int nimg_gated_residual(int64_t rows, int64_t S, int64_t d, int32_t dtype, const void* x,
                        const void* r, const float* th, void* out, void* stream) {
  const void* p[] = {x, r, th, out};
  NIMG_TRY(check_rows(rows, S, d, dtype, p, 4));
  CUDA_TRY(launch_row_modulate(2, dtype == NIMG_BF16, x, r, th, nullptr, nullptr, out, nullptr, rows,
                               (int)S, (int)d, 0.f, (cudaStream_t)stream));
  return NIMG_OK;
}

int nimg_qk_norm_rope(int64_t rows, int64_t S, int64_t H, int64_t dh, int32_t dtype, const void* x,
                      int64_t x_token_stride, const float* cos_t, const float* sin_t, void* out,
                      float eps, void* stream) {
  if (rows < 0 || S < 1 || H < 1 || dh < 2 || dh % 2 || rows % (S * H) || x_token_stride < H * dh)
    return fail(NIMG_ERR_SHAPE, "bad head geometry");
  if (dtype != NIMG_BF16 && dtype != NIMG_F32) return fail(NIMG_ERR_CONFIG, "unsupported dtype %d", dtype);
  if (!x || !cos_t || !sin_t || !out) return fail(NIMG_ERR_SHAPE, "null pointer");
  CUDA_TRY(launch_qk_norm_rope(dtype == NIMG_BF16, x, x_token_stride, cos_t, sin_t, out, rows, (int)S,
                               (int)H, (int)dh, eps, (cudaStream_t)stream));
  return NIMG_OK;
}

int nimg_moe_workspace_bytes(const nimg_moe_desc* d, size_t* bytes) {
  NIMG_TRY(check_moe_desc(d));
  if (!bytes) return fail(NIMG_ERR_CONFIG, "null output");
  const nimg_ffn_desc f = layer_ffn_desc(d);
  int32_t path, ydt;
  nimg_ffn_path(&f, &path, &ydt);
  // the gathered-row buffer exists only when the gather is not fused into GEMM1
  const size_t xg = d->act_dtype == NIMG_BF16 && use_fused_gather(path, d->d)
                        ? 0 : align_up((size_t)f.n_rows * d->d * elt(d->act_dtype));
  // the training forward (moe_forward_impl with a state blob) keeps the shared
  // expert's outputs in fp32 on the CUDA-core training path: size for both
  const size_t ys_elt = std::max<size_t>(elt(ydt), train_use_tc(d) ? 2 : 4);
  *bytes = route_ws_bytes(d) + xg + ffn_ws_bytes(&f) + align_up((size_t)f.n_rows * d->d * elt(ydt)) +
           align_up((size_t)f.n_shared_rows * d->d * ys_elt);
  return NIMG_OK;
}

// moe.py:138-164; with resid_h, the combine writes h + th_ff * moe (backbone.py:606).
// state != null: training forward -- the gathered rows, h1 | h3, pre and the
// routed expert outputs land in the caller's state blob (train_state_layout).
static int moe_forward_impl(const nimg_moe_desc* d, const nimg_moe_ptrs* p, void* ws, size_t ws_bytes,
                            cudaStream_t st, const void* resid_h, const void* th_ff,
                            void* state = nullptr) {
  NIMG_TRY(check_moe_desc(d));
  if (!p) return fail(NIMG_ERR_SHAPE, "null pointers");
  size_t need = 0;
  NIMG_TRY(nimg_moe_workspace_bytes(d, &need));
  if (!ws || ws_bytes < need) return fail(NIMG_ERR_CONFIG, "workspace too small (%zu < %zu)", ws_bytes, need);
  const nimg_ffn_desc f = layer_ffn_desc(d);
  int32_t path, ydt;
  nimg_ffn_path(&f, &path, &ydt);
  // the workspace carve follows nimg_moe_workspace_bytes (inference dtypes);
  // the training forward only re-types the outputs it writes
  const int32_t ydt_ws = ydt;
  FfnTrain tr{};
  TrainState ts{};
  if (state) {
    ts = train_state_layout(d, state);
    tr = FfnTrain{!ts.tc, ts.pre_r, ts.pre_s, ts.h_r, ts.h_s};
    ydt = ts.tc ? NIMG_BF16 : NIMG_F32;
    path = ts.tc ? NIMG_PATH_TCGEN05 : NIMG_PATH_SIMT;
  }
  // gathers inside GEMM1 copy bf16 rows of the bf16 tcgen05 path (fp32 layers
  // on the tensor cores split their gathered rows first)
  const bool bf_tc = path == NIMG_PATH_TCGEN05 && d->act_dtype == NIMG_BF16;
  const bool fused_gather = !state && bf_tc && use_fused_gather(path, d->d);
  uint8_t* w = static_cast<uint8_t*>(ws);
  void* route_ws = w;                 w += route_ws_bytes(d);
  void* xg = w;                       if (!fused_gather) w += align_up((size_t)f.n_rows * d->d * elt(d->act_dtype));
  void* ffn_ws = w;                   w += ffn_ws_bytes(&f);
  void* yr = w;                       w += align_up((size_t)f.n_rows * d->d * elt(ydt_ws));
  void* ys = w;
  if (state) { xg = ts.xg; yr = ts.y_r; }

  // the routed-row gather runs inside GEMM1 (background warps) on the tcgen05
  // pair path; NIMG_BG_GATHER=0 keeps the separate gather kernel
  const bool bg_gather = !fused_gather && bf_tc && use_pair_kernels() &&
                         use_bg_gather() && f.n_rows > 0 && f.n_shared_rows > 0 &&
                         (d->d * elt(d->act_dtype)) % 16 == 0;
  BgGather bg{};
  if (bg_gather)
    bg = BgGather{p->x_mod, p->route.token_flat, xg, carve_route(d, route_ws).bg_flags,
                  (int)f.n_rows, (int)(d->d * elt(d->act_dtype)), 0, 0, nullptr};
  // inference on one GPU: the combine forms the gates (no gate kernel)
  const bool tok_order_pre = !state && bf_tc && use_pair_kernels() && gate_tok_supported() &&
                             use_tok_order() && f.n_rows > 0;
  const bool fuse_gates = !state && d->act_dtype != NIMG_F64 && d->E <= 64 &&
                          select_blk_path((int)d->S) && !tok_order_pre && gates_in_combine();
  mark(0, st);
  NIMG_TRY(route_impl(d, p->x_norm, p->t_emb, p->w_r, &p->route, route_ws, route_ws_bytes(d), st,
                      fuse_gates));
  mark(1, st);
  if (!fused_gather && !bg_gather)
    CUDA_TRY(launch_gather_rows(p->x_mod, d->d * (int64_t)elt(d->act_dtype), p->route.token_flat,
                                f.n_rows, xg, st));
  mark(2, st);
  int64_t off[kMaxSeg + 1];
  if (f.nseg > kMaxSeg - 8) return fail(NIMG_ERR_CONFIG, "too many experts for one grouped launch");
  for (int e = 0; e <= f.nseg; ++e) off[e] = (int64_t)e * d->B * d->cap;  // moe.py:154
  // token-ordered expert outputs: GEMM2 writes each routed row where its
  // token's rows are consecutive, the combine streams them (same sums, same
  // expert-ascending order: bitwise equal). Inference on the bf16 pair path.
  const RouteWs rw = carve_route(d, route_ws);
  const bool tok_order = !state && bf_tc && use_pair_kernels() && gate_tok_supported() &&
                         use_tok_order() && f.n_rows > 0;
  // fused path: GEMM1 gathers x_mod rows by token_flat itself (TMA gather4)
  NIMG_TRY(expert_ffn_impl(&f, off, nullptr, fused_gather ? p->x_mod : xg, p->w1, p->w3, p->w2, yr,
                           p->x_mod, p->sw1, p->sw3, p->sw2, ys, ffn_ws, ffn_ws_bytes(&f), st,
                           fused_gather ? p->route.token_flat : nullptr, d->B * d->S,
                           state ? &tr : nullptr, bg_gather ? &bg : nullptr,
                           tok_order ? rw.row_map : nullptr));
  mark(4, st);
  if (d->act_dtype == NIMG_F64)
    CUDA_TRY(launch_combine_f64(static_cast<const double*>(yr), static_cast<const double*>(ys),
                                static_cast<const double*>(p->route.gates), p->route.comb_rows,
                                p->route.comb_cnt, static_cast<double*>(p->out), d->B * d->S,
                                (int)d->d, (int)d->E, st));
  else {
    const GateFuse gf{rw.tokmask, rw.tokent, static_cast<float*>(p->route.gates), d->gate_eps,
                      d->gate_scale};
    CUDA_TRY(launch_combine(ydt == NIMG_BF16, d->act_dtype == NIMG_BF16, yr, ys,
                            tok_order ? rw.gate_tok : static_cast<const float*>(p->route.gates),
                            p->route.comb_rows, p->route.comb_cnt, p->out, d->B * d->S, (int)d->d,
                            (int)d->E, st, resid_h, th_ff, (int)d->S, tok_order ? rw.tok_off : nullptr,
                            fuse_gates ? &gf : nullptr));
  }
  mark(5, st);
  return NIMG_OK;
}

int nimg_moe_forward(const nimg_moe_desc* d, const nimg_moe_ptrs* p, void* ws, size_t ws_bytes,
                     void* stream) {
  return moe_forward_impl(d, p, ws, ws_bytes, (cudaStream_t)stream, nullptr, nullptr);
}

// ------------------------------------------------------------------ training
// Training entry points: fp32 / bf16 layers whose router input has the
// activation dtype (the router pullback reads x_norm as an operand of the same
// GEMM path as x_mod).
static int check_train_desc(const nimg_moe_desc* d) {
  NIMG_TRY(check_moe_desc(d));
  if (d->act_dtype == NIMG_F64)
    return fail(NIMG_ERR_CONFIG, "the f64 storage mode is forward-only (no training path)");
  if (d->router_dtype != d->act_dtype)
    return fail(NIMG_ERR_CONFIG, "training needs x_norm in the activation dtype (router_dtype %d != "
                "act_dtype %d)", d->router_dtype, d->act_dtype);
  return NIMG_OK;
}

int nimg_moe_train_state_bytes(const nimg_moe_desc* d, size_t* bytes) {
  NIMG_TRY(check_train_desc(d));
  if (!bytes) return fail(NIMG_ERR_CONFIG, "null output");
  *bytes = train_state_layout(d, nullptr).bytes;
  return NIMG_OK;
}

int nimg_moe_forward_train(const nimg_moe_desc* d, const nimg_moe_ptrs* p, void* state,
                           size_t state_bytes, void* ws, size_t ws_bytes, void* stream) {
  NIMG_TRY(check_train_desc(d));
  if (!state || state_bytes < train_state_layout(d, nullptr).bytes)
    return fail(NIMG_ERR_CONFIG, "training state too small");
  return moe_forward_impl(d, p, ws, ws_bytes, (cudaStream_t)stream, nullptr, nullptr, state);
}

int nimg_moe_backward_workspace_bytes(const nimg_moe_desc* d, size_t* bytes) {
  NIMG_TRY(check_train_desc(d));
  if (!bytes) return fail(NIMG_ERR_CONFIG, "null output");
  *bytes = bwd_ws_layout(d, nullptr).bytes;
  return NIMG_OK;
}

static int bwd_grouped(int mode, bool tc, bool b_bf16, BwdParams& P, const TmapSetBwd& tm, int sms,
                       const nimg_moe_desc* d, cudaStream_t st, int ks_shared = 1) {
  const int bm = tc ? tc_bwd_tile_rows(mode) : simt_bwd_bm();
  const int bn = tc ? tc_bwd_bn(mode) : simt_bwd_bn();
  NIMG_TRY(fill_bwd_segments(P, mode, d, bm, bn, ks_shared));
  if (tc) CUDA_TRY(launch_grouped_tc_bwd(mode, tm, P, sms, st));
  else CUDA_TRY(launch_grouped_simt_bwd(mode, b_bf16, P, st));
  return NIMG_OK;
}

// The layer's pullback (moe.py:138-164 under backward(tape, loss),
// tensor.py:590-628): see backward_kernels.cu / grouped_gemm_bwd_sm100.cu.
int nimg_moe_backward(const nimg_moe_desc* d, const nimg_moe_ptrs* p, const void* state,
                      size_t state_bytes, const nimg_moe_grads* g, void* ws, size_t ws_bytes,
                      void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  NIMG_TRY(check_train_desc(d));
  if (!p || !g) return fail(NIMG_ERR_SHAPE, "null pointers");
  if (d->E + 5 > kMaxSeg) return fail(NIMG_ERR_CONFIG, "too many experts for one grouped launch");
  const TrainState ts = train_state_layout(d, const_cast<void*>(state));
  if (!state || state_bytes < ts.bytes) return fail(NIMG_ERR_CONFIG, "training state too small");
  const BwdWs w = bwd_ws_layout(d, ws);
  if (!ws || ws_bytes < w.bytes) return fail(NIMG_ERR_CONFIG, "workspace too small (%zu < %zu)", ws_bytes, w.bytes);
  if (!g->g_out || !g->g_x_norm || !g->g_x_mod || !g->g_t_emb || !g->g_w_r || !g->g_w1 || !g->g_w3 ||
      !g->g_w2 || !g->g_sw1 || !g->g_sw3 || !g->g_sw2)
    return fail(NIMG_ERR_SHAPE, "null gradient pointer");
  const nimg_route_out& rv = p->route;
  // training is fp32 / bf16 only (check_train_desc): routing values are fp32
  struct {
    const float *logits, *gates, *gate_raw;
    const int32_t *comb_rows, *comb_cnt, *token_flat;
  } ro{static_cast<const float*>(rv.logits), static_cast<const float*>(rv.gates),
       static_cast<const float*>(rv.gate_raw), rv.comb_rows, rv.comb_cnt, rv.token_flat};
  const float* w_r = static_cast<const float*>(p->w_r);
  const float* t_emb = static_cast<const float*>(p->t_emb);
  if (!ro.logits || !ro.gates || !ro.gate_raw || !ro.comb_rows || !ro.comb_cnt)
    return fail(NIMG_ERR_SHAPE, "null routing pointer");
  const bool tc = ts.tc, bf = d->act_dtype == NIMG_BF16;
  const int ks = shared_wgrad_chunks(d);
  const int64_t T = d->B * d->S, R = d->E * d->B * d->cap, rows_e = d->B * d->cap;
  const int dd = (int)d->d, h = (int)d->h, hs = (int)d->h_shared, E = (int)d->E;
  if (tc) {
    const void* ptrs[] = {g->g_out, p->x_mod, p->w1, p->w3, p->w2, p->sw1, p->sw3, p->sw2, g->g_x_mod};
    for (const void* q : ptrs)
      if (!aligned16(q)) return fail(NIMG_ERR_SHAPE, "tensor not 16-byte aligned");
  }
  int sms = 0;
  NIMG_TRY(device_sms(&sms));
  mark(0, st);
  // 1. combine / gate / softmax pullback -> dY rows, dlogits
  const bool rtc = router_bwd_tc(d);
  CUDA_TRY(launch_combine_bwd(bf, tc, tc, g->g_out, ts.y_r, ro.gates, ro.gate_raw, ro.comb_rows,
                              ro.comb_cnt, ro.logits, w.dy_r, w.dy_s, w.dlogits, w.dl16, T, dd, E,
                              (int)rows_e, d->gate_eps, d->gate_scale, st));
  // 2. router pullback -> g_x_norm, g_t_emb, g_w_r
  int nchunks = 0;
  if (rtc && d->B > kMaxSeg) return fail(NIMG_ERR_CONFIG, "batch too large for one grouped launch");
  if (rtc) {
    // dx_norm = dl W_r[:d]^T: the forward's GEMM2 kernel (A = dl rows, K = E; B = W_r[:d] rows)
    CUDA_TRY(launch_f32_to_bf16(w_r, w.wr16, dd * (int64_t)E, st));
    {
      const bool pair = use_pair_kernels();
      const int bn = tc_bn_out(1), box = pair ? tc_b_box(1) / 2 : tc_b_box(1);
      const int rows_tile = pair ? tc_pair_rows() : 128;
      GroupedParams P;
      memset(&P, 0, sizeof(P));
      TmapSet tmf;
      memset(&tmf, 0, sizeof(tmf));
      NIMG_TRY(map_2d(&tmf.a[0], w.dl16, T, E, 128));
      NIMG_TRY(map_3d(&tmf.b[0], w.wr16, 1, dd, E, box));
      tmf.a[1] = tmf.a[0]; tmf.b[1] = tmf.b[0]; tmf.b3[0] = tmf.b[0]; tmf.b3[1] = tmf.b[0];
      P.bank[0] = GBank{g->g_x_norm, dd, E, dd, (dd + bn - 1) / bn, 0, nullptr, nullptr, nullptr};
      P.bank[1] = P.bank[0];
      P.nseg0 = P.nseg = 1;
      P.seg_row0[0] = 0;
      P.seg_rows[0] = (int)T;
      P.seg_expert[0] = 0;
      P.seg_tile0[0] = 0;
      P.total_tiles = P.seg_tile0[1] = (int)((T + rows_tile - 1) / rows_tile) * ((dd + bn - 1) / bn);
      if (pair) CUDA_TRY(launch_grouped_tc_pair(1, tmf, P, sms, st));
      else CUDA_TRY(launch_grouped_tc(1, tmf, P, sms, st));
    }
    // dW_r[:d] partials, one per sample: x_norm[b]^T dl[b] (both MN-major), TMA-stored
    {
      BwdParams P;
      memset(&P, 0, sizeof(P));
      TmapSetBwd tmr;
      memset(&tmr, 0, sizeof(tmr));
      P.bank[0] = BwdBank{p->x_norm, dd, w.dl16, nullptr, E, nullptr, w.part, nullptr, 0, dd, E, 0,
                          1 << 30, (E + tc_bwd_bn(BWD_WR) - 1) / tc_bwd_bn(BWD_WR), (dd + 127) / 128};
      P.bank[1] = P.bank[0];
      int64_t tiles = 0;
      for (int b = 0; b < (int)d->B; ++b) {
        P.seg_row0[b] = (int)(b * d->S);
        P.seg_rows[b] = (int)d->S;
        P.seg_expert[b] = b;
        P.seg_bank[b] = 0;
        P.seg_tile0[b] = (int)tiles;
        tiles += (int64_t)P.bank[0].ntm * P.bank[0].ntn;
      }
      P.nseg = (int)d->B;
      P.seg_tile0[P.nseg] = P.total_tiles = (int)tiles;
      NIMG_TRY(map_3d(&tmr.a[0], p->x_norm, d->B, d->S, dd, 64));
      NIMG_TRY(map_3d(&tmr.b[0], w.dl16, d->B, d->S, E, 64));
      NIMG_TRY(map_3d_f32_out(&tmr.o[0], w.part, d->B, dd, E));
      tmr.a[1] = tmr.a[0]; tmr.b[1] = tmr.b[0]; tmr.b3[0] = tmr.b3[1] = tmr.b[0];
      tmr.o3[0] = tmr.o[0]; tmr.o[1] = tmr.o3[1] = tmr.o[0];
      CUDA_TRY(launch_grouped_tc_bwd(BWD_WR, tmr, P, sms, st));
    }
    nchunks = (int)d->B;
  } else {
    CUDA_TRY(launch_router_bwd_simt(bf, p->x_norm, w_r, w.dlogits, g->g_x_norm, w.part, T, dd, E,
                                    st, &nchunks));
  }
  CUDA_TRY(launch_router_bwd_fold(w.dlogits, t_emb, w_r, w.part, nchunks, w.colsum, g->g_w_r,
                                  g->g_t_emb, (int)d->B, (int)d->S, dd, E, st));
  mark(1, st);
  const void* dys = tc ? g->g_out : w.dy_s;
  TmapSetBwd tm;
  // 3. dH = SwiGLU'(dY W2)
  {
    BwdParams P;
    memset(&P, 0, sizeof(P));
    memset(&tm, 0, sizeof(tm));
    P.bank[0] = BwdBank{w.dy_r, dd, p->w2, nullptr, 0, ts.h_r, w.dh_r, nullptr, 2 * (int64_t)h, 0, h, dd, h, 0, 0};
    P.bank[1] = BwdBank{dys, dd, p->sw2, nullptr, 0, ts.h_s, w.dh_s, nullptr, 2 * (int64_t)hs, 0, hs, dd, hs, 0, 0};
    if (tc) {
      NIMG_TRY(map_2d(&tm.a[0], w.dy_r, R, dd, 128));
      NIMG_TRY(map_3d(&tm.b[0], p->w2, E, dd, h, 64));
      NIMG_TRY(map_2d(&tm.a[1], dys, T, dd, 128));
      NIMG_TRY(map_3d(&tm.b[1], p->sw2, 1, dd, hs, 64));
      tm.b3[0] = tm.b[0]; tm.b3[1] = tm.b[1];
    }
    NIMG_TRY(bwd_grouped(BWD_D2, tc, bf, P, tm, sms, d, st));
  }
  mark(2, st);
  // 4. dW2 = dY^T pre
  {
    BwdParams P;
    memset(&P, 0, sizeof(P));
    memset(&tm, 0, sizeof(tm));
    P.bank[0] = BwdBank{w.dy_r, dd, ts.pre_r, nullptr, h, nullptr, g->g_w2, nullptr, 0, dd, h, 0, h, 0, 0};
    // (shared bank with ks > 1: the row-chunk partials, folded below)
    P.bank[1] = BwdBank{dys, dd, ts.pre_s, nullptr, hs, nullptr, ks > 1 ? (void*)w.sp2 : g->g_sw2, nullptr,
                        0, dd, hs, 0, hs, 0, 0};
    if (tc) {
      NIMG_TRY(map_3d(&tm.a[0], w.dy_r, E, rows_e, dd, 64));
      NIMG_TRY(map_3d(&tm.b[0], ts.pre_r, E, rows_e, h, 64));
      NIMG_TRY(map_3d(&tm.a[1], dys, 1, T, dd, 64));
      NIMG_TRY(map_3d(&tm.b[1], ts.pre_s, 1, T, hs, 64));
      tm.b3[0] = tm.b[0]; tm.b3[1] = tm.b[1];
      NIMG_TRY(map_3d_f32_out(&tm.o[0], g->g_w2, E, dd, h));
      if (ks > 1) NIMG_TRY(map_3d_f32_out(&tm.o[1], w.sp2, ks, dd, hs));
      else NIMG_TRY(map_3d_f32_out(&tm.o[1], g->g_sw2, 1, dd, hs));
      tm.o3[0] = tm.o[0]; tm.o3[1] = tm.o[1];
    }
    NIMG_TRY(bwd_grouped(BWD_W2, tc, false, P, tm, sms, d, st, ks));
    if (ks > 1) CUDA_TRY(launch_sum_partials(w.sp2, ks, (int64_t)dd * hs, g->g_sw2, st));
  }
  mark(3, st);
  // 5. dX = dH [W1; W3]
  {
    BwdParams P;
    memset(&P, 0, sizeof(P));
    memset(&tm, 0, sizeof(tm));
    P.bank[0] = BwdBank{w.dh_r, 2 * (int64_t)h, p->w1, p->w3, 0, nullptr, w.dx_r, nullptr, dd, 0, dd, 2 * h, h, 0, 0};
    P.bank[1] = BwdBank{w.dh_s, 2 * (int64_t)hs, p->sw1, p->sw3, 0, nullptr, w.dx_s, nullptr, dd, 0, dd, 2 * hs, hs, 0, 0};
    if (tc) {
      NIMG_TRY(map_2d(&tm.a[0], w.dh_r, R, 2 * h, 128));
      NIMG_TRY(map_3d(&tm.b[0], p->w1, E, h, dd, 64));
      NIMG_TRY(map_3d(&tm.b3[0], p->w3, E, h, dd, 64));
      NIMG_TRY(map_2d(&tm.a[1], w.dh_s, T, 2 * hs, 128));
      NIMG_TRY(map_3d(&tm.b[1], p->sw1, 1, hs, dd, 64));
      NIMG_TRY(map_3d(&tm.b3[1], p->sw3, 1, hs, dd, 64));
    }
    NIMG_TRY(bwd_grouped(BWD_D1, tc, bf, P, tm, sms, d, st));
  }
  mark(4, st);
  // 6. [dW1; dW3] = dH^T X
  {
    BwdParams P;
    memset(&P, 0, sizeof(P));
    memset(&tm, 0, sizeof(tm));
    P.bank[0] = BwdBank{w.dh_r, 2 * (int64_t)h, ts.xg, nullptr, dd, nullptr, g->g_w1, g->g_w3, 0, 2 * h, dd, 0, h, 0, 0};
    P.bank[1] = BwdBank{w.dh_s, 2 * (int64_t)hs, p->x_mod, nullptr, dd, nullptr,
                        ks > 1 ? (void*)w.sp1 : g->g_sw1, ks > 1 ? (void*)w.sp3 : g->g_sw3, 0, 2 * hs, dd, 0,
                        hs, 0, 0};
    if (tc) {
      NIMG_TRY(map_3d(&tm.a[0], w.dh_r, E, rows_e, 2 * h, 64));
      NIMG_TRY(map_3d(&tm.b[0], ts.xg, E, rows_e, dd, 64));
      NIMG_TRY(map_3d(&tm.a[1], w.dh_s, 1, T, 2 * hs, 64));
      NIMG_TRY(map_3d(&tm.b[1], p->x_mod, 1, T, dd, 64));
      tm.b3[0] = tm.b[0]; tm.b3[1] = tm.b[1];
      NIMG_TRY(map_3d_f32_out(&tm.o[0], g->g_w1, E, h, dd));
      NIMG_TRY(map_3d_f32_out(&tm.o3[0], g->g_w3, E, h, dd));
      NIMG_TRY(map_3d_f32_out(&tm.o[1], ks > 1 ? (void*)w.sp1 : (void*)g->g_sw1, ks, hs, dd));
      NIMG_TRY(map_3d_f32_out(&tm.o3[1], ks > 1 ? (void*)w.sp3 : (void*)g->g_sw3, ks, hs, dd));
    }
    NIMG_TRY(bwd_grouped(BWD_W1, tc, bf, P, tm, sms, d, st, ks));
    if (ks > 1) {
      CUDA_TRY(launch_sum_partials(w.sp1, ks, (int64_t)hs * dd, g->g_sw1, st));
      CUDA_TRY(launch_sum_partials(w.sp3, ks, (int64_t)hs * dd, g->g_sw3, st));
    }
  }
  mark(5, st);
  // 7. gather pullback: g_x_mod[t] = dX_shared[t] + sum of its routed dX rows
  CUDA_TRY(launch_combine(tc, bf, w.dx_r, w.dx_s, nullptr, ro.comb_rows, ro.comb_cnt, g->g_x_mod, T,
                          dd, E, st));
  mark(6, st);
  return NIMG_OK;
}

static size_t block_extra_bytes(const nimg_moe_desc* d) {
  return 2 * align_up((size_t)d->B * d->d * 8) + 3 * align_up((size_t)d->B * d->d * 4);
}

int nimg_moe_block_workspace_bytes(const nimg_moe_desc* d, size_t* bytes) {
  NIMG_TRY(nimg_moe_workspace_bytes(d, bytes));
  *bytes += block_extra_bytes(d);
  return NIMG_OK;
}

// The block computes x_norm itself, in the activation dtype: the router reads
// it in that dtype whatever router_dtype says. fp32 / bf16 only.
static int check_block_desc(const nimg_moe_desc* d, nimg_moe_desc* local) {
  NIMG_TRY(check_moe_desc(d));
  if (d->act_dtype == NIMG_F64)
    return fail(NIMG_ERR_CONFIG, "the fused MoE block has no f64 path (use the layer entry points)");
  *local = *d;
  local->router_dtype = d->act_dtype;
  return NIMG_OK;
}

int nimg_moe_block_forward(const nimg_moe_desc* d_in, const nimg_block_ptrs* b, int32_t layer, void* ws,
                           size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  nimg_moe_desc dl;
  NIMG_TRY(check_block_desc(d_in, &dl));
  const nimg_moe_desc* d = &dl;
  if (!b || !b->x || !b->r_attn || !b->sa_gate || !b->ff_scale || !b->ff_gate || !b->t_vec ||
      !b->h || !b->x_norm || !b->x_mod || !b->out)
    return fail(NIMG_ERR_SHAPE, "null block pointer");
  if (layer < 0) return fail(NIMG_ERR_CONFIG, "layer must be >= 0");
  size_t need = 0;
  NIMG_TRY(nimg_moe_block_workspace_bytes(d, &need));
  if (!ws || ws_bytes < need) return fail(NIMG_ERR_CONFIG, "workspace too small (%zu < %zu)", ws_bytes, need);
  const size_t bd = (size_t)d->B * d->d;
  uint8_t* w = static_cast<uint8_t*>(ws);
  double* th_sa = reinterpret_cast<double*>(w);          w += align_up(bd * 8);
  double* th_ff = reinterpret_cast<double*>(w);          w += align_up(bd * 8);
  float* onep = reinterpret_cast<float*>(w);             w += align_up(bd * 4);
  float* th_sa_f = reinterpret_cast<float*>(w);          w += align_up(bd * 4);
  float* th_ff_f = reinterpret_cast<float*>(w);          w += align_up(bd * 4);
  const bool bf = d->act_dtype == NIMG_BF16;
  // as_tensor(1/sqrt(layer+1), like=rmsnorm output): the scalar is stored in the
  // operand dtype (tensor.py:183-187)
  float scale_t = (float)(1.0 / std::sqrt((double)layer + 1.0));
  if (bf) scale_t = __bfloat162float(__float2bfloat16_rn(scale_t));
  CUDA_TRY(launch_block_modvec(b->sa_gate, b->ff_scale, b->ff_gate, th_sa, th_ff, onep, th_sa_f,
                               th_ff_f, (int64_t)bd, st));
  CUDA_TRY(launch_block_prologue(bf, b->x, b->r_attn, th_sa, th_sa_f, onep, b->h, b->x_norm,
                                 b->x_mod, d->B * d->S, (int)d->S, (int)d->d, scale_t, st));
  nimg_moe_ptrs p;
  p.x_norm = b->x_norm;
  p.x_mod = b->x_mod;
  p.t_emb = b->t_vec;
  p.w_r = b->w_r;
  p.w1 = b->w1; p.w3 = b->w3; p.w2 = b->w2;
  p.sw1 = b->sw1; p.sw3 = b->sw3; p.sw2 = b->sw2;
  p.out = b->out;
  p.route = b->route;
  return moe_forward_impl(d, &p, w, ws_bytes - (size_t)(w - static_cast<uint8_t*>(ws)), st, b->h,
                          bf ? (const void*)th_ff_f : (const void*)th_ff);
}

int nimg_moe_block_prologue_workspace_bytes(const nimg_moe_desc* d, size_t* bytes) {
  NIMG_TRY(check_moe_desc(d));
  if (!bytes) return fail(NIMG_ERR_CONFIG, "null output");
  *bytes = block_extra_bytes(d);
  return NIMG_OK;
}

int nimg_moe_block_prologue(const nimg_moe_desc* d_in, const void* x, const void* r_attn,
                            const float* sa_gate, const float* ff_scale, const float* ff_gate,
                            int32_t layer, void* h, void* x_norm, void* x_mod, void* th_ff, void* ws,
                            size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  nimg_moe_desc dl;
  NIMG_TRY(check_block_desc(d_in, &dl));
  const nimg_moe_desc* d = &dl;
  if (!x || !r_attn || !sa_gate || !ff_scale || !ff_gate || !h || !x_norm || !x_mod || !th_ff)
    return fail(NIMG_ERR_SHAPE, "null block pointer");
  if (layer < 0) return fail(NIMG_ERR_CONFIG, "layer must be >= 0");
  if (!ws || ws_bytes < block_extra_bytes(d)) return fail(NIMG_ERR_CONFIG, "workspace too small");
  const size_t bd = (size_t)d->B * d->d;
  const bool bf = d->act_dtype == NIMG_BF16;
  uint8_t* w = static_cast<uint8_t*>(ws);
  double* th_sa = reinterpret_cast<double*>(w);          w += align_up(bd * 8);
  double* th_ff_d = reinterpret_cast<double*>(w);        w += align_up(bd * 8);
  float* onep = reinterpret_cast<float*>(w);             w += align_up(bd * 4);
  float* th_sa_f = reinterpret_cast<float*>(w);          w += align_up(bd * 4);
  float* th_ff_f = reinterpret_cast<float*>(w);
  // th_ff lands in the caller's buffer in the precision of the combine epilogue
  if (bf) th_ff_f = static_cast<float*>(th_ff);
  else th_ff_d = static_cast<double*>(th_ff);
  float scale_t = (float)(1.0 / std::sqrt((double)layer + 1.0));
  if (bf) scale_t = __bfloat162float(__float2bfloat16_rn(scale_t));
  CUDA_TRY(launch_block_modvec(sa_gate, ff_scale, ff_gate, th_sa, th_ff_d, onep, th_sa_f, th_ff_f,
                               (int64_t)bd, st));
  CUDA_TRY(launch_block_prologue(bf, x, r_attn, th_sa, th_sa_f, onep, h, x_norm, x_mod, d->B * d->S,
                                 (int)d->S, (int)d->d, scale_t, st));
  return NIMG_OK;
}

int nimg_combine_residual(int64_t T, int64_t d, int64_t E, int64_t S, int32_t y_dtype,
                          int32_t out_dtype, const void* y_routed, const void* y_shared,
                          const float* gates, const int32_t* comb_rows, const int32_t* comb_cnt,
                          const void* hres, const void* th_ff, void* out, void* stream) {
  if (T < 0 || d < 1 || E < 1 || S < 1 || T % S) return fail(NIMG_ERR_SHAPE, "bad combine shape");
  if (T == 0) return NIMG_OK;
  if (!y_shared || !comb_cnt || !comb_rows || !out || !gates || !hres || !th_ff)
    return fail(NIMG_ERR_SHAPE, "null pointer");
  CUDA_TRY(launch_combine(y_dtype == NIMG_BF16, out_dtype == NIMG_BF16, y_routed, y_shared, gates,
                          comb_rows, comb_cnt, out, T, (int)d, (int)E, (cudaStream_t)stream, hres,
                          th_ff, (int)S));
  return NIMG_OK;
}

int nimg_profile_events(void* const* events, int32_t n) {
  if (n < 0 || n > 8 || (n > 0 && !events)) return fail(NIMG_ERR_CONFIG, "bad event list");
  for (int i = 0; i < n; ++i) g_events[i] = (cudaEvent_t)events[i];
  g_nevents = n;
  return NIMG_OK;
}

// ------------------------------------------------------------------ EP transport
typedef CUresult (*StreamWriteValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*StreamWaitValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

static void* driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPointByVersion(name, &p, 12000, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return p;
}

int nimg_ipc_alloc(size_t bytes, void** dev_ptr, void* handle) {
  if (!dev_ptr || !handle || bytes == 0) return fail(NIMG_ERR_CONFIG, "bad ipc_alloc arguments");
  CUDA_TRY(cudaMalloc(dev_ptr, bytes));
  CUDA_TRY(cudaMemset(*dev_ptr, 0, bytes));
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, *dev_ptr));
  static_assert(sizeof(h) == 64, "ipc handle size");
  memcpy(handle, &h, sizeof(h));
  return NIMG_OK;
}

int nimg_ipc_open(const void* handle, void** dev_ptr) {
  if (!handle || !dev_ptr) return fail(NIMG_ERR_CONFIG, "bad ipc_open arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  CUDA_TRY(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return NIMG_OK;
}

int nimg_ipc_close(void* dev_ptr) {
  CUDA_TRY(cudaIpcCloseMemHandle(dev_ptr));
  return NIMG_OK;
}

int nimg_free(void* dev_ptr) {
  CUDA_TRY(cudaFree(dev_ptr));
  return NIMG_OK;
}

int nimg_copy_async(void* dst, const void* src, size_t bytes, void* stream) {
  if (bytes == 0) return NIMG_OK;
  CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return NIMG_OK;
}

int nimg_stream_write_u32(void* dev_addr, uint32_t value, void* stream) {
  static StreamWriteValue32Fn fn = (StreamWriteValue32Fn)driver_fn("cuStreamWriteValue32");
  if (!fn) return fail(NIMG_ERR_CUDA, "cuStreamWriteValue32 unavailable");
  CUresult r = fn((CUstream)stream, (CUdeviceptr)dev_addr, value, CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) return fail(NIMG_ERR_CUDA, "cuStreamWriteValue32 failed (%d)", (int)r);
  return NIMG_OK;
}

int nimg_stream_wait_geq_u32(void* dev_addr, uint32_t value, void* stream) {
  static StreamWaitValue32Fn fn = (StreamWaitValue32Fn)driver_fn("cuStreamWaitValue32");
  if (!fn) return fail(NIMG_ERR_CUDA, "cuStreamWaitValue32 unavailable");
  CUresult r = fn((CUstream)stream, (CUdeviceptr)dev_addr, value, CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return fail(NIMG_ERR_CUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
  return NIMG_OK;
}

}  // extern "C"
