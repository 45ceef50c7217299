// Internal (C++) declarations shared by the kernel translation units and the
// C-ABI layer. Nothing here is part of the public ABI (include/nimg_moe.h).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace nimg {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device and per
// kernel: a process that drives several GPUs must set it on each of them.
cudaError_t set_max_dyn_smem(const void* kernel, int bytes);
template <typename K>
inline cudaError_t set_max_dyn_smem(K* kernel, int bytes) {
  return set_max_dyn_smem(reinterpret_cast<const void*>(kernel), bytes);
}

typedef uint16_t bf16_raw;   // bf16 storage in host-visible signatures
// elements of the row-blocked h1 | h3 buffer (hblk_off in common.cuh)
inline int64_t hblk_elems(int64_t rows, int64_t h) { return (rows + 127) / 128 * 128 * 2 * h; }

constexpr int kMaxSeg = 264;  // routed segments + shared; EP: R * E/R + 1

// One weight bank of a grouped launch: bank 0 = routed experts (3-D weights
// [E, N, K]), bank 1 = the shared expert (3-D with E = 1).
constexpr int kSplit3Out = 1, kF32Out = 2;
struct GBank {
  void* out;       // output rows (bank-local row index), row stride out_ld elements
  int64_t out_ld;
  int K;           // reduction length (d for GEMM1, h for GEMM2)
  int N;           // output columns (h for GEMM1, d for GEMM2)
  int ntn;         // N tiles
  int flags;       // output form: 0 bf16; kSplit3Out (GEMM1, fp32 mode): bf16 [hi | hi | lo]
                   // rows of 3N (out_ld = 3N); kF32Out (GEMM2, fp32 mode): fp32 rows
  const int32_t* a_idx;  // GEMM1 only: A row r is source row a_idx[r]; null = contiguous
  const void* a_src;     // gather source rows (bf16, K elements per row) when a_idx != null
  void* h_out;           // GEMM1, training forward: h1 | h3 rows (2N bf16 per row) or null
};

// Segments [0, nseg0) use bank 0, [nseg0, nseg) bank 1. Segment i covers rows
// [seg_row0[i], seg_row0[i] + seg_rows[i]) of its bank's A / out tensors and
// multiplies them by expert seg_expert[i] of that bank.
// Background gather (GEMM1, 1-GPU layer): extra warps of the GEMM copy the
// routed rows bg_dst[r] = bg_src[bg_idx[r]] in 32-row sub-blocks while the
// shared expert's tiles (scheduled first) run, and publish bg_flags[sub] = 1;
// a routed tile's TMA producer waits for the flags of its rows.
struct BgGather {
  const void* src;       // x_mod rows
  const int32_t* idx;    // token_flat
  void* dst;             // gathered rows (the routed bank's A operand)
  int* flags;            // one per 32-row sub-block + the claim counter, zeroed by gate_norm
  int rows, row_bytes;   // null src: off
  int row_off;           // gathered row of the routed bank's row 0 (flag index base)
  int chunk_rows;        // > 0: chunk_done[c] += 1 per finished sub-block overlapping
  unsigned* chunk_done;  //   rows [c chunk_rows, (c+1) chunk_rows) (expert parallel:
                         //   the dispatch copy of chunk c waits on it)
};
struct GroupedParams {
  GBank bank[2];
  BgGather bg;
  int nseg0, nseg, total_tiles, pad_;
  int seg_tile0[kMaxSeg + 1];
  int seg_row0[kMaxSeg];
  int seg_rows[kMaxSeg];
  int seg_expert[kMaxSeg];
};

struct __align__(64) TmapSet {
  CUtensorMap a[2];   // A operand per bank: 2-D [rows, K]
  CUtensorMap b[2];   // B operand per bank: 3-D [E, N, K] (W1 for GEMM1, W2 for GEMM2)
  CUtensorMap b3[2];  // GEMM1 only: W3
};

// SIMT (CUDA-core) grouped path: fp32 parity mode and shapes the TMA path
// cannot take. Pointers instead of tensor maps.
struct SimtBank {
  const void* a;     // [rows, K] activations (T_IN)
  int64_t a_ld;
  const void* w;     // [E, N, K]   (W1 or W2)
  const void* w3;    // [E, N, K]   (W3, GEMM1 only)
  void* out;         // [rows, N] fp32 (f64 in the f64 storage mode)
  int64_t out_ld;
  int K, N, ntn, pad_;
  float* h_out;      // GEMM1, training forward: h1 | h3 rows (2N fp32 per row) or null
};
struct SimtParams {
  SimtBank bank[2];
  int nseg0, nseg, total_tiles, pad_;
  int seg_tile0[kMaxSeg + 1];
  int seg_row0[kMaxSeg];
  int seg_rows[kMaxSeg];
  int seg_expert[kMaxSeg];
};

// Backward grouped GEMMs (backward_kernels.cu SIMT, grouped_gemm_bwd_sm100.cu
// tcgen05). Modes: see backward_kernels.cu.
enum { BWD_D2 = 0, BWD_D1 = 1, BWD_W2 = 2, BWD_W1 = 3, BWD_WR = 4 };
struct BwdBank {
  const void* a;     // D2: dY rows [rows, K=d]; D1: dH rows [rows, 2h]; W2: dY rows [rows, M=d];
                     // W1: dH rows [rows, M=2h]
  int64_t a_ld;
  const void* b;     // D2: W2 [E][d][h]; D1: W1 [E][h][d]; W modes: row operand (pre / X) [rows, N]
  const void* b3;    // D1: W3 [E][h][d]
  int64_t b_ld;      // W modes: row stride of b
  const void* aux;   // D2: H rows (h1 | h3, 2h per row)
  void* out;         // D2: dH rows (2h); D1: dX rows (out_ld); W2: dW2 [E][d][h]; W1: dW1 [E][h][d]
  void* out3;        // W1: dW3 [E][h][d]
  int64_t out_ld;
  int M, N, K, h;    // D modes: K (= d or 2h), N; W modes: M, N (K = segment rows)
  int ntn, ntm;
};
struct BwdParams {
  BwdBank bank[2];
  int nseg, total_tiles;
  int seg_tile0[kMaxSeg + 1];
  int seg_row0[kMaxSeg];
  int seg_rows[kMaxSeg];
  int seg_expert[kMaxSeg];
  int seg_bank[kMaxSeg];
};
int simt_bwd_bm();
int simt_bwd_bn();
cudaError_t launch_grouped_simt_bwd(int mode, bool b_bf16, const BwdParams& p, cudaStream_t s);
// tcgen05 backward GEMMs (bf16 operands, MN-major where the pullback needs a
// transposed operand): tile rows 128, N tile tc_bwd_bn(mode).
int tc_bwd_bn(int mode);
int tc_bwd_tile_rows(int mode);   // 256 for the CTA-pair kernels, else 128
// Backward tensor maps: operands as TmapSet, plus the weight-gradient outputs
// (fp32 [E][M][N], stored by TMA from a swizzled staging tile).
struct __align__(64) TmapSetBwd {
  CUtensorMap a[2], b[2], b3[2];
  CUtensorMap o[2], o3[2];   // W modes: dW2 / dW1, dW3 per bank
};
cudaError_t launch_grouped_tc_bwd(int mode, const TmapSetBwd& tm, const BwdParams& p, int num_sms,
                                  cudaStream_t stream);
// dl16 != null: also a bf16 copy of dlogits (A / B operand of the tcgen05 router pullback)
cudaError_t launch_combine_bwd(bool g_bf16, bool y_bf16, bool dy_bf16, const void* g_out,
                               const void* yr, const float* gates, const float* gate_raw,
                               const int32_t* comb_rows, const int32_t* comb_cnt,
                               const float* logits, void* dyr, void* dys, float* dlogits,
                               bf16_raw* dl16, int64_t T, int d, int E, int rows_per_expert,
                               float eps32, float alpha32, cudaStream_t s);
size_t router_bwd_part_bytes(int64_t T, int d, int E);
// CUDA-core router pullback: dx_norm and the token-chunk partials of dW_r[:d]
cudaError_t launch_router_bwd_simt(bool x_bf16, const void* x_norm, const float* w_r,
                                   const float* dl, void* dx, float* part, int64_t T, int d, int E,
                                   cudaStream_t s, int* nchunks);
// sum_s dl -> colsum; fold the partials (fixed order) into g_w_r[:d]; g_w_r[d:], g_t_emb
cudaError_t launch_router_bwd_fold(const float* dl, const float* t_emb, const float* w_r,
                                   const float* part, int nchunks, float* colsum, float* g_wr,
                                   float* g_t, int B, int S, int d, int E, cudaStream_t s);
cudaError_t launch_f32_to_bf16(const float* src, bf16_raw* dst, int64_t n, cudaStream_t s);
cudaError_t launch_sum_partials(const float* part, int ks, int64_t n, float* out, cudaStream_t s);

// Launch with programmatic stream serialization (PDL) unless NIMG_PDL=0. The
// kernel must call pdl_wait() before touching global memory (common.cuh).
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

int tc_bn_out(int mode);
int tc_pair_rows();
// CTA-pair (cta_group::2) variant: 256-row tiles, B split across the pair.
cudaError_t launch_grouped_tc_pair(int mode, const TmapSet& tm, const GroupedParams& p, int num_sms,
                                   cudaStream_t stream);
int tc_b_box(int mode);
cudaError_t launch_grouped_tc(int mode, const TmapSet& tm, const GroupedParams& p, int num_sms,
                              cudaStream_t stream);
// in_bf16: activations/weights dtype (bf16 vs fp32); GEMM2 reads fp32 `pre`.
int simt_bm();
int simt_bn();
cudaError_t launch_grouped_simt(int mode, bool in_bf16, const SimtParams& p, cudaStream_t stream,
                                bool f64 = false);

// fp32 mode on the bf16 tensor cores (split_kernels.cu): rows -> bf16 [hi|hi|lo]
// (pattern 0, activations) or [hi|lo|hi] (pattern 1, weights), K' = 3K
cudaError_t launch_split3_rows(const float* src, const int32_t* idx, void* dst, int64_t rows, int K,
                               int pattern, cudaStream_t s);

// f64 storage mode (f64_kernels.cu): routing and combine with every value in f64
cudaError_t launch_route_f64(const double* x_norm, const double* t_emb, const double* w_r,
                             double* logits, double* scores_bes, int32_t* token_flat,
                             double* gate_raw, double* gates, int32_t* comb_rows,
                             int32_t* comb_cnt, int16_t* slot_of, int B, int S, int d, int E,
                             int cap, double eps, double alpha, cudaStream_t st);
cudaError_t launch_combine_f64(const double* yr, const double* ys, const double* gates,
                               const int32_t* comb_rows, const int32_t* comb_cnt, double* out,
                               int64_t T, int d, int E, cudaStream_t st);

// routing / data-movement kernels (route_kernels.cu)
// router prep (t-half bias + f64 copy of W_r[:d]) and FP64 scores kernel.
// E <= 64 (DMMA): one prep kernel writes tb and wd (no counters / part, may
// be null); the scores kernel is its PDL secondary.
// E > 64 (DFMA): counters = B unsigned per-sample completion counters,
// 0xFFFFFFFF on entry (re-armed by the kernel).
bool router_uses_dmma(int E);
cudaError_t launch_router(bool x_bf16, const void* x_norm, const float* t_emb, const float* w_r,
                          double* tb, double* part, unsigned* counter, double* wd, float* logits,
                          float* scores_bes, int B, int S, int d, int E, cudaStream_t s);
size_t router_wd_bytes(int d, int E);
// Exact INT8 tensor-core router (router_i8.cu): bf16 x_norm, E == 64, d % 128 == 0.
// NIMG_ROUTER=dmma forces the FP64 router.
bool router_i8_eligible(bool x_bf16, int d, int E, const void* x_norm, const void* w_r);
size_t router_i8_ws_bytes(int64_t T, int d);
// spans the INT8 router's prep kernel zeroes on the way (n = 0: none)
struct ZeroSpans {
  unsigned long long* p64 = nullptr;
  int64_t n64 = 0;
  int* p32 = nullptr;
  int64_t n32 = 0;
};
cudaError_t launch_router_i8(const void* x_norm, const float* t_emb, const float* w_r, double* part,
                             void* i8ws, float* logits, float* scores_bes, int B, int S, int d,
                             cudaStream_t s, ZeroSpans zs = ZeroSpans{});
size_t router_part_bytes(int B, int d, int E);
// tokmask (E <= 64, block select path): each selected (token, e) also sets bit
// e of the token's mask and writes its (routed row, raw score) into the
// token-major tokent (the combine then forms the gates itself, GateFuse)
cudaError_t launch_ec_select(const float* scores_bes, int32_t* token_flat, float* gate_raw,
                             int16_t* slot_of, int B, int S, int E, int cap, cudaStream_t s,
                             int* cursor = nullptr, unsigned long long* tokmask = nullptr,
                             int2* tokent = nullptr);
bool select_blk_path(int S);
// Gates formed inside the combine (1-GPU inference): token t's selecting experts
// are the set bits of tokmask[t] (ascending), their rows / raw scores come from
// tokent, the gate chain is gate_tile_kernel's and every gate is also
// written to gates_out (the routing output)
struct GateFuse {
  const unsigned long long* tokmask;
  const int2* tokent;      // [T][E]: (routed row, raw score bits) of (token, e), valid where the mask bit is set
  float* gates_out;
  float eps32, alpha32;
};
// Token-ordered expert outputs for the 1-GPU combine (gate_tile_kernel):
// null tok_off = off
struct TokOrder {
  int* tok_off;
  int* row_map;
  float* gate_tok;
  int* cursor;
};
bool gate_tok_supported();   // the gate kernel that fills TokOrder is in use
cudaError_t launch_gate_norm(const float* scores_bes, const int16_t* slot_of, float* gates,
                             int32_t* comb_rows, int32_t* comb_cnt, int B, int S, int E, int cap,
                             float gate_eps, float gate_scale, cudaStream_t s, int* bg_flags = nullptr,
                             int n_bg_flags = 0, TokOrder tko = TokOrder{nullptr, nullptr, nullptr, nullptr});
// chunk_done[c] += number of 32-row sub-blocks of [0, rows) overlapping chunk c
cudaError_t launch_bg_count(int rows, int chunk_rows, unsigned* chunk_done, cudaStream_t s);
cudaError_t launch_gather_rows(const void* src, int64_t row_bytes, const int32_t* idx,
                               int64_t n_idx, void* dst, cudaStream_t s);
// out[t] = fp32(fp32(sum_k fp32(Y[rows[k][t]] * gate)) + shared[t]) -- see combine kernel.
// hres != null: out[t] = h[t] + th_gate[b] * (that) instead (backbone.py:606);
// th_gate is double* for fp32 output (f64 chain), float* for bf16 output.
cudaError_t launch_combine(bool y_bf16, bool out_bf16, const void* y_routed, const void* y_shared,
                           const float* gates, const int32_t* comb_rows, const int32_t* comb_cnt,
                           void* out, int64_t T, int d, int E, cudaStream_t s,
                           const void* hres = nullptr, const void* th_gate = nullptr, int S = 1,
                           const int32_t* tok_off = nullptr, const GateFuse* gf = nullptr);
// backbone MoE branch prologue (block_kernels.cu)
cudaError_t launch_block_modvec(const float* sa_gate, const float* ff_scale, const float* ff_gate,
                                double* th_sa, double* th_ff, float* onep, float* th_sa_f,
                                float* th_ff_f, int64_t n, cudaStream_t s);
cudaError_t launch_block_prologue(bool bf, const void* x, const void* r_attn, const double* th_sa,
                                  const float* th_sa_f, const float* onep, void* h, void* xn,
                                  void* xm, int64_t T, int S, int d, float scale_t, cudaStream_t s);

// denoising-step stack helpers (stack_kernels.cu). mode 0: m = LN(x)(1+scale)
// (+ shift); 1: h = x + th*r, m = LN(h)(1+scale); 2: h = x + th*r.
cudaError_t launch_row_modulate(int mode, bool bf, const void* x, const void* r, const float* th,
                                const float* scale, const float* shift, void* h, void* m,
                                int64_t rows, int S, int d, float eps, cudaStream_t s);
cudaError_t launch_qk_norm_rope(bool bf, const void* x, int64_t xs, const float* cs, const float* sn,
                                void* out, int64_t rows, int S, int H, int dh, float eps,
                                cudaStream_t s);

}  // namespace nimg
