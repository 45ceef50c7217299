/*
 * nimg_moe.h -- C ABI of the B200 (sm_100a) expert-choice MoE layer.
 *
 * Drop-in boundary for the reference's MoE operator API
 * (/root/reference/pkg/src/nimg). The reference is pure Python with no FFI;
 * each entry point below replaces one reference function, cited file:line.
 * The Python mirror (paper_2604_12163_b200/{router,moe}.py) binds these with
 * ctypes -- see INTEGRATION.md.
 *
 * Conventions
 *  - Plain C: pointers, sizes, host scalars. No torch / C++ types.
 *  - All tensor pointers are DEVICE pointers (CUDA global memory), dense and
 *    row-major, 16-byte aligned. Host arrays are marked "host".
 *  - `stream` is a cudaStream_t passed as void*. Every call only enqueues work
 *    on that stream: no allocation, no host synchronisation, capturable in a
 *    CUDA graph. The caller owns every buffer, including the workspace.
 *  - Return 0 on success, else an NIMG_ERR_* code; nimg_last_error() returns a
 *    thread-local message. Codes map to the reference's exceptions:
 *    NIMG_ERR_SHAPE -> nimg.tensor.ShapeError (tensor.py:19-20),
 *    NIMG_ERR_CONFIG -> nimg.router.ConfigError (router.py:22-23).
 *  - dtypes: NIMG_F32 = float32, NIMG_BF16 = bfloat16, NIMG_F64 = float64.
 *    In the fp32 / bf16 modes the router weight, the timestep embedding and
 *    every routing output are float32 (routing stays bit-exact with the
 *    reference's fp32 mode). NIMG_F64 is the reference's float64 storage mode
 *    (tensor.py:39-47; the backbone runs its MoE on f64 inputs,
 *    backbone.py:259-261): every input, weight, routing output and the layer
 *    output are float64, and no intermediate is rounded to fp32.
 *  - ABI version 2 (nimg_abi_version): nimg_moe_desc.router_dtype replaced the
 *    v1 `reserved` field and the f64 gate parameters were appended; routing
 *    value pointers became void* (their element type follows act_dtype).
 */
#ifndef NIMG_MOE_H_
#define NIMG_MOE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NIMG_OK 0
#define NIMG_ERR_SHAPE 1
#define NIMG_ERR_CONFIG 2
#define NIMG_ERR_CUDA 3

#define NIMG_F32 0
#define NIMG_BF16 1
#define NIMG_F64 2

#define NIMG_PATH_TCGEN05 0 /* bf16 tcgen05/TMEM/TMA grouped GEMM */
#define NIMG_PATH_SIMT 1    /* fp32-accumulate CUDA-core grouped GEMM */

/* One MoE layer problem. Mirrors RouterConfig (router.py:36-56) + ExpertBank
 * shapes (moe.py:73-94). cap must equal capacity_for(S, E, C). */
typedef struct nimg_moe_desc {
  int64_t B, S, d, E, cap, h, h_shared;
  float gate_scale; /* RouterConfig.gate_scale (alpha) */
  float gate_eps;   /* RouterConfig.gate_eps */
  int32_t act_dtype;    /* x_mod, expert weights and out */
  int32_t router_dtype; /* x_norm (the router input). NIMG_F32 or NIMG_BF16 in the
                           fp32 / bf16 modes -- routing is computed on x_norm's own
                           values, as the reference does (router.py:120-122) --
                           and NIMG_F64 iff act_dtype is NIMG_F64. The training
                           entry points require router_dtype == act_dtype. */
  double gate_scale_f64; /* RouterConfig.gate_scale / gate_eps as Python floats: */
  double gate_eps_f64;   /* used (unrounded) in the NIMG_F64 mode             */
} nimg_moe_desc;

/* Routing results (router.py:104-162). Expert-major flat order (e, b, slot)
 * of length E*B*cap, as the reference's routing["token_flat"]. */
/* "fp32" below is float64 in the NIMG_F64 mode. */
typedef struct nimg_route_out {
  void* logits;        /* (B,S,E) fp32        routing["logits"]              */
  void* scores_bes;    /* (B,E,S) fp32        softmax scores, expert-major   */
  int32_t* token_flat; /* (E*B*cap) int32     routing["token_flat"]          */
  void* gate_raw;      /* (E*B*cap) fp32      RouterDecision.affinity         */
  void* gates;         /* (E*B*cap) fp32      routing["gates"]               */
  int32_t* comb_rows;  /* (B*S,E) int32       per token: routed rows, expert-ascending */
  int32_t* comb_cnt;   /* (B*S) int32         number of experts that picked the token */
} nimg_route_out;

typedef struct nimg_moe_ptrs {
  const void* x_norm; /* (B,S,d) router_dtype: router input (unmodulated) */
  const void* x_mod;  /* (B,S,d) act: expert input (modulated)     */
  const void* t_emb;  /* (B,d)   fp32 (f64 in the NIMG_F64 mode)    */
  const void* w_r;    /* (2d,E)  fp32 (f64 in the NIMG_F64 mode)    */
  const void *w1, *w3, *w2;    /* (E,h,d), (E,h,d), (E,d,h) act     */
  const void *sw1, *sw3, *sw2; /* (hs,d), (hs,d), (d,hs) act        */
  void* out;          /* (B,S,d) act                                */
  nimg_route_out route; /* all members required                     */
} nimg_moe_ptrs;

/* Expert FFN over explicit segments (grouped_forward, moe.py:115-135) plus an
 * optional shared-expert bank over other rows (moe.py:160). */
typedef struct nimg_ffn_desc {
  int64_t n_rows;        /* rows of x_routed / y_routed            */
  int64_t n_shared_rows; /* rows of x_shared / y_shared, 0 = none  */
  int64_t d, h, h_shared;
  int64_t n_experts;     /* experts in the w1/w3/w2 tensors        */
  int32_t act_dtype;
  int32_t nseg;          /* routed segments, <= 256                */
} nimg_ffn_desc;

/* ------------------------------------------------------------------ misc */
const char* nimg_last_error(void);
int nimg_abi_version(void);
/* Number of SMs the persistent kernels size their grid by (device of stream). */
int nimg_device_sms(int* sms);

/* Profiling hook: up to 8 cudaEvent_t (as void*) recorded on the launch stream
 * by nimg_moe_forward at its stage boundaries: [0] start, [1] routed,
 * [2] gathered, [3] GEMM1 done, [4] GEMM2 done, [5] combined; by
 * nimg_moe_backward: [0] start, [1] combine + router pullbacks, [2] dH,
 * [3] dW2, [4] dX, [5] dW1/dW3, [6] g_x_mod. n = 0 turns it off.
 * Thread-local; no reference counterpart (instrumentation only). */
int nimg_profile_events(void* const* events, int32_t n);

/* router.py:70-74  capacity_for(S, E, C) = min(ceil(C*S/E), S) */
int nimg_capacity_for(int64_t S, int64_t E, double C, int64_t* cap);

/* ------------------------------------------------------------------ layer */
/* Workspace for nimg_moe_forward (bytes, 256-B aligned regions). */
int nimg_moe_workspace_bytes(const nimg_moe_desc* desc, size_t* bytes);
/* moe.py:138-164  moe_forward: route on x_norm/t_emb, experts on x_mod,
 * weighted combine + shared expert -> out. */
int nimg_moe_forward(const nimg_moe_desc* desc, const nimg_moe_ptrs* ptrs, void* ws,
                     size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------ training
 * The layer's backward: what reference backward(tape, loss) (tensor.py:590-628)
 * accumulates through moe_forward (moe.py:138-164) -- the swiglu pullback
 * (moe.py:53-62), the gate chain and softmax pullbacks (router.py:137-143,
 * tensor.py:467-477) and the router matmul pullback (tensor.py:280-296).
 *
 * nimg_moe_forward_train is nimg_moe_forward that also keeps, in a
 * caller-owned state blob, what the pullback needs (gathered rows, h1 | h3,
 * pre, routed expert outputs). The route outputs (ptrs->route) must stay
 * alive until nimg_moe_backward. bf16 layers with d, h, h_shared multiples
 * of 64 run the tcgen05 path (bf16 intermediates); all others the CUDA-core
 * path (fp32 intermediates). */
typedef struct nimg_moe_grads {
  const void* g_out; /* (B,S,d) act: d loss / d out                       */
  void* g_x_norm;    /* (B,S,d) act                                        */
  void* g_x_mod;     /* (B,S,d) act                                        */
  float* g_t_emb;    /* (B,d)  fp32                                        */
  float* g_w_r;      /* (2d,E) fp32                                        */
  float *g_w1, *g_w3, *g_w2;    /* (E,h,d), (E,h,d), (E,d,h) fp32        */
  float *g_sw1, *g_sw3, *g_sw2; /* (hs,d), (hs,d), (d,hs) fp32            */
} nimg_moe_grads;
int nimg_moe_train_state_bytes(const nimg_moe_desc* desc, size_t* bytes);
int nimg_moe_forward_train(const nimg_moe_desc* desc, const nimg_moe_ptrs* ptrs, void* state,
                           size_t state_bytes, void* ws, size_t ws_bytes, void* stream);
int nimg_moe_backward_workspace_bytes(const nimg_moe_desc* desc, size_t* bytes);
/* ptrs: the same inputs / routing buffers as the forward (out unused). Writes
 * every gradient in full (no accumulation into existing values). */
int nimg_moe_backward(const nimg_moe_desc* desc, const nimg_moe_ptrs* ptrs, const void* state,
                      size_t state_bytes, const nimg_moe_grads* grads, void* ws, size_t ws_bytes,
                      void* stream);

/* The backbone's MoE branch around the layer (backbone.py:583-606):
 *   h = x + tanh(sa_gate) r_attn;  x_norm = rmsnorm(h) / sqrt(layer+1);
 *   x_mod = x_norm (1 + ff_scale);  moe = moe_forward(h, x_norm, x_mod, t_vec);
 *   out = h + tanh(ff_gate) moe.
 * The prologue is one fused pass; the gated residual is the combine's epilogue. */
typedef struct nimg_block_ptrs {
  const void* x;         /* (B,S,d) act: residual stream entering the branch */
  const void* r_attn;    /* (B,S,d) act: attention output */
  const float* sa_gate;  /* (B,d) fp32 */
  const float* ff_scale; /* (B,d) fp32 */
  const float* ff_gate;  /* (B,d) fp32 */
  const float* t_vec;    /* (B,d) fp32: router timestep input */
  const float* w_r;      /* (2d,E) fp32 */
  const void *w1, *w3, *w2, *sw1, *sw3, *sw2;
  void* h;               /* (B,S,d) act out */
  void* x_norm;          /* (B,S,d) act out */
  void* x_mod;           /* (B,S,d) act out */
  void* out;             /* (B,S,d) act out: h + tanh(ff_gate) * moe */
  nimg_route_out route;
} nimg_block_ptrs;
int nimg_moe_block_workspace_bytes(const nimg_moe_desc* desc, size_t* bytes);
int nimg_moe_block_forward(const nimg_moe_desc* desc, const nimg_block_ptrs* ptrs, int32_t layer,
                           void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------ stages */
int nimg_route_workspace_bytes(const nimg_moe_desc* desc, size_t* bytes);
/* router.py:104-162  route_full (logits, softmax, per-(b,e) top-cap,
 * expert-major token_flat, renormalised gates) + combine tables. */
int nimg_route(const nimg_moe_desc* desc, const void* x_norm, const void* t_emb,
               const void* w_r, const nimg_route_out* out, void* ws, size_t ws_bytes,
               void* stream);

/* nimg_route for a routing that nimg_combine_routed consumes: router.py:137-143
 * (the gates) is left to the combine, so no gate kernel runs and gates /
 * comb_rows / comb_cnt are not written here; per-token expert masks and
 * (row, raw score) entries stay in ws, which must live until the combine.
 * Applies when nimg_route_fusable() returns 1 (E <= 64, S <= 4096, fp32 / bf16). */
int nimg_route_fusable(const nimg_moe_desc* desc);
int nimg_route_for_combine(const nimg_moe_desc* desc, const void* x_norm, const void* t_emb,
                           const void* w_r, const nimg_route_out* out, void* ws, size_t ws_bytes,
                           void* stream);
/* nimg_combine (hres == NULL) or nimg_combine_residual for a routing made by
 * nimg_route_for_combine with route_ws: the combine forms every gate
 * (router.py:137-143, the same bits as nimg_route) and also writes it to gates
 * (E*B*cap, the routing output). T = B*S of desc. */
int nimg_combine_routed(const nimg_moe_desc* desc, const void* route_ws, int32_t y_dtype,
                        int32_t out_dtype, const void* y_routed, const void* y_shared, void* gates,
                        const void* hres, const void* th_ff, void* out, void* stream);

/* tensor.py:348-363  gather_rows: dst[i,:] = src[idx[i],:] (row_bytes each) */
int nimg_gather_rows(const void* src, int64_t n_src_rows, int64_t row_bytes, const int32_t* idx,
                     int64_t n_idx, void* dst, void* stream);

/* Which GEMM path and which y dtype nimg_expert_ffn uses for this problem. */
int nimg_ffn_path(const nimg_ffn_desc* desc, int32_t* path, int32_t* y_dtype);
int nimg_ffn_workspace_bytes(const nimg_ffn_desc* desc, size_t* bytes);
/* moe.py:115-135 grouped_forward / moe.py:31-51 swiglu: for each segment i,
 * rows [seg_offsets[i], seg_offsets[i+1]) of x_routed go through expert
 * seg_expert[i] (host arrays). If n_shared_rows > 0, x_shared goes through
 * the shared expert. y dtype: see nimg_ffn_path.
 * seg_expert[i] == -1 marks a skip segment: its rows are neither read nor
 * written (the expert-parallel path runs a subset of the received chunks in
 * one grouped launch over the whole receive buffer). */
int nimg_expert_ffn(const nimg_ffn_desc* desc, const int64_t* seg_offsets,
                    const int32_t* seg_expert, const void* x_routed, const void* w1,
                    const void* w3, const void* w2, void* y_routed, const void* x_shared,
                    const void* sw1, const void* sw3, const void* sw2, void* y_shared, void* ws,
                    size_t ws_bytes, void* stream);

/* The routed-row gather (moe.py:152-153) run by background warps of the
 * GEMM1 launch of nimg_expert_ffn_gather (expert parallel: the rank-local
 * gather of every chunk, fused into the first grouped launch):
 * dst[r] = src[idx[r]] for r < rows (row_bytes each). The launch's routed
 * bank reads rows [row_off, row_off + n_rows) of dst (x_routed must be
 * dst + row_off * row_bytes); its tiles wait on the sub-block flags. flags:
 * nimg_route_bg_flags() of the nimg_route call that produced idx (it zeroes
 * them). chunk_rows > 0: every finished 32-row sub-block adds 1 to
 * chunk_done[c] of each chunk c (rows [c chunk_rows, (c+1) chunk_rows)) it
 * overlaps -- persistent counters the caller owns and never resets; a copy of
 * chunk c may start once the counter reached its running total (stream wait).
 * If the launch cannot fuse the gather (not the CTA-pair tcgen05 path, or no
 * shared bank) the library runs the gather kernel first and counts the same. */
typedef struct nimg_bg_gather {
  const void* src;
  const int32_t* idx;
  void* dst;
  int32_t* flags;
  uint32_t* chunk_done;
  int32_t rows, row_bytes, row_off, chunk_rows;
} nimg_bg_gather;
int nimg_route_bg_flags(const nimg_moe_desc* desc, void* route_ws, int32_t** flags);
int nimg_expert_ffn_gather(const nimg_ffn_desc* desc, const int64_t* seg_offsets,
                           const int32_t* seg_expert, const void* x_routed, const void* w1,
                           const void* w3, const void* w2, void* y_routed, const void* x_shared,
                           const void* sw1, const void* sw3, const void* sw2, void* y_shared,
                           void* ws, size_t ws_bytes, const nimg_bg_gather* gather, void* stream);

/* moe.py:156-161 + tensor.py:366-378: out[t] = round(f64(fp32(sum_k
 * fp32(y_routed[rows_k] * gates[rows_k]))) + f64(y_shared[t])), experts in
 * ascending order (deterministic; same bits for any expert-parallel split). */
int nimg_combine(int64_t T, int64_t d, int64_t E, int32_t y_dtype, int32_t out_dtype,
                 const void* y_routed, const void* y_shared, const void* gates,
                 const int32_t* comb_rows, const int32_t* comb_cnt, void* out, void* stream);

/* backbone.py:584-589 alone (the expert-parallel block runs the layer between
 * this and nimg_combine_residual): h, x_norm, x_mod exactly as
 * nimg_moe_block_forward computes them, and th_ff = tanh(ff_gate) (B, d) in
 * the combine epilogue's precision (double for an fp32 layer, float for bf16). */
int nimg_moe_block_prologue_workspace_bytes(const nimg_moe_desc* desc, size_t* bytes);
int nimg_moe_block_prologue(const nimg_moe_desc* desc, const void* x, const void* r_attn,
                            const float* sa_gate, const float* ff_scale, const float* ff_gate,
                            int32_t layer, void* h, void* x_norm, void* x_mod, void* th_ff, void* ws,
                            size_t ws_bytes, void* stream);
/* nimg_combine with backbone.py:606 in its epilogue:
 * out[t] = h[t] + th_ff[t / S] * combined[t] (th_ff from nimg_moe_block_prologue). */
int nimg_combine_residual(int64_t T, int64_t d, int64_t E, int64_t S, int32_t y_dtype,
                          int32_t out_dtype, const void* y_routed, const void* y_shared,
                          const float* gates, const int32_t* comb_rows, const int32_t* comb_cnt,
                          const void* hres, const void* th_ff, void* out, void* stream);

/* ------------------------------------------------------------------ denoising-step stack
 * Fused element-wise chains around attention and the dense FFN of the
 * backbone (backbone.py:42-121, :128-182, tensor.py:518-531), used by the
 * stack (dit.py) in fp32 / bf16. Rows are (B*S) tokens of width d; per-sample
 * vectors are (B, d) fp32; th = tanh(gate). d * elt must be a multiple of 16 B,
 * pointers 16-B aligned. */
/* out = LayerNorm(x) * (1 + scale[b]) (+ shift[b] if shift != NULL) */
int nimg_ln_modulate(int64_t rows, int64_t S, int64_t d, int32_t dtype, const void* x,
                     const float* scale, const float* shift, void* out, float eps, void* stream);
/* h = x + th[b] * r; m = LayerNorm(h) * (1 + scale[b]) */
int nimg_gate_res_ln_modulate(int64_t rows, int64_t S, int64_t d, int32_t dtype, const void* x,
                              const void* r, const float* th, const float* scale, void* h_out,
                              void* m_out, float eps, void* stream);
/* out = x + th[b] * r */
int nimg_gated_residual(int64_t rows, int64_t S, int64_t d, int32_t dtype, const void* x,
                        const void* r, const float* th, void* out, void* stream);
/* per (token, head) row of dh: RMSNorm then the 2-axis rotary rotation with
 * per-position tables cos_t / sin_t (S, dh) fp32; rows = B*S*H. Token t's
 * heads start at x + t * x_token_stride elements (a slice of a fused QKV
 * projection); out is contiguous (rows, dh). */
int nimg_qk_norm_rope(int64_t rows, int64_t S, int64_t H, int64_t dh, int32_t dtype, const void* x,
                      int64_t x_token_stride, const float* cos_t, const float* sin_t, void* out,
                      float eps, void* stream);

/* ------------------------------------------------------------------ expert-parallel transport
 * Copy-engine exchange over NVLink (no SMs, so transfers overlap the persistent
 * GEMMs). Setup-time: peer-writable buffers shared between the ranks of one
 * node through CUDA IPC. Hot path: stream-ordered copies and 32-bit flags. */
int nimg_ipc_alloc(size_t bytes, void** dev_ptr, void* handle /* 64 B out */);
int nimg_ipc_open(const void* handle /* 64 B */, void** dev_ptr);
int nimg_ipc_close(void* dev_ptr);
int nimg_free(void* dev_ptr);
/* cudaMemcpyAsync device-to-device (peer pointers allowed: copy engine). */
int nimg_copy_async(void* dst, const void* src, size_t bytes, void* stream);
/* Stream-ordered 32-bit store (after a full memory barrier) / wait until
 * *addr >= value. addr may be a peer-mapped flag. */
int nimg_stream_write_u32(void* dev_addr, uint32_t value, void* stream);
int nimg_stream_wait_geq_u32(void* dev_addr, uint32_t value, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NIMG_MOE_H_ */
