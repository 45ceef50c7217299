"""Denoising-step stack on the GPU: MoEDiT.forward.

Mirrors the reference backbone (/root/reference/pkg/src/nimg/backbone.py):
same ModelConfig fields and checks (:342-376), same parameter names
(:420-440, :467-477), same seeded initialisation order (:450-465, :391-418),
same hash text encoder and per-layer text-KV precompute (:299-311, :488-519),
and the same forward (:548-635):

    tokens = patchify(z_t); x = tokens W_p + b_p; t_vec = MLP(sinusoid(t))
    per block: (sa_shift, sa_scale, sa_gate, ff_scale, ff_gate) = t_vec W_mod + b_mod
               a_in = LN(x)(1 + sa_scale) + sa_shift
               r    = joint_attention(rope(rmsnorm(a_in W_q)), rope(rmsnorm(a_in W_k)),
                                      a_in W_v, text KV) W_o
               dense: h, f_in = gated residual + LN-scale; x = h + tanh(ff_gate) swiglu(f_in)
               MoE:   x = moe block (gated residual, RMSNorm prologue, expert-choice
                      layer, gated residual)
    y = LN(x)(1 + f_scale) + f_shift; vel = unpatchify(y W_out + b_out)

Execution. The MoE blocks run through the library's fused block entry point
(`block.moe_block_forward`: prologue kernel, router, grouped tcgen05 GEMMs,
combine with the gated residual in its epilogue), the dense FFNs of layers
0..dense_layers-1 through the same grouped GEMM as a single group
(`nimg_expert_ffn`, shared-expert slot). Everything else -- patch and
timestep embeddings, modulation, LayerNorm-scale, QK-RMSNorm, 2-axis RoPE and
the joint attention (torch SDPA over image + cached text KV) -- is plain
PyTorch in `compute_dtype`; SURVEY 8(d) cfg5 puts the non-MoE parts there.

The MoE / dense-FFN stage is a `backend` object (dense_ffn, moe_block); the
product backend is `CudaBackend`. Tests substitute a CPU double to pin the
PyTorch parts against the reference in float64.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.nn.functional as F

from .errors import ConfigError, DomainError, ShapeError
from .moe import ExpertBank, bank_on_device
from .router import DENSE, RouterConfig, StageId, capacity_schedule

__all__ = ["ModelConfig", "NUCLEUS_IMAGE", "MoEDiT", "TextContext", "CudaBackend",
           "init_parameters", "random_parameters", "encode_prompt", "hash_token_embedding",
           "trunc_normal"]


@dataclass
class ModelConfig:
    """backbone.py:342-376 (same fields, defaults and checks)."""
    n_layers: int = 4
    d_model: int = 32
    n_q_heads: int = 4
    n_kv_heads: int = 1
    head_dim: int = 8
    n_experts: int = 4
    expert_hidden: int = 16
    shared_hidden: int | None = None
    dense_hidden: int | None = None
    dense_layers: int = 3
    latent_channels: int = 4
    patch: int = 2
    gate_scale: float = 1.0
    gate_eps: float = 1e-6
    capacity_override: float | None = None
    seed: int = 0
    dtype: str = "float64"

    def __post_init__(self):
        if self.n_q_heads % self.n_kv_heads != 0:
            raise ConfigError("n_q_heads must be a multiple of n_kv_heads")
        if self.n_q_heads * self.head_dim != self.d_model:
            raise ConfigError("n_q_heads * head_dim must equal d_model")
        if self.head_dim % 4 != 0:
            raise ConfigError("head_dim must be divisible by 4 for 2-axis rope")
        if self.shared_hidden is None:
            self.shared_hidden = self.expert_hidden
        if self.dense_hidden is None:
            self.dense_hidden = self.d_model

    @property
    def np_dtype(self):
        return np.float64 if self.dtype == "float64" else np.float32


# Nucleus-Image: 32 layers, d 2048, 16 / 4 heads of
# 128, 3 dense layers (hidden 2048), 64 routed experts of hidden 1344 + shared.
NUCLEUS_IMAGE = dict(n_layers=32, d_model=2048, n_q_heads=16, n_kv_heads=4, head_dim=128,
                     n_experts=64, expert_hidden=1344, dense_hidden=2048, dense_layers=3,
                     latent_channels=16, patch=2, dtype="float32")


def trunc_normal(rng: np.random.Generator, shape, std: float = 0.02) -> np.ndarray:
    """backbone.py:332-339: Normal(0, std) resampled until inside +-2 std."""
    out = rng.standard_normal(shape) * std
    bad = np.abs(out) > 2.0 * std
    while np.any(bad):
        out[bad] = rng.standard_normal(int(bad.sum())) * std
        bad = np.abs(out) > 2.0 * std
    return out


def init_parameters(cfg: ModelConfig) -> dict[str, np.ndarray]:
    """The reference model's parameters for cfg.seed, by name, in cfg's dtype:
    MoEDiT.__init__ (backbone.py:450-465) and Block.__init__ (:391-418) draw
    from one default_rng(seed) in this exact order."""
    rng = np.random.default_rng(cfg.seed)
    d, dt = cfg.d_model, cfg.np_dtype
    kv = cfg.n_kv_heads * cfg.head_dim
    in_dim = cfg.latent_channels * cfg.patch * cfg.patch
    tn = lambda shape, std=0.02: trunc_normal(rng, shape, std).astype(dt)
    z = lambda shape: np.zeros(shape, dtype=dt)
    p = {"patch_embed.weight": tn((in_dim, d)), "patch_embed.bias": z(d)}
    p["time_embed.fc1.weight"] = tn((d, d))
    p["time_embed.fc1.bias"] = z(d)
    p["time_embed.fc2.weight"] = tn((d, d))
    p["time_embed.fc2.bias"] = z(d)
    for i in range(cfg.n_layers):
        pre = f"blocks.{i}"
        for name, shape in (("wq", (d, d)), ("wk", (d, kv)), ("wv", (d, kv)), ("wo", (d, d)),
                            ("wk_txt", (d, kv)), ("wv_txt", (d, kv))):
            p[f"{pre}.attn.{name}"] = tn(shape)
        p[f"{pre}.img_mod.weight"] = z((d, 5 * d))
        p[f"{pre}.img_mod.bias"] = z(5 * d)
        if i < cfg.dense_layers:
            h = cfg.dense_hidden
            p[f"{pre}.ffn.w1"] = tn((h, d))
            p[f"{pre}.ffn.w3"] = tn((h, d))
            p[f"{pre}.ffn.w2"] = tn((d, h))
        else:
            E, h, hs = cfg.n_experts, cfg.expert_hidden, cfg.shared_hidden
            p[f"{pre}.router.gate"] = tn((2 * d, E), 0.006)
            p[f"{pre}.moe.w1"] = tn((E, h, d))
            p[f"{pre}.moe.w3"] = tn((E, h, d))
            p[f"{pre}.moe.w2"] = tn((E, d, h))
            p[f"{pre}.moe.shared_w1"] = tn((hs, d))
            p[f"{pre}.moe.shared_w3"] = tn((hs, d))
            p[f"{pre}.moe.shared_w2"] = tn((d, hs))
    p["final_mod.weight"] = z((d, 2 * d))
    p["final_mod.bias"] = z(2 * d)
    p["final_proj.weight"] = tn((d, in_dim))
    p["final_proj.bias"] = z(in_dim)
    return p


def random_parameters(cfg: ModelConfig, device, expert_dtype=torch.bfloat16, seed: int = 0):
    """Device-side random init with the reference's distributions (trunc
    normal 0.02, router 0.006, zero biases; modulation N(0, 0.02) instead of
    zero so the blocks are not identities) for full-size benchmarking, where
    the numpy draw of init_parameters would take minutes. Expert and dense
    FFN matrices are created in `expert_dtype`."""
    g = torch.Generator(device=device).manual_seed(seed)
    dt = torch.float64 if cfg.dtype == "float64" else torch.float32

    def tn(shape, std=0.02, dtype=dt):
        out = torch.empty(shape, device=device, dtype=torch.float32)
        out.normal_(0.0, std, generator=g).clamp_(-2 * std, 2 * std)
        return out.to(dtype)
    shapes = {k: v.shape for k, v in init_parameters(
        ModelConfig(**{**cfg.__dict__, "n_layers": 0})).items()}
    p = {k: (tn(s) if k.endswith(("weight",)) and not k.startswith("final_mod")
             else torch.zeros(s, device=device, dtype=dt)) for k, s in shapes.items()}
    d, kv = cfg.d_model, cfg.n_kv_heads * cfg.head_dim
    p["final_mod.weight"] = tn((d, 2 * d))
    for i in range(cfg.n_layers):
        pre = f"blocks.{i}"
        for name, shape in (("wq", (d, d)), ("wk", (d, kv)), ("wv", (d, kv)), ("wo", (d, d)),
                            ("wk_txt", (d, kv)), ("wv_txt", (d, kv))):
            p[f"{pre}.attn.{name}"] = tn(shape)
        p[f"{pre}.img_mod.weight"] = tn((d, 5 * d))
        p[f"{pre}.img_mod.bias"] = torch.zeros(5 * d, device=device, dtype=dt)
        if i < cfg.dense_layers:
            h = cfg.dense_hidden
            for name, shape in (("w1", (h, d)), ("w3", (h, d)), ("w2", (d, h))):
                p[f"{pre}.ffn.{name}"] = tn(shape, dtype=expert_dtype)
        else:
            E, h, hs = cfg.n_experts, cfg.expert_hidden, cfg.shared_hidden
            p[f"{pre}.router.gate"] = tn((2 * d, E), 0.006)
            for name, shape in (("w1", (E, h, d)), ("w3", (E, h, d)), ("w2", (E, d, h)),
                                ("shared_w1", (hs, d)), ("shared_w3", (hs, d)),
                                ("shared_w2", (d, hs))):
                p[f"{pre}.moe.{name}"] = tn(shape, dtype=expert_dtype)
    return p


# ---------------------------------------------------------------- text encoder
def hash_token_embedding(token: str, dim: int) -> np.ndarray:
    """backbone.py:299-303: deterministic per-token embedding from sha256."""
    seed = int.from_bytes(hashlib.sha256(token.encode("utf-8")).digest()[:8], "little")
    return np.random.default_rng(seed).standard_normal(dim) / math.sqrt(dim)


def encode_prompt(prompt: str, dim: int) -> np.ndarray:
    """backbone.py:306-311."""
    toks = prompt.split()
    if not toks:
        return np.zeros((0, dim))
    return np.stack([hash_token_embedding(tok, dim) for tok in toks])


@dataclass
class TextContext:
    """backbone.py:314-329: per-layer text K/V (B, S_t, H_kv, d_h), fixed for
    a prompt set and reused across denoising steps."""
    k_txt: list
    v_txt: list
    mask: torch.Tensor            # (B, S_t) bool, True = valid token
    s_t: int
    prompts: tuple = ()
    all_valid: bool = True        # no padding: attention needs no mask


# ---------------------------------------------------------------- backends
class CudaBackend:
    """The library's kernels: fused MoE block (block.moe_block_forward) and
    the dense SwiGLU FFN through the grouped GEMM as one group."""

    name = "cuda"

    def __init__(self, act_dtype: torch.dtype = torch.bfloat16, ep=None):
        if act_dtype not in (torch.bfloat16, torch.float32):
            raise ConfigError(f"unsupported activation dtype {act_dtype}")
        self.act = act_dtype
        self.ep = ep          # ep.EPContext: MoE blocks expert-parallel over its ranks
        from .stages import CudaStages
        self._stages = CudaStages()

    def prepare_bank(self, bank: ExpertBank) -> ExpertBank:
        if self.ep is not None and self.ep.world > 1:
            from .ep import shard_bank
            bank = shard_bank(bank, self.ep.rank, self.ep.world)
        return bank_on_device(bank, self.act)

    def prepare_dense(self, w1, w3, w2):
        return tuple(w.to(dtype=self.act).contiguous() for w in (w1, w3, w2))

    def dense_ffn(self, f_in: torch.Tensor, w1, w3, w2) -> torch.Tensor:
        """moe.py:31-51 swiglu on (T, d) rows (backbone.py:577-580)."""
        _, y = self._stages.expert_ffn(None, None, None, None, None, None,
                                       f_in.to(self.act).contiguous(), w1, w3, w2)
        return y

    def moe_block(self, x, sa_gate, r_attn, ff_scale, ff_gate, t_vec, layer, rcfg, bank, w_r,
                  return_routing: bool):
        """backbone.py:583-606 through nimg_moe_block_forward."""
        from .block import moe_block_forward
        f32 = torch.float32
        if self.ep is not None:
            from .ep import ep_moe_block_forward
            return ep_moe_block_forward(x.to(self.act).contiguous(), sa_gate.to(f32),
                                        r_attn.to(self.act), ff_scale.to(f32), ff_gate.to(f32),
                                        t_vec.to(f32), layer, rcfg, bank, w_r, self.ep,
                                        return_routing=return_routing)
        return moe_block_forward(x.to(self.act).contiguous(), sa_gate.to(f32), r_attn.to(self.act),
                                 ff_scale.to(f32), ff_gate.to(f32), t_vec.to(f32), layer, rcfg,
                                 bank, w_r, return_routing=return_routing)


class _StackKernels:
    """The fused element-wise chains (csrc/stack_kernels.cu) for fp32 / bf16."""

    def __init__(self, act: torch.dtype):
        from . import _lib
        from ._tensors import nimg_dtype
        self.L, self.dt, self.act = _lib, nimg_dtype(act), act

    def _s(self):
        return torch.cuda.current_stream().cuda_stream

    def ln_mod(self, x, scale, shift=None, eps=1e-6):
        B, S, d = x.shape
        out = torch.empty_like(x)
        self.L.check(self.L.lib.nimg_ln_modulate(B * S, S, d, self.dt, x.data_ptr(),
                                                 scale.data_ptr(),
                                                 None if shift is None else shift.data_ptr(),
                                                 out.data_ptr(), eps, self._s()))
        return out

    def gate_res_ln(self, x, th, r, scale, eps=1e-6):
        B, S, d = x.shape
        h, m = torch.empty_like(x), torch.empty_like(x)
        self.L.check(self.L.lib.nimg_gate_res_ln_modulate(B * S, S, d, self.dt, x.data_ptr(),
                                                          r.data_ptr(), th.data_ptr(),
                                                          scale.data_ptr(), h.data_ptr(),
                                                          m.data_ptr(), eps, self._s()))
        return h, m

    def gated_res(self, x, th, r):
        B, S, d = x.shape
        out = torch.empty_like(x)
        self.L.check(self.L.lib.nimg_gated_residual(B * S, S, d, self.dt, x.data_ptr(),
                                                    r.data_ptr(), th.data_ptr(), out.data_ptr(),
                                                    self._s()))
        return out

    def qk_norm_rope(self, x, token_stride, B, S, H, dh, cos, sin, eps=1e-6):
        out = torch.empty((B, S, H, dh), dtype=self.act, device=x.device)
        self.L.check(self.L.lib.nimg_qk_norm_rope(B * S * H, S, H, dh, self.dt, x.data_ptr(),
                                                  token_stride, cos.data_ptr(), sin.data_ptr(),
                                                  out.data_ptr(), eps, self._s()))
        return out


# ---------------------------------------------------------------- model
def _ln_scale(x: torch.Tensor, s: torch.Tensor, eps: float = 1e-6) -> torch.Tensor:
    """backbone.py:62-88 fused_ln_scale: LayerNorm(x) * (1 + s), s (B, d)."""
    xw = x if x.dtype == torch.float64 else x.float()
    mu = xw.mean(dim=-1, keepdim=True)
    xc = xw - mu
    var = (xc * xc).mean(dim=-1, keepdim=True)
    out = xc * (1.0 / torch.sqrt(var + eps)) * (1.0 + s.to(xw.dtype)[:, None, :])
    return out.to(x.dtype)


def _rmsnorm(x: torch.Tensor, eps: float = 1e-6) -> torch.Tensor:
    """tensor.py:518-531 over the last axis, no affine."""
    xw = x if x.dtype == torch.float64 else x.float()
    return (xw * (1.0 / torch.sqrt((xw * xw).mean(dim=-1, keepdim=True) + eps))).to(x.dtype)


def _rope_tables(pos_h, pos_w, d_h: int, base: float = 10000.0):
    """backbone.py:128-137 (numpy f64, exactly the reference's tables)."""
    quarter = d_h // 4
    freqs = base ** (-np.arange(quarter, dtype=np.float64) / quarter)
    ang = np.concatenate([np.multiply.outer(np.asarray(pos_h, dtype=np.float64), freqs),
                          np.multiply.outer(np.asarray(pos_w, dtype=np.float64), freqs)], axis=-1)
    ang = np.repeat(ang, 2, axis=-1)
    return np.cos(ang), np.sin(ang)


def _rotate_pairs(t: torch.Tensor) -> torch.Tensor:
    """backbone.py:140-153: (x0, x1) -> (-x1, x0) per adjacent pair."""
    t2 = t.unflatten(-1, (-1, 2))
    return torch.stack((-t2[..., 1], t2[..., 0]), dim=-1).flatten(-2)


class MoEDiT:
    """GPU MoEDiT (backbone.py:447-635). `params`: name -> array/tensor as in
    the reference's named_parameters() (default: init_parameters(cfg))."""

    def __init__(self, cfg: ModelConfig, params: dict | None = None, *,
                 compute_dtype: torch.dtype = torch.float32, backend=None, device=None):
        self.cfg = cfg
        self.dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        self.cd = compute_dtype
        self.store = torch.float64 if cfg.dtype == "float64" else torch.float32
        self.backend = backend if backend is not None else CudaBackend(
            torch.float32 if compute_dtype in (torch.float32, torch.float64) else torch.bfloat16)
        params = init_parameters(cfg) if params is None else params
        t = lambda a, dt: torch.as_tensor(np.asarray(a) if not isinstance(a, torch.Tensor) else a
                                          ).to(self.dev, dt).contiguous()
        # expert / dense-FFN matrices stay in the dtype given (a bf16 bank is
        # used in place); everything else is held in the storage dtype
        big = lambda k: ".moe." in k or ".ffn." in k
        self.params = {k: (t(v, v.dtype) if big(k) and isinstance(v, torch.Tensor) else
                           t(v, self.store)) for k, v in params.items()}
        P, cd = self.params, compute_dtype
        # working copies: attention / embeddings in compute dtype, modulation in f64
        self.w = {k: v.to(cd) for k, v in P.items()
                  if ".attn." in k or k.startswith(("patch_embed", "final_proj"))}
        self.f64 = {k: v.double() for k, v in P.items() if k.startswith("time_embed")}
        # modulation in f64 only for the f64 pin; fp32 otherwise (B x d x 5d)
        self.mdt = torch.float64 if compute_dtype == torch.float64 else torch.float32
        self.modw = {k: v.to(self.mdt) for k, v in P.items() if "mod." in k}
        # fused element-wise kernels for fp32 / bf16 on CUDA, one QKV GEMM
        self.fast = (compute_dtype in (torch.float32, torch.bfloat16) and self.dev.type == "cuda"
                     and cfg.d_model % 8 == 0)
        self.K = _StackKernels(compute_dtype) if self.fast else None
        if self.fast:
            for i in range(cfg.n_layers):
                pre = f"blocks.{i}.attn"
                self.w[f"{pre}.wqkv"] = torch.cat([self.w[f"{pre}.wq"], self.w[f"{pre}.wk"],
                                                   self.w[f"{pre}.wv"]], dim=1).contiguous()
        self.banks, self.dense = {}, {}
        for i in range(cfg.n_layers):
            pre = f"blocks.{i}"
            if i < cfg.dense_layers:
                self.dense[i] = self.backend.prepare_dense(P[f"{pre}.ffn.w1"], P[f"{pre}.ffn.w3"],
                                                           P[f"{pre}.ffn.w2"])
            else:
                b = ExpertBank(*(P[f"{pre}.moe.{n}"] for n in ("w1", "w3", "w2", "shared_w1",
                                                               "shared_w3", "shared_w2")))
                self.banks[i] = self.backend.prepare_bank(b)
        self._rope_cache = {}
        self.text_kv_recompute_count = 0

    def named_parameters(self) -> dict:
        return dict(self.params)

    def router_weights(self) -> dict:
        return {i: self.params[f"blocks.{i}.router.gate"] for i in self.banks}

    # ---- helpers
    def _rope(self, pos_h, pos_w, d_h: int, dtype=None):
        dtype = self.cd if dtype is None else dtype
        key = (tuple(np.asarray(pos_h).tolist()), tuple(np.asarray(pos_w).tolist()), d_h, dtype)
        if key not in self._rope_cache:
            c, s = _rope_tables(pos_h, pos_w, d_h)
            self._rope_cache[key] = (torch.from_numpy(c).to(self.dev, dtype).contiguous(),
                                     torch.from_numpy(s).to(self.dev, dtype).contiguous())
        return self._rope_cache[key]

    def _apply_rope(self, x: torch.Tensor, pos_h, pos_w) -> torch.Tensor:
        """backbone.py:172-182 on (B, S, H, d_h)."""
        c, s = self._rope(pos_h, pos_w, x.shape[-1])
        return x * c[None, :, None, :] + _rotate_pairs(x) * s[None, :, None, :]

    def _linear(self, x: torch.Tensor, w: torch.Tensor, b: torch.Tensor | None = None):
        y = x @ w
        return y if b is None else y + b

    # ---- text
    def precompute_text_kv(self, prompts: list[str]) -> TextContext:
        """backbone.py:488-519: per-layer text K (QK-RMSNorm + RoPE on the
        width axis) and V, once per prompt set."""
        self.text_kv_recompute_count += 1
        cfg = self.cfg
        d = cfg.d_model
        enc = [encode_prompt(p, d) for p in prompts]
        s_t = max((e.shape[0] for e in enc), default=0)
        B = len(prompts)
        mask = np.zeros((B, s_t), dtype=bool)
        cmat = np.zeros((B, s_t, d))
        for b, e in enumerate(enc):
            mask[b, :e.shape[0]] = True
            cmat[b, :e.shape[0]] = e
        mask_t = torch.from_numpy(mask).to(self.dev)
        if s_t == 0:
            return TextContext([], [], mask_t, 0, tuple(prompts), True)
        c = torch.from_numpy(cmat).to(self.dev, self.store).to(self.cd)
        # projections and the K RMSNorm of storage-dtype operands round to the
        # storage dtype; RoPE's f64 tables promote K (backbone.py:505-512)
        rd = lambda a: a.to(self.store).to(self.cd)
        pos_w, pos_h = np.arange(s_t), np.zeros(s_t)
        ks, vs = [], []
        for i in range(cfg.n_layers):
            pre = f"blocks.{i}.attn"
            k = rd(self._linear(c, self.w[f"{pre}.wk_txt"])).view(B, s_t, cfg.n_kv_heads,
                                                                  cfg.head_dim)
            ks.append(self._apply_rope(rd(_rmsnorm(k)), pos_h, pos_w))
            vs.append(rd(self._linear(c, self.w[f"{pre}.wv_txt"])).view(B, s_t, cfg.n_kv_heads,
                                                                         cfg.head_dim))
        return TextContext(ks, vs, mask_t, s_t, tuple(prompts), bool(mask.all()))

    # ---- layout
    def patchify(self, z: torch.Tensor):
        """backbone.py:521-529."""
        B, C, H, W = z.shape
        p = self.cfg.patch
        if H % p or W % p:
            raise ShapeError(f"latent {H}x{W} not divisible by patch {p}")
        gh, gw = H // p, W // p
        t = z.reshape(B, C, gh, p, gw, p).permute(0, 2, 4, 1, 3, 5)
        return t.reshape(B, gh * gw, C * p * p), (gh, gw)

    def unpatchify(self, tokens: torch.Tensor, grid, shape):
        """backbone.py:531-538."""
        B, C, H, W = shape
        p = self.cfg.patch
        gh, gw = grid
        return tokens.reshape(B, gh, gw, C, p, p).permute(0, 3, 1, 4, 2, 5).reshape(B, C, H, W)

    def capacity_factor_for(self, layer: int, stage: StageId) -> float:
        """backbone.py:540-546."""
        if self.cfg.capacity_override is not None:
            return self.cfg.capacity_override
        cf = capacity_schedule(max(layer, 3), stage, n_layers=max(32, self.cfg.n_layers))
        assert cf is not DENSE
        return cf

    # ---- forward
    def time_embed(self, t) -> torch.Tensor:
        """backbone.py:244-281 (f64, as in the reference, where the f64
        frequency table promotes the timestep features)."""
        d = self.cfg.d_model
        if d % 2 != 0:
            raise ConfigError(f"feature dim {d} must be even")
        vals = np.asarray(t, dtype=np.float64).reshape(-1)
        if np.any(vals < 0.0) or np.any(vals > 1.0):
            raise DomainError(f"timestep outside [0, 1]: {vals}")
        half = d // 2
        freqs = np.exp(np.linspace(0.0, math.log(10000.0), half))
        tt = torch.from_numpy(vals.astype(self.cfg.np_dtype).astype(np.float64)).to(self.dev)
        args = tt[:, None] * torch.from_numpy(freqs).to(self.dev)[None, :]
        feats = torch.cat([torch.sin(args), torch.cos(args)], dim=-1)
        W = self.f64
        h = F.silu(feats @ W["time_embed.fc1.weight"] + W["time_embed.fc1.bias"])
        return h @ W["time_embed.fc2.weight"] + W["time_embed.fc2.bias"]

    def _attention(self, i: int, a_in: torch.Tensor, ctx: TextContext | None, pos_h, pos_w):
        """backbone.py:621-635 + joint_attention :195-232 (SDPA)."""
        cfg = self.cfg
        B, S, _ = a_in.shape
        pre = f"blocks.{i}.attn"
        if self.fast:
            return self._attention_fast(i, a_in, ctx, pos_h, pos_w)
        q = self._linear(a_in, self.w[f"{pre}.wq"]).view(B, S, cfg.n_q_heads, cfg.head_dim)
        k = self._linear(a_in, self.w[f"{pre}.wk"]).view(B, S, cfg.n_kv_heads, cfg.head_dim)
        v = self._linear(a_in, self.w[f"{pre}.wv"]).view(B, S, cfg.n_kv_heads, cfg.head_dim)
        q = self._apply_rope(_rmsnorm(q), pos_h, pos_w)
        k = self._apply_rope(_rmsnorm(k), pos_h, pos_w)
        mask = None
        if ctx is not None and ctx.s_t > 0:
            k = torch.cat([k, ctx.k_txt[i]], dim=1)
            v = torch.cat([v, ctx.v_txt[i]], dim=1)
            valid = torch.cat([torch.ones((B, S), dtype=torch.bool, device=self.dev), ctx.mask], 1)
            mask = valid[:, None, None, :]
        n_rep = cfg.n_q_heads // cfg.n_kv_heads
        qh = q.transpose(1, 2)
        kh = k.transpose(1, 2).repeat_interleave(n_rep, dim=1)
        vh = v.transpose(1, 2).repeat_interleave(n_rep, dim=1)
        out = F.scaled_dot_product_attention(qh, kh, vh, attn_mask=mask,
                                             scale=1.0 / math.sqrt(cfg.head_dim))
        return self._linear(out.transpose(1, 2).reshape(B, S, cfg.d_model), self.w[f"{pre}.wo"])

    def _attention_fast(self, i, a_in, ctx, pos_h, pos_w):
        """One QKV GEMM, fused QK-RMSNorm + RoPE kernel, cuDNN SDPA with native
        GQA (no mask unless the text context has padding)."""
        cfg = self.cfg
        B, S, d = a_in.shape
        Hq, Hkv, dh = cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim
        kv = Hkv * dh
        pre = f"blocks.{i}.attn"
        qkv = a_in @ self.w[f"{pre}.wqkv"]                       # (B, S, d + 2 kv)
        cos, sin = self._rope(pos_h, pos_w, dh, torch.float32)
        ld = d + 2 * kv
        q = self.K.qk_norm_rope(qkv, ld, B, S, Hq, dh, cos, sin)
        k = self.K.qk_norm_rope(qkv[..., d:], ld, B, S, Hkv, dh, cos, sin)
        v = qkv[..., d + kv:].view(B, S, Hkv, dh)
        mask = None
        if ctx is not None and ctx.s_t > 0:
            k = torch.cat([k, ctx.k_txt[i].to(k.dtype)], dim=1)
            v = torch.cat([v, ctx.v_txt[i].to(v.dtype)], dim=1)
            if not ctx.all_valid:
                valid = torch.cat([torch.ones((B, S), dtype=torch.bool, device=self.dev),
                                   ctx.mask], 1)
                mask = valid[:, None, None, :]
        out = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2),
                                             v.transpose(1, 2), attn_mask=mask,
                                             scale=1.0 / math.sqrt(dh), enable_gqa=True)
        return out.transpose(1, 2).reshape(B, S, d) @ self.w[f"{pre}.wo"]

    def forward(self, z_t, t, ctx: TextContext | None, stage: StageId,
                capture_step: int | None = None, return_aux: bool = True):
        """backbone.py:548-619. Returns (velocity, aux); aux has the per-MoE-
        layer router logits and decisions (and RouteRecords when capture_step
        is set) unless return_aux=False (no device->host traffic)."""
        cfg, cd = self.cfg, self.cd
        z = torch.as_tensor(z_t).to(self.dev, self.store)
        B = z.shape[0]
        tokens, (gh, gw) = self.patchify(z)
        # patch embedding in the storage dtype (backbone.py:552-554)
        x = (tokens.to(cd) @ self.w["patch_embed.weight"]).to(self.store)
        x = (x.to(cd) + self.w["patch_embed.bias"]).to(self.store).to(cd)
        t_vec = self.time_embed(t if not np.isscalar(t) else np.full(B, float(t)))
        pos_h = np.repeat(np.arange(gh), gw)
        pos_w = np.tile(np.arange(gw), gh)
        d = cfg.d_model
        aux = {"router_logits": [], "decisions": [], "records": []}
        K = self.K
        t_m = t_vec.to(self.mdt)
        for i in range(cfg.n_layers):
            pre = f"blocks.{i}"
            mod = t_m @ self.modw[f"{pre}.img_mod.weight"] + self.modw[f"{pre}.img_mod.bias"]
            sa_shift, sa_scale, sa_gate, ff_scale, ff_gate = (mod[:, j * d:(j + 1) * d]
                                                              for j in range(5))
            if self.fast:
                a_in = K.ln_mod(x, sa_scale.float().contiguous(), sa_shift.float().contiguous())
            else:
                a_in = (_ln_scale(x, sa_scale).to(cd) + sa_shift.to(cd)[:, None, :])
            r_attn = self._attention(i, a_in, ctx, pos_h, pos_w)
            if i in self.dense and self.fast:
                h, f_in = K.gate_res_ln(x, torch.tanh(sa_gate).float().contiguous(), r_attn,
                                        ff_scale.float().contiguous())
                f_out = self.backend.dense_ffn(f_in.reshape(B * gh * gw, d), *self.dense[i])
                x = K.gated_res(h, torch.tanh(ff_gate).float().contiguous(),
                                f_out.to(cd).view(B, gh * gw, d))
            elif i in self.dense:
                # fused_gate_res_ln_scale (backbone.py:91-121, :577-580)
                h = x + torch.tanh(sa_gate).to(cd)[:, None, :] * r_attn
                f_in = _ln_scale(h, ff_scale)
                f_out = self.backend.dense_ffn(f_in.reshape(B * gh * gw, d), *self.dense[i])
                x = h + torch.tanh(ff_gate).to(cd)[:, None, :] * f_out.to(cd).view(B, gh * gw, d)
            else:
                rcfg = RouterConfig(d_model=d, n_experts=cfg.n_experts,
                                    capacity_factor=self.capacity_factor_for(i, stage),
                                    gate_scale=cfg.gate_scale, gate_eps=cfg.gate_eps, seed=cfg.seed)
                res = self.backend.moe_block(x, sa_gate, r_attn, ff_scale, ff_gate, t_vec, i, rcfg,
                                             self.banks[i], self.params[f"{pre}.router.gate"],
                                             return_routing=return_aux)
                if return_aux:
                    out, decisions, routing = res
                    aux["router_logits"].append(routing["logits"])
                    aux["decisions"].append((i, decisions))
                    if capture_step is not None:
                        for dec in decisions:
                            aux["records"].append(dict(layer=i, step=capture_step,
                                                       logits=dec.logits,
                                                       top_indices=dec.top_indices,
                                                       grid=(gh, gw)))
                else:
                    out = res
                x = out.to(cd)
        fmod = t_m @ self.modw["final_mod.weight"] + self.modw["final_mod.bias"]
        f_shift, f_scale = fmod[:, :d], fmod[:, d:]
        if self.fast:
            y = K.ln_mod(x, f_scale.float().contiguous(), f_shift.float().contiguous())
        else:
            y = _ln_scale(x, f_scale).to(cd) + f_shift.to(cd)[:, None, :]
        out = y @ self.w["final_proj.weight"] + self.w["final_proj.bias"]
        vel = self.unpatchify(out, (gh, gw), tuple(z.shape))
        return vel, aux
