"""Seeded synthetic inputs for the MoE layer -- TEST INFRASTRUCTURE ONLY.

Recipe follows SURVEY.md section 8(d) / the reference backbone's init:
x ~ N(0,1); x_norm = rmsnorm(x)/sqrt(layer+1) (backbone.py:585-586,
tensor.py:518-531); x_mod = x_norm * (1 + s2) with s2 ~ N(0, 0.1^2) per
sample (backbone.py:587-589); t_emb ~ N(0,1); W_r ~ trunc_normal(0.006)
(backbone.py:415); expert / shared weights ~ trunc_normal(0.02)
(backbone.py:332-339, :394-395, :416-418).

bf16 mode: the activations and expert weights are rounded to
bf16-representable values (round-to-nearest-even) but stored as fp32 so the
oracle (which has no bf16, tensor.py:42-47) sees exactly the values the GPU
sees; W_r and t_emb stay fp32 so routing stays bit-comparable.
"""

from __future__ import annotations

import hashlib
import math

import numpy as np


def trunc_normal(rng, shape, std=0.02):
    """backbone.py:332-339 -- N(0, std) resampled until inside +-2 std."""
    out = rng.standard_normal(shape) * std
    bad = np.abs(out) > 2.0 * std
    while np.any(bad):
        out[bad] = rng.standard_normal(int(bad.sum())) * std
        bad = np.abs(out) > 2.0 * std
    return out


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest bf16 (ties to even); returns fp32."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def make_layer_inputs(seed: int, B: int, S: int, d: int, E: int, h: int,
                      h_shared: int | None = None, layer: int = 3,
                      mode: str = "fp32", expert_std: float = 0.02,
                      router_std: float = 0.006):
    """Returns a dict of fp32 arrays: x_norm, x_mod (B,S,d), t_emb (B,d),
    w_r (2d,E), w1, w3 (E,h,d), w2 (E,d,h), sw1, sw3 (hs,d), sw2 (d,hs)."""
    hs = h if h_shared is None else h_shared
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((B, S, d))
    ms = (x * x).mean(axis=-1, keepdims=True) + 1e-6
    x_norm = x / np.sqrt(ms) / math.sqrt(layer + 1)
    s2 = rng.standard_normal((B, d)) * 0.1
    x_mod = x_norm * (1.0 + s2[:, None, :])
    t_emb = rng.standard_normal((B, d))
    w_r = trunc_normal(rng, (2 * d, E), router_std)
    w1 = trunc_normal(rng, (E, h, d), expert_std)
    w3 = trunc_normal(rng, (E, h, d), expert_std)
    w2 = trunc_normal(rng, (E, d, h), expert_std)
    sw1 = trunc_normal(rng, (hs, d), expert_std)
    sw3 = trunc_normal(rng, (hs, d), expert_std)
    sw2 = trunc_normal(rng, (d, hs), expert_std)
    out = dict(x_norm=x_norm, x_mod=x_mod, t_emb=t_emb, w_r=w_r, w1=w1, w3=w3,
               w2=w2, sw1=sw1, sw3=sw3, sw2=sw2)
    out = {k: np.ascontiguousarray(v, dtype=np.float32) for k, v in out.items()}
    if mode == "bf16":
        for k in ("x_norm", "x_mod", "w1", "w3", "w2", "sw1", "sw3", "sw2"):
            out[k] = bf16_round(out[k])
    elif mode != "fp32":
        raise ValueError(mode)
    return out


def make_router_inputs(seed: int, B: int, S: int, d: int, E: int,
                       layer: int = 3, mode: str = "fp32"):
    """Router-only inputs (same recipe, no expert weights)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((B, S, d))
    ms = (x * x).mean(axis=-1, keepdims=True) + 1e-6
    x_norm = (x / np.sqrt(ms) / math.sqrt(layer + 1)).astype(np.float32)
    t_emb = rng.standard_normal((B, d)).astype(np.float32)
    w_r = trunc_normal(rng, (2 * d, E), 0.006).astype(np.float32)
    if mode == "bf16":
        x_norm = bf16_round(x_norm)
    return dict(x_norm=x_norm, t_emb=t_emb, w_r=w_r)


def digest(arrays: dict) -> str:
    """Stable content hash of a dict of arrays (detects generator drift)."""
    h = hashlib.sha256()
    for k in sorted(arrays):
        a = np.ascontiguousarray(arrays[k])
        h.update(k.encode())
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def make_block_inputs(seed: int, B: int, S: int, d: int, E: int, h: int, mode: str = "fp32"):
    """Inputs of the backbone's MoE branch (backbone.py:583-606): residual x,
    attention output r_attn (act dtype), per-sample modulation vectors
    sa_gate / ff_scale / ff_gate (fp32, small, as from the zero-init mod_w
    after training), t_vec (fp32), router and expert weights."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((B, S, d))
    r_attn = rng.standard_normal((B, S, d)) * 0.5
    sa_gate = rng.standard_normal((B, d)) * 0.3
    ff_scale = rng.standard_normal((B, d)) * 0.1
    ff_gate = rng.standard_normal((B, d)) * 0.3
    t_vec = rng.standard_normal((B, d))
    w_r = trunc_normal(rng, (2 * d, E), 0.006)
    ws = {k: trunc_normal(rng, s, 0.02) for k, s in (("w1", (E, h, d)), ("w3", (E, h, d)),
                                                     ("w2", (E, d, h)), ("sw1", (h, d)),
                                                     ("sw3", (h, d)), ("sw2", (d, h)))}
    out = dict(x=x, r_attn=r_attn, sa_gate=sa_gate, ff_scale=ff_scale, ff_gate=ff_gate,
               t_vec=t_vec, w_r=w_r, **ws)
    out = {k: np.ascontiguousarray(v, dtype=np.float32) for k, v in out.items()}
    if mode == "bf16":
        for k in ("x", "r_attn", "w1", "w3", "w2", "sw1", "sw3", "sw2"):
            out[k] = bf16_round(out[k])
    elif mode != "fp32":
        raise ValueError(mode)
    return out


def perturb_modulation(params: dict, seed: int, w_std: float = 0.2, b_std: float = 0.1):
    """Zero-initialised modulation makes every block an exact identity
    (backbone.py:1-6); for parity fixtures, overwrite the modulation weights
    and biases IN PLACE (same arrays the model holds) with seeded values, in
    sorted-name order so both sides draw identically."""
    rng = np.random.default_rng(seed)
    names = sorted(k for k in params if k.endswith(("img_mod.weight", "img_mod.bias",
                                                     "final_mod.weight", "final_mod.bias")))
    for k in names:
        a = params[k]
        std = w_std if k.endswith("weight") else b_std
        a[...] = (trunc_normal(rng, a.shape, std) if k.endswith("weight")
                  else rng.standard_normal(a.shape) * std).astype(a.dtype)
    return params


def make_latent(seed: int, B: int, C: int, H: int, W: int):
    """Noisy latent z_t ~ N(0, 1) (B, C, H, W) fp32 and per-sample timesteps
    spread over [0.2, 0.8]."""
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((B, C, H, W)).astype(np.float32)
    return z, np.linspace(0.2, 0.8, B)


DIT_PROMPTS = ("a red fox in fresh snow at dawn", "two cups of coffee on a wooden table",
               "mountain lake")


def make_bwd_inputs(p: dict):
    """Layer inputs plus a seeded upstream gradient g_out (B,S,d) in the
    activation dtype's values (bf16-representable in bf16 mode)."""
    inp = make_layer_inputs(p["seed"], p["B"], p["S"], p["d"], p["E"], p["h"],
                            layer=p.get("layer", 3), mode=p["mode"])
    rng = np.random.default_rng(p["seed"] + 1000)
    g = rng.standard_normal((p["B"], p["S"], p["d"])).astype(np.float32)
    inp["g_out"] = bf16_round(g) if p["mode"] == "bf16" else g
    return inp
