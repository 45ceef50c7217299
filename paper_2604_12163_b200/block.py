"""The backbone's MoE branch around the layer.

Mirrors the MoE arm of MoEDiT.forward (/root/reference/pkg/src/nimg/
backbone.py:583-606):

    h      = fused_gated_residual(x, sa_gate, r_attn)        # backbone.py:584
    x_norm = rmsnorm(h) * 1/sqrt(layer + 1)                  # :585-586
    x_mod  = x_norm * (1 + ff_scale)                         # :587-589
    moe_out, decisions, routing = moe_forward(h, x_norm, x_mod, t_vec, ...)  # :595-597
    x      = fused_gated_residual(h, ff_gate, moe_out)       # :606

as one library call (`nimg_moe_block_forward`): a fused prologue kernel
(gated residual + RMSNorm + scale + modulation in one pass, numpy-exact
rounding chain), the MoE layer, and the gated residual fused into the
combine's epilogue (the layer output is never written to HBM).
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from ._tensors import ptr, stream_handle, to_device, workspace
from .errors import ConfigError, ShapeError
from .moe import ExpertBank, _check_bank_shapes, bank_on_device
from .router import RouterConfig, alloc_route_out, build_routing, capacity_for, make_desc, route_struct

__all__ = ["moe_block_forward", "moe_block_prologue"]


def moe_block_forward(x, sa_gate, r_attn, ff_scale, ff_gate, t_vec, layer: int,
                      cfg: RouterConfig, bank: ExpertBank, w_r, return_routing: bool = False,
                      return_intermediates: bool = False):
    """Returns the updated residual stream (B, S, d) in x's dtype; optionally
    (out, decisions, routing) and/or a dict with h, x_norm, x_mod."""
    xt = to_device(x)
    act = xt.dtype
    B, S, d = xt.shape
    ra = to_device(r_attn, act)
    if tuple(ra.shape) != (B, S, d):
        raise ShapeError(f"r_attn shape {tuple(ra.shape)} != {(B, S, d)}")
    mods = [to_device(m, torch.float32) for m in (sa_gate, ff_scale, ff_gate, t_vec)]
    for m in mods:
        if tuple(m.shape) != (B, d):
            raise ShapeError(f"modulation shape {tuple(m.shape)} != {(B, d)}")
    cfg.validate_weight(w_r)
    wr = to_device(w_r, torch.float32)
    E = cfg.n_experts
    if d != cfg.d_model:
        raise ConfigError(f"width {d} != d_model {cfg.d_model}")
    cap = capacity_for(S, E, cfg.capacity_factor)
    w = bank_on_device(bank, act)
    _, h, hs = _check_bank_shapes(w.w1, w.w3, w.w2, w.shared_w1, w.shared_w3, w.shared_w2, d)
    desc = make_desc(B, S, d, E, cap, h, hs, cfg, act)
    nbytes = C.c_size_t()
    _lib.check(_lib.lib.nimg_moe_block_workspace_bytes(C.byref(desc), C.byref(nbytes)))
    ws = workspace(nbytes.value)
    outs = {k: torch.empty((B, S, d), dtype=act, device=xt.device) for k in ("h", "x_norm", "x_mod", "out")}
    r = alloc_route_out(B, S, E, cap, xt.device)
    bp = _lib.BlockPtrs(ptr(xt), ptr(ra), *(ptr(m) for m in mods), ptr(wr), ptr(w.w1), ptr(w.w3),
                        ptr(w.w2), ptr(w.shared_w1), ptr(w.shared_w3), ptr(w.shared_w2),
                        ptr(outs["h"]), ptr(outs["x_norm"]), ptr(outs["x_mod"]), ptr(outs["out"]),
                        route_struct(r))
    _lib.check(_lib.lib.nimg_moe_block_forward(C.byref(desc), C.byref(bp), int(layer), ptr(ws),
                                               ws.numel(), stream_handle()))
    res = [outs["out"]]
    if return_routing:
        decisions, routing = build_routing(r, B, S, E, cap)
        res += [decisions, routing]
    if return_intermediates:
        res.append({k: outs[k] for k in ("h", "x_norm", "x_mod")})
    return res[0] if len(res) == 1 else tuple(res)


def moe_block_prologue(x, sa_gate, r_attn, ff_scale, ff_gate, layer: int, cfg: RouterConfig):
    """backbone.py:584-589 alone, with the kernels moe_block_forward uses:
    returns (h, x_norm, x_mod, th_ff) where th_ff = tanh(ff_gate) in the
    precision of the combine epilogue (f64 for fp32 activations, fp32 for
    bf16). The expert-parallel block (ep.ep_moe_block_forward) runs the layer
    between this and a residual combine, so its output equals the 1-GPU block."""
    xt = to_device(x)
    act = xt.dtype
    B, S, d = xt.shape
    ra = to_device(r_attn, act)
    if tuple(ra.shape) != (B, S, d):
        raise ShapeError(f"r_attn shape {tuple(ra.shape)} != {(B, S, d)}")
    mods = [to_device(m, torch.float32) for m in (sa_gate, ff_scale, ff_gate)]
    for m in mods:
        if tuple(m.shape) != (B, d):
            raise ShapeError(f"modulation shape {tuple(m.shape)} != {(B, d)}")
    if d != cfg.d_model:
        raise ConfigError(f"width {d} != d_model {cfg.d_model}")
    cap = capacity_for(S, cfg.n_experts, cfg.capacity_factor)
    desc = make_desc(B, S, d, cfg.n_experts, cap, d, d, cfg, act)
    nbytes = C.c_size_t()
    _lib.check(_lib.lib.nimg_moe_block_prologue_workspace_bytes(C.byref(desc), C.byref(nbytes)))
    ws = workspace(nbytes.value)
    h, xn, xm = (torch.empty((B, S, d), dtype=act, device=xt.device) for _ in range(3))
    th = torch.empty((B, d), dtype=torch.float64 if act == torch.float32 else torch.float32,
                     device=xt.device)
    _lib.check(_lib.lib.nimg_moe_block_prologue(C.byref(desc), ptr(xt), ptr(ra), *(ptr(m) for m in mods),
                                                int(layer), ptr(h), ptr(xn), ptr(xm), ptr(th),
                                                ptr(ws), ws.numel(), stream_handle()))
    return h, xn, xm, th
