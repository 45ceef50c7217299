"""Expert-choice routing on decoupled inputs -- B200 operator API.

Mirrors /root/reference/pkg/src/nimg/router.py: same names, fields, argument
meaning and exceptions. The routing pass itself (f64-accumulated logits,
softmax, per-(sample, expert) top-capacity radix-select, gate
renormalisation) runs in libnimg_moe.so (`nimg_route`).
"""

from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._tensors import any_f64, nimg_dtype, ptr, stream_handle, to_device, workspace
from .errors import ConfigError

__all__ = ["ConfigError", "StageId", "DENSE", "RouterConfig", "RouterDecision",
           "capacity_for", "capacity_schedule", "route_full", "route"]


class StageId(enum.Enum):
    """router.py:26-29"""
    S256 = "s256"
    S512 = "s512"
    S1024 = "s1024"


#: Sentinel returned by capacity_schedule for layers that run a dense FFN (router.py:33).
DENSE = "dense"


@dataclass
class RouterConfig:
    """router.py:36-56"""
    d_model: int
    n_experts: int
    capacity_factor: float
    gate_scale: float = 1.0
    gate_eps: float = 1e-6
    seed: int = 0

    def __post_init__(self):
        if self.n_experts < 1:
            raise ConfigError("n_experts must be >= 1")
        if self.capacity_factor <= 0:
            raise ConfigError("capacity_factor must be > 0")
        if self.gate_eps <= 0:
            raise ConfigError("gate_eps must be > 0")

    def validate_weight(self, w_r) -> None:
        want = (2 * self.d_model, self.n_experts)
        if tuple(w_r.shape) != want:
            raise ConfigError(f"router weight shape {tuple(w_r.shape)}, expected {want}")


@dataclass
class RouterDecision:
    """router.py:59-67 -- detached record of one routing pass over one sample."""
    top_indices: np.ndarray   # (E, capacity) token positions
    affinity: np.ndarray      # (E, capacity) raw softmax scores
    gates: np.ndarray         # (E, capacity) normalized * gate_scale
    logits: np.ndarray        # (S, E)
    capacity: int


def capacity_for(S: int, E: int, C_: float) -> int:
    """router.py:70-74 -- per-expert token budget ceil(C*S/E), clamped to S."""
    if S < 1 or E < 1 or C_ <= 0:
        raise ConfigError(f"invalid capacity arguments S={S} E={E} C={C_}")
    return min(math.ceil(C_ * S / E), S)


def capacity_schedule(layer: int, stage: StageId, n_layers: int = 32):
    """router.py:77-95 -- DENSE for layers 0-2; 8/4/(4,2) by stage."""
    if not 0 <= layer < n_layers:
        raise IndexError(f"layer {layer} out of range [0, {n_layers})")
    if layer < 3:
        return DENSE
    if stage == StageId.S256:
        return 8.0
    if stage == StageId.S512:
        return 4.0
    if stage == StageId.S1024:
        return 4.0 if layer <= 4 else 2.0
    raise ConfigError(f"unknown stage {stage!r}")


def make_desc(B, S, d, E, cap, h, hs, cfg: RouterConfig, act: torch.dtype,
              router: torch.dtype | None = None) -> _lib.MoeDesc:
    """act: dtype of x_mod / expert weights / out; router: dtype of x_norm
    (default act). float64 (both) is the reference's f64 storage mode."""
    return _lib.MoeDesc(B=B, S=S, d=d, E=E, cap=cap, h=h, h_shared=hs,
                        gate_scale=float(cfg.gate_scale), gate_eps=float(cfg.gate_eps),
                        act_dtype=nimg_dtype(act), router_dtype=nimg_dtype(router or act),
                        gate_scale_f64=float(cfg.gate_scale), gate_eps_f64=float(cfg.gate_eps))


def alloc_route_out(B: int, S: int, E: int, cap: int, dev, value_dtype=torch.float32) -> dict:
    """Routing buffers; logits / scores / gates are fp32, or float64 in the f64 mode."""
    n = E * B * cap
    f32, i32 = value_dtype, torch.int32
    return {
        "logits": torch.empty((B, S, E), dtype=f32, device=dev),
        "scores_bes": torch.empty((B, E, S), dtype=f32, device=dev),
        "token_flat": torch.empty(n, dtype=i32, device=dev),
        "gate_raw": torch.empty(n, dtype=f32, device=dev),
        "gates": torch.empty(n, dtype=f32, device=dev),
        "comb_rows": torch.empty((B * S, E), dtype=i32, device=dev),
        "comb_cnt": torch.empty(B * S, dtype=i32, device=dev),
    }


def route_struct(r: dict) -> _lib.RouteOut:
    return _lib.RouteOut(*(ptr(r[k]) for k in ("logits", "scores_bes", "token_flat", "gate_raw",
                                                "gates", "comb_rows", "comb_cnt")))


def build_routing(r: dict, B: int, S: int, E: int, cap: int, with_decisions: bool = True):
    """Assemble the reference's (decisions, routing) pair (router.py:145-161).
    Decisions are detached host copies, as in the reference."""
    routing = {
        "gates": r["gates"],
        "logits": r["logits"],
        "token_flat": r["token_flat"].to(torch.int64),
        "capacity": cap,
        "shape": (B, S, E),
        # device-side extras used by the MoE layer / expert parallel path
        # (comb_rows / comb_cnt are filled by route() and the training forward;
        # the 1-GPU inference forward forms the gates in its combine instead)
        "gate_raw": r["gate_raw"],
        "scores_bes": r["scores_bes"],
        "comb_rows": r["comb_rows"],
        "comb_cnt": r["comb_cnt"],
        "token_flat_i32": r["token_flat"],
    }
    if not with_decisions:
        return None, routing
    tf = r["token_flat"].view(E, B, cap).cpu().numpy().astype(np.int64)
    aff = r["gate_raw"].view(E, B, cap).cpu().numpy().astype(np.float64)
    gts = r["gates"].view(E, B, cap).cpu().numpy().astype(np.float64)
    lg = r["logits"].cpu().numpy().astype(np.float64)
    decisions = [RouterDecision(top_indices=tf[:, b, :] - b * S, affinity=aff[:, b, :].copy(),
                                gates=gts[:, b, :].copy(), logits=lg[b].copy(), capacity=cap)
                 for b in range(B)]
    return decisions, routing


def route_full(x_norm, t_emb, w_r, cfg: RouterConfig):
    """router.py:104-162 -- routing pass; returns (decisions, routing).

    x_norm (B,S,d) fp32 or bf16; t_emb (B,d); w_r (2d,E). Logits and scores
    are fp32 (bit-exact with the reference's fp32 mode); token_flat is the
    expert-major (e, b, slot) flat row index into (B*S, d). If any input is
    float64, routing runs in the reference's f64 mode (logits, scores and
    gates stay float64, router.py:120-143).
    """
    cfg.validate_weight(w_r)
    f64 = any_f64(x_norm, t_emb, w_r)
    xn = to_device(x_norm, torch.float64 if f64 else None)
    B, S, d = xn.shape
    E = cfg.n_experts
    if d != cfg.d_model:
        raise ConfigError(f"x_norm width {d} != d_model {cfg.d_model}")
    cap = capacity_for(S, E, cfg.capacity_factor)
    if cap < 1:
        raise ConfigError("computed capacity is zero")
    vdt = torch.float64 if f64 else torch.float32
    te = to_device(t_emb, vdt)
    wr = to_device(w_r, vdt)
    if tuple(te.shape) != (B, d):
        raise ConfigError(f"t_emb shape {tuple(te.shape)}, expected {(B, d)}")
    desc = make_desc(B, S, d, E, cap, 1, 1, cfg, xn.dtype)
    nbytes = C.c_size_t()
    _lib.check(_lib.lib.nimg_route_workspace_bytes(C.byref(desc), C.byref(nbytes)))
    ws = workspace(nbytes.value)
    r = alloc_route_out(B, S, E, cap, xn.device, vdt)
    ro = route_struct(r)
    _lib.check(_lib.lib.nimg_route(C.byref(desc), ptr(xn), ptr(te), ptr(wr), C.byref(ro),
                                   ptr(ws), ws.numel(), stream_handle()))
    return build_routing(r, B, S, E, cap)


def route(x_norm, t_emb, w_r, cfg: RouterConfig) -> list[RouterDecision]:
    """router.py:165-170 -- one detached RouterDecision per sample."""
    decisions, _ = route_full(x_norm, t_emb, w_r, cfg)
    return decisions
