"""Sparse expert computation -- B200 operator API.

Mirrors /root/reference/pkg/src/nimg/moe.py (names, dataclasses, argument
meaning, exceptions). The whole layer -- routing, gather, the grouped SwiGLU
GEMMs (tcgen05 in bf16, CUDA cores in fp32), the deterministic weighted
combine and the shared expert -- is one call into libnimg_moe.so
(`nimg_moe_forward`); grouped_forward / swiglu call `nimg_expert_ffn`.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._tensors import any_f64, nimg_dtype, ptr, stream_handle, to_device, workspace
from .errors import ConfigError, ShapeError
from .router import (RouterConfig, alloc_route_out, build_routing, capacity_for, make_desc,
                     route_full, route_struct)

__all__ = ["ShapeError", "swiglu", "swiglu_arrays", "swiglu_composed", "ExpertBank",
           "GroupedBatch", "grouped_forward", "moe_forward"]


@dataclass
class ExpertBank:
    """moe.py:73-94 -- routed expert weights plus the always-on shared expert.
    w1, w3: (E, h, d); w2: (E, d, h); shared_w1/w3: (hs, d); shared_w2: (d, hs)."""
    w1: object
    w3: object
    w2: object
    shared_w1: object
    shared_w3: object
    shared_w2: object

    @property
    def n_experts(self) -> int:
        return self.w1.shape[0]

    def expert_weights(self, e: int):
        return self.w1[e], self.w3[e], self.w2[e]

    def on_device(self, dtype: torch.dtype) -> "ExpertBank":
        """Device copies in the kernel dtype (no copy if already there)."""
        return bank_on_device(self, dtype)


def bank_on_device(bank, dtype: torch.dtype) -> ExpertBank:
    """Any bank with w1..shared_w2 fields (ours or the reference's moe.ExpertBank,
    moe.py:73-94) -> device ExpertBank in the kernel dtype."""
    return ExpertBank(*(to_device(w, dtype) for w in (bank.w1, bank.w3, bank.w2, bank.shared_w1,
                                                      bank.shared_w3, bank.shared_w2)))


@dataclass
class GroupedBatch:
    """moe.py:97-112 -- expert-concatenated rows with prefix-sum offsets."""
    tokens: object            # (N_total, d)
    offsets: np.ndarray       # (E+1,) non-decreasing, offsets[0] == 0
    meta: dict = field(default_factory=dict)

    def __post_init__(self):
        off = np.asarray(self.offsets, dtype=np.int64)
        if off.ndim != 1 or off[0] != 0 or np.any(np.diff(off) < 0):
            raise ShapeError(f"invalid offsets {off}")
        if off[-1] != self.tokens.shape[0]:
            raise ShapeError(f"offsets end {off[-1]} != token count {self.tokens.shape[0]}")
        self.offsets = off


def _check_bank_shapes(w1, w3, w2, sw1, sw3, sw2, d):
    E, h, dd = w1.shape
    if dd != d or tuple(w3.shape) != (E, h, d) or tuple(w2.shape) != (E, d, h):
        raise ShapeError(f"expert weight shapes w1={tuple(w1.shape)} w3={tuple(w3.shape)} "
                         f"w2={tuple(w2.shape)} inconsistent with d={d}")
    hs = sw1.shape[0]
    if tuple(sw1.shape) != (hs, d) or tuple(sw3.shape) != (hs, d) or tuple(sw2.shape) != (d, hs):
        raise ShapeError(f"shared weight shapes {tuple(sw1.shape)} {tuple(sw3.shape)} "
                         f"{tuple(sw2.shape)} inconsistent with d={d}")
    return E, h, hs


def _ffn(x, offsets, experts, w1, w3, w2, out_dtype):
    """Run nimg_expert_ffn over routed segments only; returns (N, d)."""
    n, d = x.shape
    E, h, _ = w1.shape
    nseg = len(offsets) - 1
    desc = _lib.FfnDesc(n_rows=n, n_shared_rows=0, d=d, h=h, h_shared=h, n_experts=E,
                        act_dtype=nimg_dtype(x.dtype), nseg=nseg)
    path, ydt = C.c_int32(), C.c_int32()
    _lib.check(_lib.lib.nimg_ffn_path(C.byref(desc), C.byref(path), C.byref(ydt)))
    ytype = {_lib.NIMG_BF16: torch.bfloat16, _lib.NIMG_F32: torch.float32,
             _lib.NIMG_F64: torch.float64}[ydt.value]
    y = torch.empty((n, d), dtype=ytype, device=x.device)
    nbytes = C.c_size_t()
    _lib.check(_lib.lib.nimg_ffn_workspace_bytes(C.byref(desc), C.byref(nbytes)))
    ws = workspace(nbytes.value)
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    ex = np.ascontiguousarray(experts, dtype=np.int32)
    _lib.check(_lib.lib.nimg_expert_ffn(
        C.byref(desc), off.ctypes.data, ex.ctypes.data, ptr(x), ptr(w1), ptr(w3), ptr(w2), ptr(y),
        None, None, None, None, None, ptr(ws), ws.numel(), stream_handle()))
    return y if y.dtype == out_dtype else y.to(out_dtype)


def swiglu(x, w1, w3, w2):
    """moe.py:31-64 -- (SiLU(x W1^T) * (x W3^T)) W2^T on the GPU. Any float64
    operand runs the f64 mode (f64 internals and output, moe.py:42-51)."""
    xt = to_device(x, torch.float64 if any_f64(x, w1, w3, w2) else None)
    act = xt.dtype
    w1t, w3t, w2t = (to_device(w, act) for w in (w1, w3, w2))
    n, d = xt.shape[-2], xt.shape[-1]
    h = w1t.shape[0]
    if tuple(w1t.shape) != (h, d) or tuple(w3t.shape) != (h, d) or tuple(w2t.shape) != (d, h):
        raise ShapeError(f"swiglu weight shapes w1={tuple(w1t.shape)} w3={tuple(w3t.shape)} "
                         f"w2={tuple(w2t.shape)} inconsistent with d={d}")
    lead = xt.shape[:-1]
    x2 = xt.reshape(-1, d)
    y = _ffn(x2, [0, x2.shape[0]], [0], w1t[None], w3t[None], w2t[None], act)
    return y.reshape(*lead, d)


def swiglu_arrays(x, w1, w3, w2):
    """moe.py:20-28 -- same gated-linear forward on raw arrays (GPU)."""
    return swiglu(x, w1, w3, w2)


def swiglu_composed(x, w1, w3, w2):
    """moe.py:67-70 -- value-identical (within rounding) to swiglu."""
    return swiglu(x, w1, w3, w2)


def grouped_forward(batch: GroupedBatch, bank: ExpertBank):
    """moe.py:115-135 -- segment e through expert e; output keeps row order."""
    E = bank.n_experts
    if len(batch.offsets) != E + 1:
        raise ShapeError(f"offsets length {len(batch.offsets)} != E+1 ({E + 1})")
    x = to_device(batch.tokens,
                  torch.float64 if any_f64(batch.tokens, bank.w1, bank.w3, bank.w2) else None)
    act = x.dtype
    w1, w3, w2 = (to_device(w, act) for w in (bank.w1, bank.w3, bank.w2))
    E_, h, d = w1.shape
    if d != x.shape[1] or tuple(w3.shape) != (E, h, d) or tuple(w2.shape) != (E, d, h):
        raise ShapeError("expert weight shapes inconsistent with tokens")
    if x.shape[0] == 0:
        return torch.zeros((0, x.shape[1]), dtype=act, device=x.device)
    return _ffn(x, batch.offsets, np.arange(E, dtype=np.int32), w1, w3, w2, act)


def moe_forward(x, x_norm, x_mod, t_emb, cfg: RouterConfig, bank: ExpertBank, w_r,
                return_routing: bool = False):
    """moe.py:138-164 -- route on x_norm + t_emb, experts on x_mod.

    Returns (B, S, d) in the activation dtype of x_mod (fp32 or bf16); with
    return_routing, (out, decisions, routing) like the reference. Routing
    reads x_norm in its own dtype (router.py:120-122). If any input or weight
    is float64 the whole layer runs in the reference's f64 mode (f64 routing,
    experts, combine and output; np.result_type promotion, tensor.py:203-204).
    When grad mode is on and any input or expert weight requires grad, the
    layer is recorded on the autograd tape (training forward +
    nimg_moe_backward), the way the reference's moe_forward records tape nodes.
    """
    B, S, d = x.shape
    cfg.validate_weight(w_r)
    f64 = any_f64(x_norm, x_mod, t_emb, w_r, bank.w1, bank.w3, bank.w2, bank.shared_w1,
                  bank.shared_w3, bank.shared_w2)
    xm = to_device(x_mod, torch.float64 if f64 else None)
    act = xm.dtype
    xn = to_device(x_norm, act if f64 else None)
    if tuple(xm.shape) != (B, S, d) or tuple(xn.shape) != (B, S, d):
        raise ShapeError(f"x_norm {tuple(xn.shape)} / x_mod {tuple(xm.shape)} != {(B, S, d)}")
    vdt = torch.float64 if f64 else torch.float32
    te = to_device(t_emb, vdt)
    wr = to_device(w_r, vdt)
    if tuple(te.shape) != (B, d):
        raise ConfigError(f"t_emb shape {tuple(te.shape)}, expected {(B, d)}")
    E = cfg.n_experts
    if bank.n_experts != E:
        raise ConfigError(f"bank has {bank.n_experts} experts, router {E}")
    cap = capacity_for(S, E, cfg.capacity_factor)
    if cap < 1:
        raise ConfigError("computed capacity is zero")
    w = bank_on_device(bank, act)
    _, h, hs = _check_bank_shapes(w.w1, w.w3, w.w2, w.shared_w1, w.shared_w3, w.shared_w2, d)

    desc = make_desc(B, S, d, E, cap, h, hs, cfg, act, xn.dtype)
    if _wants_grad(xn, xm, te, wr, w.w1, w.w3, w.w2, w.shared_w1, w.shared_w3, w.shared_w2):
        if f64:
            raise ConfigError("the f64 mode is forward-only: no training path in float64")
        if xn.dtype != act:
            raise ConfigError(f"training needs x_norm in x_mod's dtype ({xn.dtype} != {act})")
        meta = {"desc": desc, "shape": (B, S, d, E, cap, h, hs)}
        out = _MoELayerFn.apply(meta, xn, xm, te, wr, w.w1, w.w3, w.w2, w.shared_w1,
                                w.shared_w3, w.shared_w2)
        if return_routing:
            decisions, routing = build_routing(meta["route"], B, S, E, cap)
            return out, decisions, routing
        return out
    nbytes = C.c_size_t()
    _lib.check(_lib.lib.nimg_moe_workspace_bytes(C.byref(desc), C.byref(nbytes)))
    ws = workspace(nbytes.value)
    out = torch.empty((B, S, d), dtype=act, device=xm.device)
    r = alloc_route_out(B, S, E, cap, xm.device, vdt)
    ptrs = _lib.MoePtrs(ptr(xn), ptr(xm), ptr(te), ptr(wr), ptr(w.w1), ptr(w.w3), ptr(w.w2),
                        ptr(w.shared_w1), ptr(w.shared_w3), ptr(w.shared_w2), ptr(out),
                        route_struct(r))
    _lib.check(_lib.lib.nimg_moe_forward(C.byref(desc), C.byref(ptrs), ptr(ws), ws.numel(),
                                         stream_handle()))
    if return_routing:
        decisions, routing = build_routing(r, B, S, E, cap)
        return out, decisions, routing
    return out


def _wants_grad(*ts) -> bool:
    return torch.is_grad_enabled() and any(isinstance(t, torch.Tensor) and t.requires_grad
                                           for t in ts)


def _sizeof(fn, desc) -> int:
    n = C.c_size_t()
    _lib.check(fn(C.byref(desc), C.byref(n)))
    return n.value


class _MoELayerFn(torch.autograd.Function):
    """moe_forward on the autograd tape: nimg_moe_forward_train keeps what the
    pullback needs; backward() is nimg_moe_backward -- the gradients the
    reference's backward(tape, loss) accumulates through moe.py:138-164
    (tensor.py:590-628): x_norm, x_mod, t_emb, w_r and every expert weight."""

    @staticmethod
    def forward(ctx, meta, xn, xm, te, wr, w1, w3, w2, sw1, sw3, sw2):
        desc = meta["desc"]
        B, S, d, E, cap, h, hs = meta["shape"]
        dev = xm.device
        ws = workspace(_sizeof(_lib.lib.nimg_moe_workspace_bytes, desc))
        state = workspace(_sizeof(_lib.lib.nimg_moe_train_state_bytes, desc))
        out = torch.empty((B, S, d), dtype=xm.dtype, device=dev)
        r = alloc_route_out(B, S, E, cap, dev)
        ptrs = _lib.MoePtrs(ptr(xn), ptr(xm), ptr(te), ptr(wr), ptr(w1), ptr(w3), ptr(w2),
                            ptr(sw1), ptr(sw3), ptr(sw2), ptr(out), route_struct(r))
        _lib.check(_lib.lib.nimg_moe_forward_train(C.byref(desc), C.byref(ptrs), ptr(state),
                                                   state.numel(), ptr(ws), ws.numel(),
                                                   stream_handle()))
        meta["route"] = r
        ctx.meta, ctx.r, ctx.state = meta, r, state
        ctx.save_for_backward(xn, xm, te, wr, w1, w3, w2, sw1, sw3, sw2)
        return out

    @staticmethod
    def backward(ctx, g_out):
        xn, xm, te, wr, w1, w3, w2, sw1, sw3, sw2 = ctx.saved_tensors
        desc, r = ctx.meta["desc"], ctx.r
        g_out = g_out.to(xm.dtype).contiguous()
        ws = workspace(_sizeof(_lib.lib.nimg_moe_backward_workspace_bytes, desc))
        f32 = torch.float32
        g = {"x_norm": torch.empty_like(xn), "x_mod": torch.empty_like(xm),
             "t_emb": torch.empty(te.shape, dtype=f32, device=xm.device),
             "w_r": torch.empty(wr.shape, dtype=f32, device=xm.device)}
        for k, t in (("w1", w1), ("w3", w3), ("w2", w2), ("sw1", sw1), ("sw3", sw3),
                     ("sw2", sw2)):
            g[k] = torch.empty(t.shape, dtype=f32, device=xm.device)
        ptrs = _lib.MoePtrs(ptr(xn), ptr(xm), ptr(te), ptr(wr), ptr(w1), ptr(w3), ptr(w2),
                            ptr(sw1), ptr(sw3), ptr(sw2), None, route_struct(r))
        grads = _lib.MoeGrads(ptr(g_out), *(ptr(g[k]) for k in ("x_norm", "x_mod", "t_emb", "w_r",
                                                                 "w1", "w3", "w2", "sw1", "sw3",
                                                                 "sw2")))
        _lib.check(_lib.lib.nimg_moe_backward(C.byref(desc), C.byref(ptrs), ptr(ctx.state),
                                              ctx.state.numel(), C.byref(grads), ptr(ws),
                                              ws.numel(), stream_handle()))
        return (None, g["x_norm"], g["x_mod"], g["t_emb"], g["w_r"], g["w1"], g["w3"], g["w2"],
                g["sw1"], g["sw3"], g["sw2"])


class MoEPlan:
    """Pre-planned MoE layer for a fixed problem shape (serving / benchmark path).

    Owns the workspace, output and routing buffers so a forward is one C-ABI
    call (`nimg_moe_forward`) with no allocation; `capture()` records that call
    in a CUDA graph on static input buffers. Same arithmetic as moe_forward.
    """

    def __init__(self, cfg: RouterConfig, bank: ExpertBank, B: int, S: int,
                 act: torch.dtype = torch.bfloat16):
        self.cfg, self.B, self.S, self.act = cfg, B, S, act
        d, E = cfg.d_model, cfg.n_experts
        self.bank = bank_on_device(bank, act)
        _, self.h, self.hs = _check_bank_shapes(self.bank.w1, self.bank.w3, self.bank.w2,
                                                self.bank.shared_w1, self.bank.shared_w3,
                                                self.bank.shared_w2, d)
        self.cap = capacity_for(S, E, cfg.capacity_factor)
        self.desc = make_desc(B, S, d, E, self.cap, self.h, self.hs, cfg, act)
        nbytes = C.c_size_t()
        _lib.check(_lib.lib.nimg_moe_workspace_bytes(C.byref(self.desc), C.byref(nbytes)))
        self.ws = workspace(nbytes.value)
        dev = self.ws.device
        self.out = torch.empty((B, S, d), dtype=act, device=dev)
        self.r = alloc_route_out(B, S, E, self.cap, dev)
        self.graph = None

    def _ptrs(self, x_norm, x_mod, t_emb, w_r):
        w = self.bank
        return _lib.MoePtrs(ptr(x_norm), ptr(x_mod), ptr(t_emb), ptr(w_r), ptr(w.w1), ptr(w.w3),
                            ptr(w.w2), ptr(w.shared_w1), ptr(w.shared_w3), ptr(w.shared_w2),
                            ptr(self.out), route_struct(self.r))

    def forward(self, x_norm, x_mod, t_emb, w_r) -> torch.Tensor:
        """Inputs must already be contiguous CUDA tensors of the plan's dtypes
        (x_norm/x_mod act dtype, t_emb/w_r fp32). Returns the plan's out buffer."""
        p = self._ptrs(x_norm, x_mod, t_emb, w_r)
        _lib.check(_lib.lib.nimg_moe_forward(C.byref(self.desc), C.byref(p), ptr(self.ws),
                                             self.ws.numel(), stream_handle()))
        return self.out

    def capture(self, x_norm, x_mod, t_emb, w_r) -> "torch.cuda.CUDAGraph":
        """Record forward() on these (static) input buffers into a CUDA graph."""
        self.forward(x_norm, x_mod, t_emb, w_r)  # warm (attributes, tensor-map fn)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.forward(x_norm, x_mod, t_emb, w_r)
        self.graph = g
        return g

    def routing(self, with_decisions: bool = False):
        return build_routing(self.r, self.B, self.S, self.cfg.n_experts, self.cap, with_decisions)


class MoETrainPlan:
    """Pre-planned training step of the layer for a fixed shape (benchmark /
    trainer path): owns the training state, both workspaces, routing buffers
    and gradient buffers, so forward() and backward() are one C-ABI call each
    (nimg_moe_forward_train, nimg_moe_backward) with no allocation. Same
    arithmetic as the autograd path of moe_forward."""

    def __init__(self, cfg: RouterConfig, bank: ExpertBank, B: int, S: int,
                 act: torch.dtype = torch.bfloat16):
        self.cfg, self.B, self.S, self.act = cfg, B, S, act
        d, E = cfg.d_model, cfg.n_experts
        self.bank = bank_on_device(bank, act)
        w = self.bank
        _, self.h, self.hs = _check_bank_shapes(w.w1, w.w3, w.w2, w.shared_w1, w.shared_w3,
                                                w.shared_w2, d)
        self.cap = capacity_for(S, E, cfg.capacity_factor)
        self.desc = make_desc(B, S, d, E, self.cap, self.h, self.hs, cfg, act)
        self.ws = workspace(_sizeof(_lib.lib.nimg_moe_workspace_bytes, self.desc))
        self.state = workspace(_sizeof(_lib.lib.nimg_moe_train_state_bytes, self.desc))
        self.bws = workspace(_sizeof(_lib.lib.nimg_moe_backward_workspace_bytes, self.desc))
        dev = self.ws.device
        self.out = torch.empty((B, S, d), dtype=act, device=dev)
        self.r = alloc_route_out(B, S, E, self.cap, dev)
        f32 = torch.float32
        self.grads = {"x_norm": torch.empty((B, S, d), dtype=act, device=dev),
                      "x_mod": torch.empty((B, S, d), dtype=act, device=dev),
                      "t_emb": torch.empty((B, d), dtype=f32, device=dev),
                      "w_r": torch.empty((2 * d, E), dtype=f32, device=dev)}
        for k, t in (("w1", w.w1), ("w3", w.w3), ("w2", w.w2), ("sw1", w.shared_w1),
                     ("sw3", w.shared_w3), ("sw2", w.shared_w2)):
            self.grads[k] = torch.empty(t.shape, dtype=f32, device=dev)
        self._inputs = None

    def _ptrs(self, x_norm, x_mod, t_emb, w_r, out):
        w = self.bank
        return _lib.MoePtrs(ptr(x_norm), ptr(x_mod), ptr(t_emb), ptr(w_r), ptr(w.w1), ptr(w.w3),
                            ptr(w.w2), ptr(w.shared_w1), ptr(w.shared_w3), ptr(w.shared_w2),
                            ptr(out), route_struct(self.r))

    def forward(self, x_norm, x_mod, t_emb, w_r) -> torch.Tensor:
        """Contiguous CUDA inputs of the plan's dtypes; returns the out buffer."""
        self._inputs = (x_norm, x_mod, t_emb, w_r)
        p = self._ptrs(x_norm, x_mod, t_emb, w_r, self.out)
        _lib.check(_lib.lib.nimg_moe_forward_train(C.byref(self.desc), C.byref(p), ptr(self.state),
                                                   self.state.numel(), ptr(self.ws),
                                                   self.ws.numel(), stream_handle()))
        return self.out

    def backward(self, g_out) -> dict:
        """Gradients of the last forward() for upstream gradient g_out (act
        dtype, contiguous); returns the plan's gradient buffers."""
        if self._inputs is None:
            raise RuntimeError("backward() before forward()")
        p = self._ptrs(*self._inputs, None)
        g = self.grads
        grads = _lib.MoeGrads(ptr(g_out), *(ptr(g[k]) for k in ("x_norm", "x_mod", "t_emb", "w_r",
                                                                 "w1", "w3", "w2", "sw1", "sw3",
                                                                 "sw2")))
        _lib.check(_lib.lib.nimg_moe_backward(C.byref(self.desc), C.byref(p), ptr(self.state),
                                              self.state.numel(), C.byref(grads), ptr(self.bws),
                                              self.bws.numel(), stream_handle()))
        return g
