"""Drop-in installation of the GPU layer into the reference's own MoE block.

The reference's `MoEDiT.forward` calls `moe_forward` through the name its
backbone module bound at import (`from .moe import ... moe_forward`,
backbone.py:24; the call is backbone.py:595-597), so the drop-in rebinds
**that** name:

    import nimg.backbone as bb
    from paper_2604_12163_b200 import compat
    compat.install(bb)          # bb.moe_forward now runs on the B200
    vel, aux = model.forward(z, t, ctx, stage)
    compat.uninstall(bb)

`install` returns the adapter. It speaks the reference's types on both sides:

* Inputs are the reference's `Tensor`s (numpy `.data`), `RouterConfig` and
  `ExpertBank` (moe.py:73-94). Expert weights are uploaded once and stay
  device-resident across calls, keyed by the identity of their numpy arrays
  (the adapter holds a reference, so an id cannot be reused). A caller that
  edits weights in place between calls calls `clear_weight_cache()`.
* The dtype follows the reference's promotion rule (np.result_type,
  tensor.py:203-204): if any operand is float64 -- as in the backbone, whose
  timestep features promote the MoE inputs to f64 (backbone.py:259-261) --
  the layer runs in the f64 mode (csrc/f64_kernels.cu); otherwise in fp32.
  Nothing is silently downcast.
* The output is a reference `Tensor` of that dtype. `routing` holds reference
  `Tensor`s for "gates" and "logits", the int64 numpy "token_flat", the
  capacity and the shape (router.py:155-161); `decisions` are the reference's
  `RouterDecision`s (router.py:59-67, :145-153). So `fused_gated_residual`
  (backbone.py:47-51) and the aux bookkeeping (backbone.py:598-605) work as
  with the stock layer.
* Errors are raised as the reference's `ConfigError` / `ShapeError`.
* Under the reference's tape (grad enabled, an active Tape and an input with
  requires_grad, tensor.py:190-200) the layer is recorded as ONE tape node
  whose pullback runs nimg_moe_backward (fp32 mode); the f64 mode is
  forward-only and raises ConfigError there.
"""

from __future__ import annotations

import importlib
import sys

import numpy as np
import torch

from . import moe as _moe
from .errors import ConfigError, ShapeError

__all__ = ["install", "uninstall", "make_moe_forward", "clear_weight_cache"]

_WEIGHTS: dict = {}


def clear_weight_cache() -> None:
    """Drop the device copies of expert weights (after in-place edits)."""
    _WEIGHTS.clear()


def _arr(x) -> np.ndarray:
    a = getattr(x, "data", x)
    return a if isinstance(a, np.ndarray) else np.asarray(a)


def _device_weight(w, dtype: torch.dtype) -> torch.Tensor:
    a = _arr(w)
    key = (id(a), a.__array_interface__["data"][0], a.shape, a.dtype.str, dtype)
    hit = _WEIGHTS.get(key)
    if hit is None:
        t = torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)
        hit = _WEIGHTS[key] = (a, t)   # keep `a` alive: its id stays unique
    return hit[1]


def _ref_modules(backbone_module):
    pkg = backbone_module.__name__.rsplit(".", 1)[0]
    nt = sys.modules.get(pkg + ".tensor") or importlib.import_module(pkg + ".tensor")
    rt = sys.modules.get(pkg + ".router") or importlib.import_module(pkg + ".router")
    return nt, rt


def _tracking(nt, tensors) -> bool:
    """tensor.py:190-195: a node is recorded iff grad is on, a tape is active
    and some input requires grad."""
    return (getattr(nt, "_GRAD_ENABLED", False) and nt.active_tape() is not None
            and any(getattr(t, "requires_grad", False) for t in tensors))


def make_moe_forward(backbone_module):
    """The adapter bound in place of backbone_module.moe_forward."""
    nt, rt = _ref_modules(backbone_module)
    RefTensor = nt.Tensor
    RefConfigError = getattr(rt, "ConfigError", ConfigError)
    RefShapeError = getattr(nt, "ShapeError", ShapeError)
    RefDecision = rt.RouterDecision

    def moe_forward(x, x_norm, x_mod, t_emb, cfg, bank, w_r, return_routing=False):
        """moe.py:138-164 on the B200; reference types in and out."""
        weights = (bank.w1, bank.w3, bank.w2, bank.shared_w1, bank.shared_w3, bank.shared_w2)
        operands = (x_norm, x_mod, t_emb, w_r) + weights
        out_np_dtype = np.result_type(*(_arr(t).dtype for t in operands))
        if out_np_dtype not in (np.float32, np.float64):
            raise RefConfigError(f"unsupported dtype {out_np_dtype}")
        dt = torch.float64 if out_np_dtype == np.float64 else torch.float32
        track = _tracking(nt, operands)
        if track and dt == torch.float64:
            raise RefConfigError("the B200 layer's f64 mode is forward-only; record the tape in "
                                 "fp32 (no float64 operands) to train through it")
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(_arr(a))).to("cuda", dt)
        xn, xm, te, wr = (dev(a) for a in (x_norm, x_mod, t_emb, w_r))
        if track:
            xn, xm, te, wr = (t.requires_grad_(True) for t in (xn, xm, te, wr))
            wts = [dev(w).requires_grad_(True) for w in weights]
        else:
            wts = [_device_weight(w, dt) for w in weights]
        dbank = _moe.ExpertBank(*wts)
        try:
            with torch.enable_grad() if track else torch.no_grad():
                out, decisions, routing = _moe.moe_forward(x, xn, xm, te, cfg, dbank, wr,
                                                           return_routing=True)
        except ConfigError as e:
            raise RefConfigError(str(e)) from None
        except ShapeError as e:
            raise RefShapeError(str(e)) from None
        out_np = out.detach().cpu().numpy().astype(out_np_dtype, copy=False)
        if track:
            leaves = [xn, xm, te, wr] + wts

            def bwd(g):
                grads = torch.autograd.grad(out, leaves, torch.from_numpy(g).to(out),
                                            retain_graph=True, allow_unused=True)
                return tuple(None if gr is None else gr.double().cpu().numpy() for gr in grads)

            # one tape node over the layer's differentiable inputs (x is shape-only, moe.py:146)
            res = nt.record("moe_forward_b200", tuple(operands), (out_np,), bwd)[0]
        else:
            res = RefTensor(out_np, dtype=out_np.dtype)
        if not return_routing:
            return res
        gdt = out_np_dtype if dt == torch.float64 else np.float32
        ref_routing = {
            "gates": RefTensor(routing["gates"].cpu().numpy().astype(gdt), dtype=gdt),
            "logits": RefTensor(routing["logits"].cpu().numpy().astype(gdt), dtype=gdt),
            "token_flat": routing["token_flat"].cpu().numpy().astype(np.int64),
            "capacity": routing["capacity"],
            "shape": routing["shape"],
        }
        ref_decisions = [RefDecision(top_indices=d.top_indices, affinity=d.affinity, gates=d.gates,
                                     logits=d.logits, capacity=d.capacity) for d in decisions]
        return res, ref_decisions, ref_routing

    moe_forward.__nimg_b200__ = True
    return moe_forward


def install(backbone_module=None):
    """Rebind backbone_module.moe_forward (default: the importable `nimg.backbone`)
    to the B200 layer; returns the adapter. Idempotent."""
    mod = backbone_module or importlib.import_module("nimg.backbone")
    cur = mod.moe_forward
    if getattr(cur, "__nimg_b200__", False):
        return cur
    fn = make_moe_forward(mod)
    fn.__nimg_prev__ = cur
    mod.moe_forward = fn
    return fn


def uninstall(backbone_module=None) -> None:
    """Restore the reference's own moe_forward."""
    mod = backbone_module or importlib.import_module("nimg.backbone")
    prev = getattr(mod.moe_forward, "__nimg_prev__", None)
    if prev is not None:
        mod.moe_forward = prev
