"""Stage-level wrappers over the C ABI (route / gather / expert FFN / combine).

These are the building blocks the expert-parallel path composes around its
all-to-all exchanges; `moe.moe_forward` uses the fused `nimg_moe_forward`
entry point instead. Every function enqueues CUDA work on the current torch
stream and allocates its outputs with torch (the C ABI never allocates).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from ._tensors import nimg_dtype, ptr, stream_handle, workspace
from .router import RouterConfig, alloc_route_out, make_desc, route_struct


class CudaStages:
    """The production backend: every stage is a libnimg_moe.so call."""

    name = "cuda"

    def route(self, x_norm: torch.Tensor, t_emb: torch.Tensor, w_r: torch.Tensor,
              cfg: RouterConfig, cap: int, for_combine: bool = False) -> dict:
        """router.py:104-162 on (B,S,d) x_norm; returns the device routing dict.
        for_combine: when the shape allows it (nimg_route_fusable), the gates
        are left to combine() (nimg_route_for_combine / nimg_combine_routed):
        no gate kernel, and gates / comb_rows / comb_cnt are valid only after
        combine() ran."""
        B, S, d = x_norm.shape
        desc = make_desc(B, S, d, cfg.n_experts, cap, 1, 1, cfg, x_norm.dtype)
        nbytes = C.c_size_t()
        _lib.check(_lib.lib.nimg_route_workspace_bytes(C.byref(desc), C.byref(nbytes)))
        ws = workspace(nbytes.value)
        r = alloc_route_out(B, S, cfg.n_experts, cap, x_norm.device)
        ro = route_struct(r)
        fused = for_combine and _lib.lib.nimg_route_fusable(C.byref(desc)) == 1
        fn = _lib.lib.nimg_route_for_combine if fused else _lib.lib.nimg_route
        _lib.check(fn(C.byref(desc), ptr(x_norm), ptr(t_emb), ptr(w_r), C.byref(ro), ptr(ws),
                      ws.numel(), stream_handle()))
        r["_route_ws"], r["_route_desc"] = ws, desc   # bg_flags() points into ws
        r["_fused"] = fused
        return r

    def bg_flags(self, r: dict) -> int:
        """Device address of the gather flags nimg_route zeroed in this
        routing's workspace (nimg_route_bg_flags); 0 if unavailable."""
        if "_route_ws" not in r:
            return 0
        p = C.c_void_p()
        _lib.check(_lib.lib.nimg_route_bg_flags(C.byref(r["_route_desc"]), ptr(r["_route_ws"]),
                                                C.byref(p)))
        return p.value or 0

    def gather(self, src: torch.Tensor, idx_i32: torch.Tensor, out: torch.Tensor | None = None
               ) -> torch.Tensor:
        """tensor.py:348-363 gather_rows: src (N, d)[idx] -> (len(idx), d)."""
        n, d = src.shape
        if out is None:
            out = torch.empty((idx_i32.numel(), d), dtype=src.dtype, device=src.device)
        _lib.check(_lib.lib.nimg_gather_rows(ptr(src), n, d * src.element_size(), ptr(idx_i32),
                                             idx_i32.numel(), ptr(out), stream_handle()))
        return out

    def ffn_y_dtype(self, act: torch.dtype, d: int, h: int, hs: int) -> torch.dtype:
        desc = _lib.FfnDesc(n_rows=1, n_shared_rows=1, d=d, h=h, h_shared=hs, n_experts=1,
                            act_dtype=nimg_dtype(act), nseg=1)
        path, ydt = C.c_int32(), C.c_int32()
        _lib.check(_lib.lib.nimg_ffn_path(C.byref(desc), C.byref(path), C.byref(ydt)))
        return torch.bfloat16 if ydt.value == _lib.NIMG_BF16 else torch.float32

    def expert_ffn(self, x_routed: torch.Tensor | None, seg_offsets: np.ndarray,
                   seg_expert: np.ndarray, w1, w3, w2, x_shared: torch.Tensor | None,
                   sw1, sw3, sw2, y_routed: torch.Tensor | None = None,
                   y_shared: torch.Tensor | None = None, gather: dict | None = None):
        """moe.py:115-135 + moe.py:160: routed segments through their experts
        and (optionally) x_shared through the shared expert, one grouped launch
        per GEMM. Returns (y_routed, y_shared).

        gather (expert parallel): {src, idx, dst, flags, row_off, chunk_rows,
        chunk_done} -- the launch itself gathers dst[r] = src[idx[r]] for all
        of dst (moe.py:152-153) while it runs; x_routed is rows row_off.. of
        dst (nimg_expert_ffn_gather)."""
        act = (x_routed if x_routed is not None else x_shared).dtype
        nr = 0 if x_routed is None else x_routed.shape[0]
        ns = 0 if x_shared is None else x_shared.shape[0]
        d = (x_routed if x_routed is not None else x_shared).shape[1]
        E, h = (w1.shape[0], w1.shape[1]) if w1 is not None else (1, sw1.shape[0])
        hs = sw1.shape[0] if sw1 is not None else h
        nseg = len(seg_offsets) - 1 if nr > 0 else 0
        desc = _lib.FfnDesc(n_rows=nr, n_shared_rows=ns, d=d, h=h, h_shared=hs, n_experts=E,
                            act_dtype=nimg_dtype(act), nseg=nseg)
        ydt = self.ffn_y_dtype(act, d, h, hs)
        dev = (x_routed if x_routed is not None else x_shared).device
        if nr and y_routed is None:
            y_routed = torch.empty((nr, d), dtype=ydt, device=dev)
        if ns and y_shared is None:
            y_shared = torch.empty((ns, d), dtype=ydt, device=dev)
        nbytes = C.c_size_t()
        _lib.check(_lib.lib.nimg_ffn_workspace_bytes(C.byref(desc), C.byref(nbytes)))
        ws = workspace(nbytes.value)
        off = np.ascontiguousarray(seg_offsets if nseg else [0], dtype=np.int64)
        ex = np.ascontiguousarray(seg_expert if nseg else [0], dtype=np.int32)
        args = (C.byref(desc), off.ctypes.data if nseg else None, ex.ctypes.data if nseg else None,
                ptr(x_routed) if nr else None, ptr(w1) if nr else None, ptr(w3) if nr else None,
                ptr(w2) if nr else None, ptr(y_routed) if nr else None,
                ptr(x_shared) if ns else None, ptr(sw1) if ns else None, ptr(sw3) if ns else None,
                ptr(sw2) if ns else None, ptr(y_shared) if ns else None, ptr(ws), ws.numel())
        if gather is None:
            _lib.check(_lib.lib.nimg_expert_ffn(*args, stream_handle()))
        else:
            dst = gather["dst"]
            g = _lib.BgGatherDesc(src=ptr(gather["src"]), idx=ptr(gather["idx"]), dst=ptr(dst),
                                  flags=gather["flags"], chunk_done=gather.get("chunk_done"),
                                  rows=dst.shape[0], row_bytes=dst.shape[1] * dst.element_size(),
                                  row_off=gather.get("row_off", 0),
                                  chunk_rows=gather.get("chunk_rows", 0))
            _lib.check(_lib.lib.nimg_expert_ffn_gather(*args, C.byref(g), stream_handle()))
        return y_routed, y_shared

    def combine(self, y_routed: torch.Tensor, y_shared: torch.Tensor, r: dict,
                out_dtype: torch.dtype, residual=None) -> torch.Tensor:
        """moe.py:156-161: deterministic expert-ascending weighted sum + shared.
        residual = (h (B, S, d), th_ff (B, d)) adds backbone.py:606 in the
        epilogue: out = h + th_ff * (that)."""
        T, d = y_shared.shape
        E = r["comb_rows"].shape[1]
        out = torch.empty((T, d), dtype=out_dtype, device=y_shared.device)
        if r.get("_fused"):   # the gates are formed here (nimg_route_for_combine routing)
            h, th = residual if residual is not None else (None, None)
            _lib.check(_lib.lib.nimg_combine_routed(
                C.byref(r["_route_desc"]), ptr(r["_route_ws"]), nimg_dtype(y_shared.dtype),
                nimg_dtype(out_dtype), ptr(y_routed) if y_routed is not None else None,
                ptr(y_shared), ptr(r["gates"]), ptr(h) if h is not None else None,
                ptr(th) if th is not None else None, ptr(out), stream_handle()))
            return out
        if residual is None:
            _lib.check(_lib.lib.nimg_combine(T, d, E, nimg_dtype(y_shared.dtype),
                                             nimg_dtype(out_dtype), ptr(y_routed), ptr(y_shared),
                                             ptr(r["gates"]), ptr(r["comb_rows"]),
                                             ptr(r["comb_cnt"]), ptr(out), stream_handle()))
            return out
        h, th = residual
        S = h.shape[1]
        _lib.check(_lib.lib.nimg_combine_residual(T, d, E, S, nimg_dtype(y_shared.dtype),
                                                  nimg_dtype(out_dtype), ptr(y_routed),
                                                  ptr(y_shared), ptr(r["gates"]),
                                                  ptr(r["comb_rows"]), ptr(r["comb_cnt"]), ptr(h),
                                                  ptr(th), ptr(out), stream_handle()))
        return out
