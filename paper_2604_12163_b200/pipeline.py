"""Host-to-host serving pipeline around the public layer call.

Each step copies its inputs from pinned host memory (H2D stream), runs the
layer through the public API (moe.moe_forward, compute stream) and copies the
output back to pinned host memory (D2H stream). Buffers are double-buffered,
so step i+1's upload and step i-1's download overlap step i's compute; PCIe is
full duplex, so the step time tends to max(H2D, compute, D2H).
"""

from __future__ import annotations

from typing import Callable, Sequence

import torch


class HostPipeline:
    def __init__(self, fn: Callable[..., torch.Tensor], host_inputs: Sequence[torch.Tensor],
                 out_shape, out_dtype, device=None, depth: int = 2):
        self.fn = fn
        self.dev = device or torch.device("cuda", torch.cuda.current_device())
        self.depth = depth
        self.h2d = torch.cuda.Stream(self.dev)
        self.d2h = torch.cuda.Stream(self.dev)
        self.comp = torch.cuda.current_stream(self.dev)
        self.host_inputs = list(host_inputs)
        self.dev_in = [[torch.empty_like(h, device=self.dev) for h in host_inputs]
                       for _ in range(depth)]
        self.host_out = [torch.empty(out_shape, dtype=out_dtype).pin_memory() for _ in range(depth)]
        self.ev_in = [torch.cuda.Event() for _ in range(depth)]
        self.ev_out = [torch.cuda.Event() for _ in range(depth)]
        self.ev_consumed = [torch.cuda.Event() for _ in range(depth)]
        self.ev_drained = [torch.cuda.Event() for _ in range(depth)]
        self._outs = [None] * depth
        self.bytes_in = sum(h.numel() * h.element_size() for h in host_inputs)
        self.bytes_out = self.host_out[0].numel() * self.host_out[0].element_size()
        self.i = 0

    def step(self) -> None:
        k = self.i % self.depth
        # upload into slot k once its previous step's compute has consumed it
        with torch.cuda.stream(self.h2d):
            if self.i >= self.depth:
                self.h2d.wait_event(self.ev_consumed[k])
            for dst, src in zip(self.dev_in[k], self.host_inputs):
                dst.copy_(src, non_blocking=True)
            self.ev_in[k].record(self.h2d)
        self.comp.wait_event(self.ev_in[k])
        if self.i >= self.depth:
            self.comp.wait_event(self.ev_drained[k])   # output slot k downloaded
        y = self.fn(*self.dev_in[k])
        self.ev_consumed[k].record(self.comp)
        self.ev_out[k].record(self.comp)
        self._outs[k] = y                             # keep alive until downloaded
        with torch.cuda.stream(self.d2h):
            self.d2h.wait_event(self.ev_out[k])
            self.host_out[k].copy_(y, non_blocking=True)
            self.ev_drained[k].record(self.d2h)
        # no y.record_stream(d2h): y stays referenced in _outs[k] until step
        # i + depth, whose compute is already ordered after ev_drained[k], so
        # its block returns to the compute stream's pool only when the download
        # is done -- without deferred frees growing the allocator (a cudaMalloc
        # mid-run, mapped into every IPC peer under EP, stalls the host)
        self.i += 1

    def drain(self) -> None:
        self.comp.wait_stream(self.d2h)
        self.comp.wait_stream(self.h2d)
