"""Out-of-bounds write check: every buffer handed to the C ABI (inputs,
routing outputs, workspace, training state, backward workspace, gradients) is
surrounded by guard bands; a forward_train + backward at several shapes must
leave every guard byte untouched. Catches workspace carves that disagree with
the *_bytes() sizing functions (the CUDA-core training path once wrote its
fp32 shared-expert outputs past the end of the forward workspace)."""

import ctypes as C

import numpy as np
import pytest
import torch

from oracle.workloads import make_layer_inputs
from tests.gpu_helpers import to_gpu

pytestmark = pytest.mark.gpu

GUARD = 1 << 16
NAMES = ("x_norm", "x_mod", "t_emb", "w_r", "w1", "w3", "w2", "sw1", "sw3", "sw2")


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_12163_b200 import _lib as L
    return L


class Guarded:
    def __init__(self):
        self.bufs = {}

    def alloc(self, name, nbytes, dtype=torch.uint8, shape=None):
        raw = torch.full((nbytes + 2 * GUARD,), 0xA5, dtype=torch.uint8, device="cuda")
        self.bufs[name] = (raw, nbytes)
        v = raw[GUARD:GUARD + nbytes]
        if dtype != torch.uint8:
            v = v.view(dtype)
            if shape is not None:
                v = v.view(shape)
        return v

    def violations(self):
        torch.cuda.synchronize()
        return [k for k, (raw, n) in self.bufs.items()
                if not bool((raw[:GUARD] == 0xA5).all()) or not bool((raw[GUARD + n:] == 0xA5).all())]


@pytest.mark.parametrize("B,S,d,E,h,Cf,mode", [
    (2, 96, 192, 8, 80, 2.0, "bf16"),     # CUDA-core training path, ragged h
    (2, 96, 192, 8, 80, 2.0, "fp32"),
    (2, 128, 256, 8, 128, 2.0, "bf16"),   # tcgen05 training path
    (2, 256, 1024, 64, 128, 4.0, "bf16"), # INT8 router path (E = 64, d % 128 == 0)
])
def test_no_out_of_bounds_writes(B, S, d, E, h, Cf, mode):
    from paper_2604_12163_b200 import _lib
    from paper_2604_12163_b200._tensors import stream_handle
    from paper_2604_12163_b200.moe import _sizeof
    from paper_2604_12163_b200.router import RouterConfig, capacity_for, make_desc, route_struct
    gd = Guarded()
    g0 = to_gpu(make_layer_inputs(7, B, S, d, E, h, mode=mode), mode)
    g = {}
    for k in NAMES:
        t = g0[k]
        g[k] = gd.alloc("in_" + k, t.numel() * t.element_size(), t.dtype, t.shape)
        g[k].copy_(t)
    act = g["x_mod"].dtype
    es = 2 if act == torch.bfloat16 else 4
    cfg = RouterConfig(d_model=d, n_experts=E, capacity_factor=Cf)
    cap = capacity_for(S, E, Cf)
    desc = make_desc(B, S, d, E, cap, h, h, cfg, act)
    n, T = E * B * cap, B * S
    f32, i32 = torch.float32, torch.int32
    r = {"logits": gd.alloc("logits", T * E * 4, f32), "scores_bes": gd.alloc("scores", T * E * 4, f32),
         "token_flat": gd.alloc("token_flat", n * 4, i32), "gate_raw": gd.alloc("gate_raw", n * 4, f32),
         "gates": gd.alloc("gates", n * 4, f32), "comb_rows": gd.alloc("comb_rows", T * E * 4, i32),
         "comb_cnt": gd.alloc("comb_cnt", T * 4, i32)}
    wsn = _sizeof(_lib.lib.nimg_moe_workspace_bytes, desc)
    stn = _sizeof(_lib.lib.nimg_moe_train_state_bytes, desc)
    bwn = _sizeof(_lib.lib.nimg_moe_backward_workspace_bytes, desc)
    ws, state, bws = gd.alloc("ws", wsn), gd.alloc("state", stn), gd.alloc("bws", bwn)
    out = gd.alloc("out", T * d * es, act)
    P = lambda t: t.data_ptr()
    ptrs = _lib.MoePtrs(*(P(g[k]) for k in NAMES), P(out), route_struct(r))
    _lib.check(_lib.lib.nimg_moe_forward_train(C.byref(desc), C.byref(ptrs), P(state), stn, P(ws),
                                               wsn, stream_handle()))
    assert gd.violations() == []
    go = gd.alloc("g_out", T * d * es, act)
    go.copy_(torch.randn(T * d, device="cuda").to(act))
    gr = {k: gd.alloc("g_" + k, g[k].numel() * (es if k in ("x_norm", "x_mod") else 4),
                      act if k in ("x_norm", "x_mod") else f32) for k in NAMES}
    grads = _lib.MoeGrads(P(go), *(P(gr[k]) for k in NAMES))
    ptrs2 = _lib.MoePtrs(*(P(g[k]) for k in NAMES), None, route_struct(r))
    _lib.check(_lib.lib.nimg_moe_backward(C.byref(desc), C.byref(ptrs2), P(state), stn,
                                          C.byref(grads), P(bws), bwn, stream_handle()))
    assert gd.violations() == []
    for k in NAMES:
        assert bool(torch.isfinite(gr[k].float()).all()), k
    # the inference forward into the same guarded workspace
    _lib.check(_lib.lib.nimg_moe_forward(C.byref(desc), C.byref(ptrs), P(ws), wsn, stream_handle()))
    assert gd.violations() == []
