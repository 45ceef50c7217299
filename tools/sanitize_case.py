"""One small layer per path, for compute-sanitizer (racecheck / synccheck /
memcheck): bf16 tcgen05 path (INT8 router, select, gate_norm, GEMM1 with the
background gather, GEMM2, combine), fp32 CUDA-core path, f64 mode, and one
bf16 training step (backward kernels).

    compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle.workloads import make_layer_inputs  # noqa: E402
from paper_2604_12163_b200 import moe as M  # noqa: E402
from paper_2604_12163_b200 import router as R  # noqa: E402

KEYS = ("w1", "w3", "w2", "sw1", "sw3", "sw2")


def layer(seed, B, S, d, E, h, C, dt, train=False):
    inp = make_layer_inputs(seed, B, S, d, E, h, mode="bf16" if dt == torch.bfloat16 else "fp32")
    T = lambda k, t: torch.from_numpy(np.ascontiguousarray(inp[k])).cuda().to(t)
    act = {k: T(k, dt) for k in ("x_norm", "x_mod") + KEYS}
    vdt = torch.float64 if dt == torch.float64 else torch.float32
    te, wr = T("t_emb", vdt), T("w_r", vdt)
    cfg = R.RouterConfig(d_model=d, n_experts=E, capacity_factor=C)
    if train:
        for k in act:
            act[k].requires_grad_(True)
    bank = M.ExpertBank(*(act[k] for k in KEYS))
    out = M.moe_forward(act["x_mod"], act["x_norm"], act["x_mod"], te, cfg, bank, wr)
    if train:
        out.float().square().sum().backward()
    torch.cuda.synchronize()
    print(f"ok {dt} B={B} S={S} d={d} E={E} h={h} train={train}", flush=True)


if __name__ == "__main__":
    torch.cuda.set_device(0)
    layer(1, 2, 256, 1024, 64, 128, 4.0, torch.bfloat16)      # INT8 router, tcgen05 pair GEMMs
    layer(2, 2, 96, 256, 8, 128, 2.0, torch.bfloat16)          # DMMA router, ragged rows
    layer(3, 2, 64, 64, 4, 40, 2.0, torch.float32)             # CUDA-core fp32 path
    layer(4, 2, 64, 64, 4, 40, 2.0, torch.float64)             # f64 mode
    layer(5, 2, 128, 256, 8, 128, 2.0, torch.bfloat16, train=True)   # tcgen05 backward
