"""Shared helpers for the -m gpu parity tests."""

from __future__ import annotations

import numpy as np
import torch

ACT_KEYS = ("x_norm", "x_mod", "w1", "w3", "w2", "sw1", "sw3", "sw2")

# north star tolerances (BASELINE.json): Frobenius relative error of the layer
# output vs the reference's CPU path.
TOL_FP32 = 1e-4
TOL_BF16 = 2e-2


def to_gpu(inp: dict, mode: str) -> dict:
    """fp32 arrays -> CUDA tensors; activations/weights in bf16 for bf16 mode
    (the arrays are already bf16-representable, so the cast is exact)."""
    act = torch.bfloat16 if mode == "bf16" else torch.float32
    out = {}
    for k, v in inp.items():
        t = torch.from_numpy(np.ascontiguousarray(v)).cuda()
        out[k] = t.to(act) if k in ACT_KEYS else t
    return out


def bank_of(g: dict):
    from paper_2604_12163_b200.moe import ExpertBank
    return ExpertBank(g["w1"], g["w3"], g["w2"], g["sw1"], g["sw3"], g["sw2"])


def rel_fro(y, y_ref) -> float:
    y = np.asarray(y, dtype=np.float64)
    y_ref = np.asarray(y_ref, dtype=np.float64)
    return float(np.linalg.norm(y - y_ref) / max(np.linalg.norm(y_ref), 1e-300))


def np_of(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().numpy()
