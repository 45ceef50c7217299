"""Names of the reference's tensor module (tensor.py) that the operator API
shares: the exceptions, and the tape entry points mapped onto torch autograd
(the B200 path records the MoE layer as one autograd node; tensor.py:135-176,
:590-628).

    with Tape() as tape:
        out = moe.moe_forward(x, x_norm, x_mod, t_emb, cfg, bank, w_r)
        loss = (out * out).sum()
    backward(tape, loss)        # fills .grad of every tensor that requires grad
"""

from __future__ import annotations

import torch

from .errors import DomainError, ShapeError


class NonScalarLoss(ValueError):
    """backward() requires a scalar loss tensor (tensor.py:27-28)."""


class Tape:
    """tensor.py:148-160 -- context in which taped ops record; here: grad mode on."""

    def __enter__(self) -> "Tape":
        self._guard = torch.enable_grad()
        self._guard.__enter__()
        return self

    def __exit__(self, *exc):
        self._guard.__exit__(*exc)
        return False


no_grad = torch.no_grad


def backward(tape: Tape, loss: torch.Tensor) -> None:
    """tensor.py:590-628 -- accumulate dLoss/dLeaf into .grad (calling twice
    accumulates, as in the reference)."""
    if loss.numel() != 1:
        raise NonScalarLoss(f"loss must be scalar, got shape {tuple(loss.shape)}")
    loss.reshape(()).backward()


__all__ = ["ShapeError", "DomainError", "NonScalarLoss", "Tape", "no_grad", "backward"]
