"""Host-side logic of the training entry points (no GPU): the reference-named
Tape / backward mapping onto torch autograd (tensor.py:148-176, :590-628)."""

import pytest
import torch

from paper_2604_12163_b200 import tensor as nt


def test_backward_fills_and_accumulates_grad():
    # tensor.py:64-70 behaviour: calling backward twice accumulates
    x = torch.tensor([2.0, -1.0], requires_grad=True)
    with nt.Tape() as tape:
        loss = (x * x).sum()
    nt.backward(tape, loss)
    torch.testing.assert_close(x.grad, torch.tensor([4.0, -2.0]))
    with nt.Tape() as tape:
        loss = (x * x).sum()
    nt.backward(tape, loss)
    torch.testing.assert_close(x.grad, torch.tensor([8.0, -4.0]))


def test_backward_rejects_nonscalar():
    x = torch.ones(3, requires_grad=True)
    with nt.Tape() as tape:
        y = x * 2
    with pytest.raises(nt.NonScalarLoss):
        nt.backward(tape, y)


def test_tape_enables_grad_inside_no_grad():
    x = torch.ones(2, requires_grad=True)
    with nt.no_grad():
        with nt.Tape():
            y = (x * 3).sum()
    assert y.requires_grad


def test_exception_types_are_value_errors():
    assert issubclass(nt.NonScalarLoss, ValueError)
    assert issubclass(nt.ShapeError, ValueError)
