"""Exception names of the reference's tensor module (tensor.py:19-20)."""

from .errors import ShapeError

__all__ = ["ShapeError"]
