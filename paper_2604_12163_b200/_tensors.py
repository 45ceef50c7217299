"""Input adaptation for the operator API: torch / numpy / reference-Tensor
inputs become contiguous CUDA tensors of a kernel dtype. Plumbing only --
all arithmetic happens in the CUDA library."""

from __future__ import annotations

import numpy as np
import torch

from .errors import ConfigError

# float64 is the reference's f64 storage mode (tensor.py:39-47), computed in
# f64 end to end (csrc/f64_kernels.cu) -- never silently downcast.
KERNEL_DTYPES = (torch.float32, torch.bfloat16, torch.float64)


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2604_12163_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def to_device(x, dtype: torch.dtype | None = None) -> torch.Tensor:
    """torch.Tensor, numpy array or reference Tensor (has a numpy `.data`)
    -> contiguous CUDA tensor of `dtype` (default: its own dtype)."""
    if not isinstance(x, torch.Tensor):
        arr = x.data if (hasattr(x, "data") and isinstance(getattr(x, "data"), np.ndarray)) else x
        x = torch.from_numpy(np.ascontiguousarray(np.asarray(arr)))
    dev = device()
    if dtype is None:
        dtype = x.dtype
    if dtype not in KERNEL_DTYPES and dtype not in (torch.int64, torch.int32):
        raise ConfigError(f"unsupported dtype {x.dtype}")
    if x.device != dev or x.dtype != dtype:
        x = x.to(device=dev, dtype=dtype, non_blocking=True)
    return x.contiguous()


def nimg_dtype(dt: torch.dtype) -> int:
    from ._lib import NIMG_BF16, NIMG_F32, NIMG_F64
    if dt == torch.bfloat16:
        return NIMG_BF16
    if dt == torch.float32:
        return NIMG_F32
    if dt == torch.float64:
        return NIMG_F64
    raise ConfigError(f"unsupported activation dtype {dt}")


def dtype_of(x) -> torch.dtype | None:
    """torch dtype of a torch tensor, numpy array or reference Tensor (None if
    it has no dtype)."""
    if isinstance(x, torch.Tensor):
        return x.dtype
    arr = x.data if (hasattr(x, "data") and isinstance(getattr(x, "data"), np.ndarray)) else x
    if isinstance(arr, np.ndarray):
        return torch.from_numpy(np.empty(0, dtype=arr.dtype)).dtype
    return None


def any_f64(*xs) -> bool:
    """The reference promotes an op to f64 when any operand is f64
    (np.result_type, tensor.py:203-204)."""
    return any(dtype_of(x) == torch.float64 for x in xs if x is not None)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def workspace(nbytes: int) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device())
