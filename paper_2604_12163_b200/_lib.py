"""ctypes binding of libnimg_moe.so (the C ABI declared in include/nimg_moe.h).

There is no fallback: if the library is missing or cannot be loaded, import
fails loudly. Build it with ``python -m paper_2604_12163_b200._build``.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import ConfigError, ShapeError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libnimg_moe.so")
# A/B experiments only (tools/): load another in-tree build of the same ABI
LIB_PATH = os.environ.get("NIMG_LIB_PATH", LIB_PATH)

NIMG_OK, NIMG_ERR_SHAPE, NIMG_ERR_CONFIG, NIMG_ERR_CUDA = 0, 1, 2, 3
NIMG_F32, NIMG_BF16, NIMG_F64 = 0, 1, 2
ABI_VERSION = 2
NIMG_PATH_TCGEN05, NIMG_PATH_SIMT = 0, 1

# Every entry point the header declares (checked by tests/test_abi.py).
EXPORTS = (
    "nimg_last_error", "nimg_abi_version", "nimg_device_sms", "nimg_capacity_for",
    "nimg_moe_workspace_bytes", "nimg_moe_forward", "nimg_route_workspace_bytes", "nimg_route",
    "nimg_gather_rows", "nimg_ffn_path", "nimg_ffn_workspace_bytes", "nimg_expert_ffn",
    "nimg_combine", "nimg_profile_events", "nimg_ipc_alloc", "nimg_ipc_open", "nimg_ipc_close",
    "nimg_free", "nimg_copy_async", "nimg_stream_write_u32", "nimg_stream_wait_geq_u32",
    "nimg_moe_block_workspace_bytes", "nimg_moe_block_forward",
    "nimg_ln_modulate", "nimg_gate_res_ln_modulate", "nimg_gated_residual", "nimg_qk_norm_rope",
    "nimg_moe_block_prologue_workspace_bytes", "nimg_moe_block_prologue", "nimg_combine_residual",
    "nimg_moe_train_state_bytes", "nimg_moe_forward_train", "nimg_moe_backward_workspace_bytes",
    "nimg_moe_backward", "nimg_route_bg_flags", "nimg_expert_ffn_gather",
    "nimg_route_fusable", "nimg_route_for_combine", "nimg_combine_routed",
)


class MoeDesc(C.Structure):
    _fields_ = [("B", C.c_int64), ("S", C.c_int64), ("d", C.c_int64), ("E", C.c_int64),
                ("cap", C.c_int64), ("h", C.c_int64), ("h_shared", C.c_int64),
                ("gate_scale", C.c_float), ("gate_eps", C.c_float),
                ("act_dtype", C.c_int32), ("router_dtype", C.c_int32),
                ("gate_scale_f64", C.c_double), ("gate_eps_f64", C.c_double)]


class RouteOut(C.Structure):
    _fields_ = [("logits", C.c_void_p), ("scores_bes", C.c_void_p), ("token_flat", C.c_void_p),
                ("gate_raw", C.c_void_p), ("gates", C.c_void_p), ("comb_rows", C.c_void_p),
                ("comb_cnt", C.c_void_p)]


class MoePtrs(C.Structure):
    _fields_ = [("x_norm", C.c_void_p), ("x_mod", C.c_void_p), ("t_emb", C.c_void_p),
                ("w_r", C.c_void_p), ("w1", C.c_void_p), ("w3", C.c_void_p), ("w2", C.c_void_p),
                ("sw1", C.c_void_p), ("sw3", C.c_void_p), ("sw2", C.c_void_p),
                ("out", C.c_void_p), ("route", RouteOut)]


class BlockPtrs(C.Structure):
    _fields_ = [("x", C.c_void_p), ("r_attn", C.c_void_p), ("sa_gate", C.c_void_p),
                ("ff_scale", C.c_void_p), ("ff_gate", C.c_void_p), ("t_vec", C.c_void_p),
                ("w_r", C.c_void_p), ("w1", C.c_void_p), ("w3", C.c_void_p), ("w2", C.c_void_p),
                ("sw1", C.c_void_p), ("sw3", C.c_void_p), ("sw2", C.c_void_p), ("h", C.c_void_p),
                ("x_norm", C.c_void_p), ("x_mod", C.c_void_p), ("out", C.c_void_p),
                ("route", RouteOut)]


class MoeGrads(C.Structure):
    _fields_ = [("g_out", C.c_void_p), ("g_x_norm", C.c_void_p), ("g_x_mod", C.c_void_p),
                ("g_t_emb", C.c_void_p), ("g_w_r", C.c_void_p), ("g_w1", C.c_void_p),
                ("g_w3", C.c_void_p), ("g_w2", C.c_void_p), ("g_sw1", C.c_void_p),
                ("g_sw3", C.c_void_p), ("g_sw2", C.c_void_p)]


class BgGatherDesc(C.Structure):
    _fields_ = [("src", C.c_void_p), ("idx", C.c_void_p), ("dst", C.c_void_p),
                ("flags", C.c_void_p), ("chunk_done", C.c_void_p), ("rows", C.c_int32),
                ("row_bytes", C.c_int32), ("row_off", C.c_int32), ("chunk_rows", C.c_int32)]


class FfnDesc(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("n_shared_rows", C.c_int64), ("d", C.c_int64),
                ("h", C.c_int64), ("h_shared", C.c_int64), ("n_experts", C.c_int64),
                ("act_dtype", C.c_int32), ("nseg", C.c_int32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the CUDA extension is required (no CPU fallback). "
            "Build it with `python -m paper_2604_12163_b200._build`.")
    lib = C.CDLL(LIB_PATH)
    P, I64, I32, SZ = C.c_void_p, C.c_int64, C.c_int32, C.c_size_t
    sig = {
        "nimg_last_error": ([], C.c_char_p),
        "nimg_abi_version": ([], C.c_int),
        "nimg_device_sms": ([C.POINTER(C.c_int)], C.c_int),
        "nimg_capacity_for": ([I64, I64, C.c_double, C.POINTER(I64)], C.c_int),
        "nimg_moe_workspace_bytes": ([C.POINTER(MoeDesc), C.POINTER(SZ)], C.c_int),
        "nimg_moe_forward": ([C.POINTER(MoeDesc), C.POINTER(MoePtrs), P, SZ, P], C.c_int),
        "nimg_route_workspace_bytes": ([C.POINTER(MoeDesc), C.POINTER(SZ)], C.c_int),
        "nimg_route": ([C.POINTER(MoeDesc), P, P, P, C.POINTER(RouteOut), P, SZ, P], C.c_int),
        "nimg_gather_rows": ([P, I64, I64, P, I64, P, P], C.c_int),
        "nimg_ffn_path": ([C.POINTER(FfnDesc), C.POINTER(I32), C.POINTER(I32)], C.c_int),
        "nimg_ffn_workspace_bytes": ([C.POINTER(FfnDesc), C.POINTER(SZ)], C.c_int),
        "nimg_expert_ffn": ([C.POINTER(FfnDesc), P, P, P, P, P, P, P, P, P, P, P, P, P, SZ, P],
                            C.c_int),
        "nimg_combine": ([I64, I64, I64, I32, I32, P, P, P, P, P, P, P], C.c_int),
        "nimg_profile_events": ([C.POINTER(C.c_void_p), I32], C.c_int),
        "nimg_ipc_alloc": ([SZ, C.POINTER(C.c_void_p), P], C.c_int),
        "nimg_ipc_open": ([P, C.POINTER(C.c_void_p)], C.c_int),
        "nimg_ipc_close": ([P], C.c_int),
        "nimg_free": ([P], C.c_int),
        "nimg_copy_async": ([P, P, SZ, P], C.c_int),
        "nimg_stream_write_u32": ([P, C.c_uint32, P], C.c_int),
        "nimg_stream_wait_geq_u32": ([P, C.c_uint32, P], C.c_int),
        "nimg_moe_block_workspace_bytes": ([C.POINTER(MoeDesc), C.POINTER(SZ)], C.c_int),
        "nimg_moe_block_forward": ([C.POINTER(MoeDesc), C.POINTER(BlockPtrs), I32, P, SZ, P],
                                   C.c_int),
        "nimg_ln_modulate": ([I64, I64, I64, I32, P, P, P, P, C.c_float, P], C.c_int),
        "nimg_moe_block_prologue_workspace_bytes": ([C.POINTER(MoeDesc), C.POINTER(SZ)], C.c_int),
        "nimg_moe_block_prologue": ([C.POINTER(MoeDesc), P, P, P, P, P, I32, P, P, P, P, P, SZ, P],
                                    C.c_int),
        "nimg_combine_residual": ([I64, I64, I64, I64, I32, I32, P, P, P, P, P, P, P, P, P],
                                  C.c_int),
        "nimg_gate_res_ln_modulate": ([I64, I64, I64, I32, P, P, P, P, P, P, C.c_float, P],
                                      C.c_int),
        "nimg_gated_residual": ([I64, I64, I64, I32, P, P, P, P, P], C.c_int),
        "nimg_qk_norm_rope": ([I64, I64, I64, I64, I32, P, I64, P, P, P, C.c_float, P], C.c_int),
        "nimg_moe_train_state_bytes": ([C.POINTER(MoeDesc), C.POINTER(SZ)], C.c_int),
        "nimg_moe_forward_train": ([C.POINTER(MoeDesc), C.POINTER(MoePtrs), P, SZ, P, SZ, P],
                                   C.c_int),
        "nimg_moe_backward_workspace_bytes": ([C.POINTER(MoeDesc), C.POINTER(SZ)], C.c_int),
        "nimg_moe_backward": ([C.POINTER(MoeDesc), C.POINTER(MoePtrs), P, SZ,
                               C.POINTER(MoeGrads), P, SZ, P], C.c_int),
        "nimg_route_bg_flags": ([C.POINTER(MoeDesc), P, C.POINTER(C.c_void_p)], C.c_int),
        "nimg_expert_ffn_gather": ([C.POINTER(FfnDesc), P, P, P, P, P, P, P, P, P, P, P, P, P, SZ,
                                    C.POINTER(BgGatherDesc), P], C.c_int),
        "nimg_route_fusable": ([C.POINTER(MoeDesc)], C.c_int),
        "nimg_route_for_combine": ([C.POINTER(MoeDesc), P, P, P, C.POINTER(RouteOut), P, SZ, P],
                                   C.c_int),
        "nimg_combine_routed": ([C.POINTER(MoeDesc), P, I32, I32, P, P, P, P, P, P, P], C.c_int),
    }
    for name in EXPORTS:
        fn = getattr(lib, name)
        fn.argtypes, fn.restype = sig[name]
    if lib.nimg_abi_version() != ABI_VERSION:
        raise ImportError(f"{LIB_PATH} has ABI {lib.nimg_abi_version()}, this binding needs "
                          f"{ABI_VERSION}: rebuild with `python -m paper_2604_12163_b200._build`")
    return lib


lib = _load()


def check(rc: int) -> None:
    """Raise the reference's exception type for a non-zero return code."""
    if rc == NIMG_OK:
        return
    msg = lib.nimg_last_error().decode(errors="replace")
    if rc == NIMG_ERR_SHAPE:
        raise ShapeError(msg)
    if rc == NIMG_ERR_CONFIG:
        raise ConfigError(msg)
    raise RuntimeError(f"nimg CUDA error: {msg}")
