"""CPU-side checks of the C ABI: the library loads without a GPU, exports every
entry point include/nimg_moe.h declares, and its host-only functions
(capacity, workspace sizing, validation -> error codes) behave like the
reference's host logic."""

import ctypes as C
import os
import re

import pytest

from oracle import nimg_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    from paper_2604_12163_b200 import _lib as L
    return L


def test_header_declares_exactly_the_exported_symbols():
    L = _lib()
    hdr = open(os.path.join(ROOT, "include", "nimg_moe.h")).read()
    declared = set(re.findall(r"\b(nimg_[a-z0-9_]+)\s*\(", hdr))
    assert declared == set(L.EXPORTS)
    for name in declared:
        assert hasattr(L.lib, name), name


def test_capacity_for_matches_reference_host_logic():
    L = _lib()
    out = C.c_int64()
    for S, E, Cf in [(256, 64, 8.0), (1024, 64, 4.0), (5, 64, 8.0), (4, 2, 100.0), (4032, 64, 2.0),
                     (3840, 64, 2.0), (4096, 64, 8.0), (37, 5, 1.7)]:
        assert L.lib.nimg_capacity_for(S, E, Cf, C.byref(out)) == 0
        assert out.value == O.capacity_for(S, E, Cf)
    assert L.lib.nimg_capacity_for(0, 2, 1.0, C.byref(out)) == L.NIMG_ERR_CONFIG
    assert L.lib.nimg_capacity_for(4, 2, 0.0, C.byref(out)) == L.NIMG_ERR_CONFIG
    assert b"invalid capacity" in L.lib.nimg_last_error()


def test_workspace_and_validation_codes():
    L = _lib()
    d = L.MoeDesc(B=16, S=1024, d=2048, E=64, cap=64, h=1344, h_shared=1344, gate_scale=1.0,
                  gate_eps=1e-6, act_dtype=L.NIMG_BF16, router_dtype=L.NIMG_BF16,
                  gate_scale_f64=1.0, gate_eps_f64=1e-6)
    n = C.c_size_t()
    assert L.lib.nimg_moe_workspace_bytes(C.byref(d), C.byref(n)) == 0
    R_rows, T = 64 * 16 * 64, 16 * 1024
    # gathered rows + pre (routed+shared) + y (routed+shared), bf16, plus routing scratch
    need = 2 * (R_rows * 2048 + (R_rows + T) * 1344 + (R_rows + T) * 2048)
    assert need <= n.value < need + (16 << 20)
    bad = L.MoeDesc(**{f: getattr(d, f) for f, _ in L.MoeDesc._fields_})
    bad.gate_eps = 0.0
    assert L.lib.nimg_moe_workspace_bytes(C.byref(bad), C.byref(n)) == L.NIMG_ERR_CONFIG
    bad.gate_eps = 1e-6
    bad.cap = 0
    assert L.lib.nimg_moe_workspace_bytes(C.byref(bad), C.byref(n)) == L.NIMG_ERR_CONFIG
    bad.cap = 2048
    assert L.lib.nimg_moe_workspace_bytes(C.byref(bad), C.byref(n)) == L.NIMG_ERR_CONFIG


def test_ffn_path_selection():
    L = _lib()
    f = L.FfnDesc(n_rows=1024, n_shared_rows=0, d=2048, h=1344, h_shared=1344, n_experts=64,
                  act_dtype=L.NIMG_BF16, nseg=64)
    p, y = C.c_int32(), C.c_int32()
    assert L.lib.nimg_ffn_path(C.byref(f), C.byref(p), C.byref(y)) == 0
    assert (p.value, y.value) == (L.NIMG_PATH_TCGEN05, L.NIMG_BF16)
    # fp32 layers whose widths tile the pair kernels run on the tensor cores
    # (bf16x3 split, fp32 output); others on the CUDA cores
    f.act_dtype = L.NIMG_F32
    L.lib.nimg_ffn_path(C.byref(f), C.byref(p), C.byref(y))
    assert (p.value, y.value) == (L.NIMG_PATH_TCGEN05, L.NIMG_F32)
    f.h = 168
    L.lib.nimg_ffn_path(C.byref(f), C.byref(p), C.byref(y))
    assert (p.value, y.value) == (L.NIMG_PATH_SIMT, L.NIMG_F32)
    f.act_dtype, f.h = L.NIMG_BF16, 20
    L.lib.nimg_ffn_path(C.byref(f), C.byref(p), C.byref(y))
    assert p.value == L.NIMG_PATH_SIMT


def test_ffn_segment_validation():
    """Host-side checks run before any device work: expert ids must lie in
    [-1, E) (-1 = skip segment), offsets start at 0, end at n_rows."""
    L = _lib()
    f = L.FfnDesc(n_rows=64, n_shared_rows=0, d=32, h=32, h_shared=32, n_experts=4,
                  act_dtype=L.NIMG_BF16, nseg=2)
    off = (C.c_int64 * 3)(0, 32, 64)
    call = lambda ex: L.lib.nimg_expert_ffn(C.byref(f), off, (C.c_int32 * 2)(*ex), None, None, None,
                                            None, None, None, None, None, None, None, None, 0, None)
    assert call((0, 4)) == L.NIMG_ERR_SHAPE
    assert b"expert 4 out of range" in L.lib.nimg_last_error()
    assert call((-2, 0)) == L.NIMG_ERR_SHAPE
    off[2] = 63
    assert call((0, -1)) == L.NIMG_ERR_SHAPE
    assert b"offsets end" in L.lib.nimg_last_error()


def test_python_api_mirrors_reference_host_functions():
    from paper_2604_12163_b200 import router as R
    assert R.capacity_for(1024, 64, 4.0) == 64
    assert R.capacity_schedule(5, R.StageId.S1024) == 2.0
    assert R.capacity_schedule(0, R.StageId.S256) is R.DENSE
    with pytest.raises(IndexError):
        R.capacity_schedule(32, R.StageId.S256)
    with pytest.raises(R.ConfigError):
        R.RouterConfig(d_model=4, n_experts=2, capacity_factor=0.0)
    import numpy as np
    from paper_2604_12163_b200 import moe as M
    with pytest.raises(M.ShapeError):
        M.GroupedBatch(np.zeros((3, 2)), np.array([0, 2, 1]))


def test_router_dtype_and_f64_mode_validation():
    """ABI v2: router_dtype is x_norm's own dtype; NIMG_F64 is the reference's
    f64 storage mode (forward only, all-f64)."""
    L = _lib()
    assert L.lib.nimg_abi_version() == L.ABI_VERSION == 2
    base = dict(B=2, S=256, d=256, E=8, cap=64, h=168, h_shared=168, gate_scale=1.0,
                gate_eps=1e-6, gate_scale_f64=1.0, gate_eps_f64=1e-6)
    n = C.c_size_t()
    ok = [(L.NIMG_BF16, L.NIMG_BF16), (L.NIMG_BF16, L.NIMG_F32), (L.NIMG_F32, L.NIMG_BF16),
          (L.NIMG_F32, L.NIMG_F32), (L.NIMG_F64, L.NIMG_F64)]
    bad = [(L.NIMG_F64, L.NIMG_F32), (L.NIMG_BF16, L.NIMG_F64), (L.NIMG_F32, 7), (5, L.NIMG_F32)]
    for act, rt in ok:
        d = L.MoeDesc(act_dtype=act, router_dtype=rt, **base)
        assert L.lib.nimg_moe_workspace_bytes(C.byref(d), C.byref(n)) == 0, (act, rt)
    for act, rt in bad:
        d = L.MoeDesc(act_dtype=act, router_dtype=rt, **base)
        assert L.lib.nimg_moe_workspace_bytes(C.byref(d), C.byref(n)) == L.NIMG_ERR_CONFIG
    # training: same dtype for x_norm and x_mod, and no f64 path
    for act, rt, want in ((L.NIMG_BF16, L.NIMG_BF16, 0), (L.NIMG_BF16, L.NIMG_F32, L.NIMG_ERR_CONFIG),
                          (L.NIMG_F64, L.NIMG_F64, L.NIMG_ERR_CONFIG)):
        d = L.MoeDesc(act_dtype=act, router_dtype=rt, **base)
        assert L.lib.nimg_moe_train_state_bytes(C.byref(d), C.byref(n)) == want
    d = L.MoeDesc(act_dtype=L.NIMG_F64, router_dtype=L.NIMG_F64, **dict(base, gate_eps_f64=0.0))
    assert L.lib.nimg_moe_workspace_bytes(C.byref(d), C.byref(n)) == L.NIMG_ERR_CONFIG
    # the f64 mode runs the CUDA-core GEMMs and returns f64 rows
    f = L.FfnDesc(n_rows=512, n_shared_rows=0, d=256, h=168, h_shared=168, n_experts=8,
                  act_dtype=L.NIMG_F64, nseg=8)
    p, y = C.c_int32(), C.c_int32()
    assert L.lib.nimg_ffn_path(C.byref(f), C.byref(p), C.byref(y)) == 0
    assert (p.value, y.value) == (L.NIMG_PATH_SIMT, L.NIMG_F64)
