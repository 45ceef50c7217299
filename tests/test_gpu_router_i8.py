"""The exact INT8 tensor-core router (csrc/router_i8.cu) against the CPU oracle
and against the FP64 (DMMA) router: fp32 logits, affinities, the token
permutation and the gates must be bit-identical (router.py:120-143).

The int8 path takes bf16 x_norm with E == 64, d % 64 == 0 and d <= 8192
(base-256 digits: a 32-bit row window, a 40-bit column window); these tests
also drive its escape hatches: x elements outside the row window (exact f64
terms, or the row recomputed in f64), W_r elements below the column window
(exact correction terms), too many of those (every token recomputed),
non-finite inputs, zero rows, subnormals, partial / sample-straddling tiles,
and K = 4096 / 8192 with digit sums near the int32 and 2^53 limits.
"""

import os

import numpy as np
import pytest
import torch

from oracle import nimg_oracle as O
from oracle.workloads import bf16_round, make_router_inputs
from tests.gpu_helpers import np_of

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_12163_b200 import _lib as L
    return L


def _gpu_route(inp, C, router=None):
    from paper_2604_12163_b200 import router as R
    B, S, d = inp["x_norm"].shape
    E = inp["w_r"].shape[1]
    old = os.environ.get("NIMG_ROUTER")
    if router:
        os.environ["NIMG_ROUTER"] = router
    try:
        cfg = R.RouterConfig(d_model=d, n_experts=E, capacity_factor=C)
        dec, routing = R.route_full(torch.from_numpy(inp["x_norm"]).cuda().to(torch.bfloat16),
                                    torch.from_numpy(inp["t_emb"]).cuda(),
                                    torch.from_numpy(inp["w_r"]).cuda(), cfg)
        torch.cuda.synchronize()
    finally:
        if router:
            if old is None:
                del os.environ["NIMG_ROUTER"]
            else:
                os.environ["NIMG_ROUTER"] = old
    return dec, routing


def _check(inp, C):
    B, S, d = inp["x_norm"].shape
    E = inp["w_r"].shape[1]
    ref = O.route_full(inp["x_norm"], inp["t_emb"], inp["w_r"], n_experts=E, capacity_factor=C)
    dec, routing = _gpu_route(inp, C)
    np.testing.assert_array_equal(np_of(routing["logits"]), ref["logits"])
    np.testing.assert_array_equal(routing["token_flat"].cpu().numpy(), ref["token_flat"])
    np.testing.assert_array_equal(np_of(routing["gates"]), ref["gates"])
    aff = np.stack([dd.affinity for dd in dec])
    np.testing.assert_array_equal(aff, ref["scores"].astype(np.float64).transpose(0, 2, 1)[
        np.arange(B)[:, None, None], np.arange(E)[None, :, None], ref["top"]])
    # and bit-identical to the FP64 tensor-pipe router
    _, r64 = _gpu_route(inp, C, router="dmma")
    np.testing.assert_array_equal(np_of(routing["logits"]), np_of(r64["logits"]))
    np.testing.assert_array_equal(routing["token_flat"].cpu().numpy(), r64["token_flat"].cpu().numpy())
    return routing


@pytest.mark.parametrize("B,S,seed", [(2, 1024, 1), (3, 200, 2), (1, 4096, 3), (5, 96, 4)])
def test_i8_router_full_width(B, S, seed):
    """d = 2048, E = 64: cfg-width inputs, including a partial last tile and
    tiles that straddle samples (S = 200, 96)."""
    inp = make_router_inputs(seed, B, S, 2048, 64, layer=17, mode="bf16")
    _check(inp, 4.0)


def test_i8_router_window_escapes():
    """x elements far below their row max (exact f64 terms / the row
    recomputed in f64), W_r elements below 2^-15 of their column max (exact corrections), zero
    rows, subnormal bf16 values, a row with a huge dynamic range."""
    rng = np.random.default_rng(11)
    inp = make_router_inputs(7, 2, 512, 1024, 64, mode="bf16")
    x = inp["x_norm"]
    x[0, 3, 17] = 1e-12            # below the row window -> f64 row
    x[0, 4, :] = 0.0               # zero row
    x[1, 5, :8] = np.float32(1e-39)   # subnormal in bf16
    x[1, 6, 100] = 3.0e4           # dynamic range: the rest truncates
    x[1, 7, ::2] *= 1e-6
    inp["x_norm"] = bf16_round(x)
    w = inp["w_r"]
    for e in range(64):            # a few tiny W elements in most columns
        ks = rng.choice(1024, size=e % 6, replace=False)
        w[ks, e] = (rng.standard_normal(len(ks)) * 1e-9).astype(np.float32)
    w[5, 9] = np.float32(1e-42)    # subnormal weight
    _check(inp, 2.0)


def test_i8_router_many_corrections():
    """A heavy-tailed column: 200 elements far below its max stay on the int8
    path as exact corrections (list of up to 256 per expert), bit-exact."""
    inp = make_router_inputs(8, 2, 256, 1024, 64, mode="bf16")
    inp["w_r"][:200, 13] = np.float32(1e-10)
    _check(inp, 4.0)


def test_i8_router_all_tokens_fallback():
    """More tiny W_r elements in one column than the correction list holds:
    every token takes the f64 path, still bit-exact."""
    inp = make_router_inputs(8, 2, 256, 1024, 64, mode="bf16")
    inp["w_r"][:300, 13] = np.float32(1e-10)
    _check(inp, 4.0)


def test_i8_router_nonfinite():
    """A NaN row of x_norm and an inf-free W_r: the NaN token is recomputed
    in f64 and sorts last (router.py:100); an inf in W_r sends every token to
    the f64 path."""
    inp = make_router_inputs(9, 1, 256, 1024, 64, mode="bf16")
    inp["x_norm"][0, [5, 9]] = np.nan
    _check(inp, 64.0)
    inp = make_router_inputs(10, 1, 128, 1024, 64, mode="bf16")
    inp["w_r"][7, 3] = np.inf
    ref = O.route_full(inp["x_norm"], inp["t_emb"], inp["w_r"], n_experts=64, capacity_factor=4.0)
    _, routing = _gpu_route(inp, 4.0)
    np.testing.assert_array_equal(np_of(routing["logits"]), ref["logits"])
    np.testing.assert_array_equal(routing["token_flat"].cpu().numpy(), ref["token_flat"])


def test_i8_router_repeatable():
    """Two calls give identical bits (the fix-up list order is atomic, the
    values are not)."""
    inp = make_router_inputs(12, 4, 1024, 2048, 64, mode="bf16")
    _, a = _gpu_route(inp, 2.0)
    _, b = _gpu_route(inp, 2.0)
    np.testing.assert_array_equal(np_of(a["logits"]), np_of(b["logits"]))
    np.testing.assert_array_equal(a["token_flat"].cpu().numpy(), b["token_flat"].cpu().numpy())


@pytest.mark.parametrize("d", [4096, 8192])
def test_i8_router_wide_k(d):
    """K = 4096 and 8192 (the int8 path's limit): random inputs, then
    same-sign inputs at the top of both windows, where every int32 digit-group
    sum is near its bound and the int64 halves exceed 2^53 (their conversions
    round; the rounding proof accounts for it)."""
    inp = make_router_inputs(13, 1, 256, d, 64, mode="bf16")
    _check(inp, 4.0)
    rng = np.random.default_rng(14)
    x = np.full((1, 128, d), 1.9921875, np.float32)          # 0x3FFF: the largest bf16 significand
    x[:, :, ::7] = -1.9921875
    inp["x_norm"] = bf16_round(x * rng.uniform(0.5, 1.0, (1, 128, 1)).astype(np.float32))
    w = np.float32(0.0059) * (1.0 + rng.uniform(0.0, 2.0 ** -20, (2 * d, 64))).astype(np.float32)
    inp["w_r"] = w.astype(np.float32)
    _check(inp, 8.0)
