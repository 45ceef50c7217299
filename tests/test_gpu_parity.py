"""GPU parity: the CUDA path (through the operator API -> C ABI) against the
reference's golden vectors and the CPU oracle.

Bars (BASELINE.json north_star): expert selection indices, token permutation
and fp32 router scores/gates bit-exact; layer output Frobenius rel-err
<= 1e-4 in fp32 mode and <= 2e-2 in bf16 mode.
"""

import numpy as np
import pytest
import torch

from oracle import nimg_oracle as O
from oracle.workloads import make_layer_inputs
from tests import golden_cases as G
from tests.gpu_helpers import TOL_BF16, TOL_FP32, bank_of, np_of, rel_fro, to_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_12163_b200 import _lib as L  # fails loudly if the .so is missing
    return L


def _route(inp, p):
    from paper_2604_12163_b200 import router as R
    g = to_gpu(inp, p["mode"])
    cfg = R.RouterConfig(d_model=p["d"], n_experts=p["E"], capacity_factor=p["C"],
                         gate_scale=p.get("gate_scale", 1.0))
    return R.route_full(g["x_norm"], g["t_emb"], g["w_r"], cfg)


def _check_routing(decisions, routing, exp, B):
    np.testing.assert_array_equal(np_of(routing["logits"]), exp["logits"])
    np.testing.assert_array_equal(routing["token_flat"].cpu().numpy(), exp["token_flat"])
    np.testing.assert_array_equal(np_of(routing["gates"]), exp["gates"])
    np.testing.assert_array_equal(np.stack([d.top_indices for d in decisions]), exp["top"])
    np.testing.assert_array_equal(np.stack([d.affinity for d in decisions]), exp["affinity"])
    assert routing["capacity"] == int(exp["capacity"])


@pytest.mark.parametrize("name", G.names("route"))
def test_route_bitexact_vs_reference_golden(name):
    kind, p, inp, exp = G.case(name)
    decisions, routing = _route(inp, p)
    _check_routing(decisions, routing, exp, p["B"])


@pytest.mark.parametrize("name", G.names("moe"))
def test_moe_forward_vs_reference_golden(name):
    from paper_2604_12163_b200 import moe as M
    from paper_2604_12163_b200 import router as R
    kind, p, inp, exp = G.case(name)
    g = to_gpu(inp, p["mode"])
    cfg = R.RouterConfig(d_model=p["d"], n_experts=p["E"], capacity_factor=p["C"],
                         gate_scale=p.get("gate_scale", 1.0))
    out, decisions, routing = M.moe_forward(g["x_mod"], g["x_norm"], g["x_mod"], g["t_emb"], cfg,
                                            bank_of(g), g["w_r"], return_routing=True)
    _check_routing(decisions, routing, exp, p["B"])
    err = rel_fro(np_of(out), exp["out"])
    tol = TOL_FP32 if p["mode"] == "fp32" else TOL_BF16
    assert err <= tol, f"{name}: rel-err {err:.3e} > {tol}"


# ---------------------------------------------------------------- KATs
def test_uniform_logits_tie_break_by_index():            # test_router.py:48-58
    from paper_2604_12163_b200 import router as R
    rng = np.random.default_rng(0)
    for S, E, C in ((6, 2, 1.0), (1024, 64, 4.0), (4096, 64, 2.0)):
        d = 8
        cfg = R.RouterConfig(d_model=d, n_experts=E, capacity_factor=C)
        xn = torch.tensor(rng.normal(size=(2, S, d)), dtype=torch.float32).cuda()
        te = torch.tensor(rng.normal(size=(2, d)), dtype=torch.float32).cuda()
        wr = torch.zeros((2 * d, E), dtype=torch.float32).cuda()
        decs = R.route(xn, te, wr, cfg)
        cap = R.capacity_for(S, E, C)
        for dec in decs:
            for e in range(E):
                np.testing.assert_array_equal(dec.top_indices[e], np.arange(cap))
            np.testing.assert_allclose(dec.affinity, 1.0 / E, atol=1e-7)


def test_full_capacity_gates_sum_to_one():               # test_router.py:61-75
    from paper_2604_12163_b200 import router as R
    rng = np.random.default_rng(1)
    cfg = R.RouterConfig(d_model=4, n_experts=2, capacity_factor=2.0)
    wr = torch.tensor(rng.normal(size=(8, 2)), dtype=torch.float32).cuda()
    xn = torch.tensor(rng.normal(size=(1, 4, 4)), dtype=torch.float32).cuda()
    te = torch.tensor(rng.normal(size=(1, 4)), dtype=torch.float32).cuda()
    (dec,) = R.route(xn, te, wr, cfg)
    assert dec.capacity == 4
    for e in range(2):
        np.testing.assert_array_equal(np.sort(dec.top_indices[e]), np.arange(4))
    per_tok = np.zeros(4)
    np.add.at(per_tok, dec.top_indices.reshape(-1), dec.gates.reshape(-1))
    np.testing.assert_allclose(per_tok, 1.0, atol=1e-5)


def test_router_weight_shape_and_config_errors():       # test_router.py:152-155, router.py:45-56
    from paper_2604_12163_b200 import router as R
    cfg = R.RouterConfig(d_model=4, n_experts=2, capacity_factor=1.0)
    with pytest.raises(R.ConfigError):
        cfg.validate_weight(torch.zeros((4, 2)))
    with pytest.raises(R.ConfigError):
        R.RouterConfig(d_model=4, n_experts=0, capacity_factor=1.0)
    with pytest.raises(R.ConfigError):
        R.route(torch.zeros((1, 4, 4)), torch.zeros((1, 4)), torch.zeros((4, 2)), cfg)


def test_swiglu_scalar_reduction_and_zero_input():       # test_moe.py:19-33
    from paper_2604_12163_b200 import moe as M
    for x in (-1.3, 0.0, 0.7, 2.5):
        one = torch.ones((1, 1))
        out = M.swiglu(torch.tensor([[x]], dtype=torch.float32), one, one, one)
        np.testing.assert_allclose(out.item(), x / (1 + np.exp(-x)) * x, rtol=1e-6)
    rng = np.random.default_rng(0)
    w1, w3, w2 = (torch.tensor(rng.normal(size=s), dtype=torch.float32) for s in ((3, 2), (3, 2), (2, 3)))
    out = M.swiglu(torch.zeros((4, 2)), w1, w3, w2)
    assert torch.all(out == 0)
    with pytest.raises(M.ShapeError):
        M.swiglu(torch.zeros((2, 3)), torch.zeros((4, 3)), torch.zeros((4, 2)), torch.zeros((3, 4)))


def test_grouped_forward_matches_loop_oracle_and_empty_segments():   # test_moe.py:69-112
    from paper_2604_12163_b200 import moe as M
    rng = np.random.default_rng(5)
    for mode, (E, h, d), counts in (("fp32", (3, 4, 5), [2, 0, 3]),
                                    ("fp32", (4, 48, 64), [130, 0, 0, 257]),
                                    ("bf16", (4, 224, 256), [300, 0, 129, 1])):
        w = {k: rng.normal(size=s).astype(np.float32) * 0.05 for k, s in
             (("w1", (E, h, d)), ("w3", (E, h, d)), ("w2", (E, d, h)))}
        toks = rng.normal(size=(sum(counts), d)).astype(np.float32)
        if mode == "bf16":
            from oracle.workloads import bf16_round
            w = {k: bf16_round(v) for k, v in w.items()}
            toks = bf16_round(toks)
        off = np.concatenate([[0], np.cumsum(counts)])
        act = torch.bfloat16 if mode == "bf16" else torch.float32
        bank = M.ExpertBank(*(torch.tensor(w[k]).cuda().to(act) for k in ("w1", "w3", "w2")),
                            None, None, None)
        y = M.grouped_forward(M.GroupedBatch(torch.tensor(toks).cuda().to(act), off), bank)
        ref = O.grouped_forward(toks, off, w["w1"], w["w3"], w["w2"])
        tol = TOL_FP32 if mode == "fp32" else TOL_BF16
        assert rel_fro(np_of(y), ref) <= tol
    with pytest.raises(M.ShapeError):
        M.GroupedBatch(torch.zeros((3, 2)), np.array([0, 2, 1]))
    with pytest.raises(M.ShapeError):
        M.GroupedBatch(torch.zeros((3, 2)), np.array([0, 1, 2]))


def test_zero_w2_gives_shared_only_and_single_expert():   # test_moe.py:147-176
    from paper_2604_12163_b200 import moe as M
    from paper_2604_12163_b200 import router as R
    rng = np.random.default_rng(6)
    d, E, h, S = 4, 2, 4, 6
    f = lambda *s: rng.normal(size=s).astype(np.float32)
    w1, w3, w2 = f(E, h, d), f(E, h, d), np.zeros((E, d, h), np.float32)
    s1, s3, s2 = f(h, d), f(h, d), f(d, h)
    xm, xn, te, wr = f(1, S, d), f(1, S, d), f(1, d), f(2 * d, E)
    cfg = R.RouterConfig(d_model=d, n_experts=E, capacity_factor=1.0)
    T = lambda a: torch.tensor(a).cuda()
    out = M.moe_forward(T(xm), T(xn), T(xm), T(te), cfg,
                        M.ExpertBank(*(T(a) for a in (w1, w3, w2, s1, s3, s2))), T(wr))
    shared = O.swiglu_arrays(xm.reshape(-1, d), s1, s3, s2)
    assert rel_fro(np_of(out).reshape(-1, d), shared) <= TOL_FP32
    # single expert, full capacity: shared + alpha/(1+eps) * expert
    alpha = 1.7
    w1, w3, w2 = f(1, 5, 3), f(1, 5, 3), f(1, 3, 5)
    s1, s3, s2 = f(5, 3), f(5, 3), f(3, 5)
    xm, xn, te, wr = f(1, 4, 3), f(1, 4, 3), f(1, 3), f(6, 1)
    cfg = R.RouterConfig(d_model=3, n_experts=1, capacity_factor=1.0, gate_scale=alpha)
    out = M.moe_forward(T(xm), T(xn), T(xm), T(te), cfg,
                        M.ExpertBank(*(T(a) for a in (w1, w3, w2, s1, s3, s2))), T(wr))
    flat = xm.reshape(-1, 3)
    expect = O.swiglu_arrays(flat, s1, s3, s2).astype(np.float64) + \
        alpha / (1 + 1e-6) * O.swiglu_arrays(flat, w1[0], w3[0], w2[0])
    assert rel_fro(np_of(out).reshape(-1, 3), expect) <= TOL_FP32


def test_decoupling_and_determinism_and_permutation():    # test_moe.py:194-217, test_router.py:137-149
    from paper_2604_12163_b200 import moe as M
    from paper_2604_12163_b200 import router as R
    inp = make_layer_inputs(10, 3, 128, 256, 8, 112, mode="bf16")
    g = to_gpu(inp, "bf16")
    cfg = R.RouterConfig(d_model=256, n_experts=8, capacity_factor=2.0)
    bank = bank_of(g)
    o1, d1, r1 = M.moe_forward(g["x_mod"], g["x_norm"], g["x_mod"], g["t_emb"], cfg, bank, g["w_r"],
                               return_routing=True)
    o1b = M.moe_forward(g["x_mod"], g["x_norm"], g["x_mod"], g["t_emb"], cfg, bank, g["w_r"])
    assert torch.equal(o1, o1b)                      # bitwise repeatable
    x10 = (g["x_mod"].float() * 10).to(torch.bfloat16)
    o2, d2, r2 = M.moe_forward(x10, g["x_norm"], x10, g["t_emb"], cfg, bank, g["w_r"],
                               return_routing=True)
    for a, b in zip(d1, d2):
        np.testing.assert_array_equal(a.top_indices, b.top_indices)
        np.testing.assert_array_equal(a.gates, b.gates)
    assert not torch.allclose(o1.float(), o2.float())
    perm = torch.tensor([2, 0, 1]).cuda()
    op = M.moe_forward(g["x_mod"][perm], g["x_norm"][perm], g["x_mod"][perm], g["t_emb"][perm],
                       cfg, bank, g["w_r"])
    assert torch.equal(op, o1[perm])


# ---------------------------------------------------------------- full size
@pytest.mark.parametrize("B,S,C,seed", [
    (16, 1024, 4.0, 2),                       # cfg2 (512px, S512 stage)
    (4, 4096, 2.0, 4),                        # cfg4 shape (1024px, C=2)
    (2, 4096, 8.0, 31), (2, 4096, 4.0, 32),   # cfg3 capacity sweep: cap 512 / 256
    (2, 4032, 2.0, 33), (2, 3840, 2.0, 34),   # multi-aspect 1024 buckets: cap 126 / 120
])
def test_full_width_layer_vs_oracle_and_properties(B, S, C, seed):
    """cfg2 / cfg3 / cfg4 / bucket shapes at full width (d=2048, h=1344, E=64) in bf16.
    Routing for every sample is checked bit-exactly against the oracle's
    router and EVERY sample's layer output against the oracle's full layer
    (run on the host cores, one call for the batch); plus size-independent
    properties over the whole batch."""
    from paper_2604_12163_b200 import moe as M
    from paper_2604_12163_b200 import router as R
    d, h, E = 2048, 1344, 64
    gen = torch.Generator(device="cuda").manual_seed(seed)
    rn = lambda *s, std=1.0: (torch.randn(*s, generator=gen, device="cuda") * std)
    tn = lambda *s, std: torch.clamp(rn(*s, std=std), -2 * std, 2 * std)
    x = rn(B, S, d)
    xn = (x * torch.rsqrt((x * x).mean(-1, keepdim=True) + 1e-6) / np.sqrt(18)).to(torch.bfloat16)
    xm = (xn.float() * (1 + 0.1 * rn(B, 1, d))).to(torch.bfloat16)
    te = rn(B, d)
    wr = tn(2 * d, E, std=0.006)
    ws = [tn(*s, std=0.02).to(torch.bfloat16) for s in ((E, h, d), (E, h, d), (E, d, h), (h, d), (h, d), (d, h))]
    cfg = R.RouterConfig(d_model=d, n_experts=E, capacity_factor=C)
    out, decisions, routing = M.moe_forward(xm, xn, xm, te, cfg, M.ExpertBank(*ws), wr,
                                            return_routing=True)
    cap = routing["capacity"]
    xn_np, te_np, wr_np = np_of(xn), np_of(te), np_of(wr)
    # --- routing of every sample, bit-exact against the oracle router
    r = O.route_full(xn_np, te_np, wr_np, n_experts=E, capacity_factor=C)
    np.testing.assert_array_equal(np_of(routing["logits"]), r["logits"])
    np.testing.assert_array_equal(routing["token_flat"].cpu().numpy(), r["token_flat"])
    np.testing.assert_array_equal(np_of(routing["gates"]), r["gates"])
    # --- properties: exact utilisation, ordering, gate identity
    top = np.stack([dd.top_indices for dd in decisions])            # (B,E,cap)
    aff = np.stack([dd.affinity for dd in decisions])
    for b in range(B):
        for e in range(E):
            assert len(np.unique(top[b, e])) == cap
    assert np.all(np.diff(aff, axis=-1) <= 0)                       # score descending
    # --- every sample's layer output against the oracle layer
    w_np = [np_of(w) for w in ws]
    o_ref = O.moe_forward(xn_np, np_of(xm), te_np, wr_np, *w_np, capacity_factor=C)
    out_np = np_of(out)
    errs = [rel_fro(out_np[b], o_ref[b]) for b in range(B)]
    assert max(errs) <= TOL_BF16, f"per-sample rel-err {errs}"
    assert rel_fro(out_np, o_ref) <= TOL_BF16


def test_host_pipeline_matches_direct_calls():
    """pipeline.HostPipeline (pinned H2D -> moe_forward -> D2H on three
    streams) returns exactly what direct moe_forward calls return."""
    from paper_2604_12163_b200 import moe as M
    from paper_2604_12163_b200 import router as R
    from paper_2604_12163_b200.pipeline import HostPipeline
    inp = make_layer_inputs(12, 2, 256, 512, 16, 224, mode="bf16")
    g = to_gpu(inp, "bf16")
    cfg = R.RouterConfig(d_model=512, n_experts=16, capacity_factor=2.0)
    bank = bank_of(g)
    want = M.moe_forward(g["x_mod"], g["x_norm"], g["x_mod"], g["t_emb"], cfg, bank, g["w_r"]).cpu()
    host = [g[k].cpu().pin_memory() for k in ("x_norm", "x_mod", "t_emb")]
    fn = lambda xn, xm, te: M.moe_forward(xm, xn, xm, te, cfg, bank, g["w_r"])
    pipe = HostPipeline(fn, host, want.shape, want.dtype)
    for _ in range(5):
        pipe.step()
    pipe.drain()
    torch.cuda.synchronize()
    for out in pipe.host_out:
        assert torch.equal(out, want)


def test_full_width_fp32_mode_layer():
    """fp32 mode (CUDA-core expert GEMMs, no TF32) at full width, one 512px
    sample: routing bit-exact, layer rel-err <= 1e-4 against the oracle."""
    from paper_2604_12163_b200 import moe as M
    from paper_2604_12163_b200 import router as R
    B, S, d, h, E, C = 1, 1024, 2048, 1344, 64, 4.0
    inp = make_layer_inputs(41, B, S, d, E, h, layer=17, mode="fp32")
    g = to_gpu(inp, "fp32")
    cfg = R.RouterConfig(d_model=d, n_experts=E, capacity_factor=C)
    out, dec, routing = M.moe_forward(g["x_mod"], g["x_norm"], g["x_mod"], g["t_emb"], cfg,
                                      bank_of(g), g["w_r"], return_routing=True)
    ref_out, ref = O.moe_forward(inp["x_norm"], inp["x_mod"], inp["t_emb"], inp["w_r"], inp["w1"],
                                 inp["w3"], inp["w2"], inp["sw1"], inp["sw3"], inp["sw2"],
                                 capacity_factor=C, return_routing=True)
    np.testing.assert_array_equal(routing["token_flat"].cpu().numpy(), ref["token_flat"])
    np.testing.assert_array_equal(np_of(routing["gates"]), ref["gates"])
    np.testing.assert_array_equal(np_of(routing["logits"]), ref["logits"])
    err = rel_fro(np_of(out), ref_out)
    assert err <= TOL_FP32, f"fp32-mode rel-err {err:.3e}"


@pytest.mark.parametrize("E,C", [(128, 4.0), (96, 2.0)])
def test_router_more_than_64_experts(E, C):
    """E > 64 takes the general FP64 router (DFMA) path: bit-exact vs the oracle."""
    from oracle.workloads import make_router_inputs
    from paper_2604_12163_b200 import router as R
    inp = make_router_inputs(51, 2, 512, 512, E, mode="bf16")
    g = to_gpu(inp, "bf16")
    cfg = R.RouterConfig(d_model=512, n_experts=E, capacity_factor=C)
    dec, routing = R.route_full(g["x_norm"], g["t_emb"], g["w_r"], cfg)
    ref = O.route_full(inp["x_norm"], inp["t_emb"], inp["w_r"], n_experts=E, capacity_factor=C)
    np.testing.assert_array_equal(np_of(routing["logits"]), ref["logits"])
    np.testing.assert_array_equal(routing["token_flat"].cpu().numpy(), ref["token_flat"])
    np.testing.assert_array_equal(np_of(routing["gates"]), ref["gates"])


def test_nan_scores_sort_last():
    """numpy's argsort(-x, stable) puts NaN last (router.py:100): a NaN row of
    x_norm makes that token's scores NaN, so no expert may pick it before any
    finite-scored token, and ties among NaNs go to the lower index."""
    from paper_2604_12163_b200 import router as R
    rng = np.random.default_rng(3)
    S, d, E = 64, 16, 4
    xn = rng.normal(size=(1, S, d)).astype(np.float32)
    xn[0, [5, 9]] = np.nan
    te = rng.normal(size=(1, d)).astype(np.float32)
    wr = rng.normal(size=(2 * d, E)).astype(np.float32)
    cfg = R.RouterConfig(d_model=d, n_experts=E, capacity_factor=float(E))   # cap = S
    dec, routing = R.route_full(torch.tensor(xn).cuda(), torch.tensor(te).cuda(),
                                torch.tensor(wr).cuda(), cfg)
    ref = O.route_full(xn, te, wr, n_experts=E, capacity_factor=float(E))
    np.testing.assert_array_equal(routing["token_flat"].cpu().numpy(), ref["token_flat"])
    for e in range(E):
        assert list(dec[0].top_indices[e][-2:]) == [5, 9]


def test_fused_gather_variants_bitwise_equal():
    """NIMG_FUSED_GATHER=1 (routed-row gather fused into GEMM1: cp.async in the
    CTA-pair kernel; TMA gather4 in the 1-CTA kernel with NIMG_PAIR=0) gives
    the same bits as the default separate gather kernel."""
    import os
    import subprocess
    import sys
    code = (
        "import torch, numpy as np, sys\n"
        "sys.path.insert(0, '.')\n"
        "from oracle.workloads import make_layer_inputs\n"
        "from tests.gpu_helpers import to_gpu, bank_of\n"
        "from paper_2604_12163_b200 import moe as M, router as R\n"
        "inp = make_layer_inputs(61, 2, 512, 512, 16, 224, mode='bf16')\n"
        "g = to_gpu(inp, 'bf16')\n"
        "cfg = R.RouterConfig(d_model=512, n_experts=16, capacity_factor=4.0)\n"
        "out = M.moe_forward(g['x_mod'], g['x_norm'], g['x_mod'], g['t_emb'], cfg, bank_of(g), g['w_r'])\n"
        "np.save(sys.argv[1], out.float().cpu().numpy())\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for tag, env in (("base", {}), ("pair", {"NIMG_FUSED_GATHER": "1"}),
                     ("g4", {"NIMG_FUSED_GATHER": "1", "NIMG_PAIR": "0"})):
        path = f"/tmp/nimg_fg_{tag}.npy"
        r = subprocess.run([sys.executable, "-c", code, path], cwd=root, capture_output=True,
                           text=True, env={**os.environ, **env}, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[tag] = np.load(path)
    np.testing.assert_array_equal(outs["pair"], outs["base"])
    # the 1-CTA kernel accumulates in a different tile order; allow rounding-level differences
    assert rel_fro(outs["g4"], outs["base"]) < 1e-2


@pytest.mark.parametrize("name", G.names("block"))
def test_block_vs_reference_golden(name):
    """MoE branch of MoEDiT.forward (backbone.py:583-606), fp32: h, x_norm,
    x_mod and the routing bit-exact with the reference; the updated residual
    stream within the fp32 bar."""
    from paper_2604_12163_b200 import block as BK
    from paper_2604_12163_b200 import moe as M
    from paper_2604_12163_b200 import router as R
    kind, p, inp, exp = G.case(name)
    T = lambda k: torch.from_numpy(inp[k]).cuda()
    cfg = R.RouterConfig(d_model=p["d"], n_experts=p["E"], capacity_factor=p["C"])
    bank = M.ExpertBank(*(T(k) for k in ("w1", "w3", "w2", "sw1", "sw3", "sw2")))
    out, dec, routing, mid = BK.moe_block_forward(
        T("x"), T("sa_gate"), T("r_attn"), T("ff_scale"), T("ff_gate"), T("t_vec"), p["layer"], cfg,
        bank, T("w_r"), return_routing=True, return_intermediates=True)
    for k in ("h", "x_norm", "x_mod"):
        np.testing.assert_array_equal(np_of(mid[k]), exp[k], err_msg=k)
    np.testing.assert_array_equal(routing["token_flat"].cpu().numpy(), exp["token_flat"])
    np.testing.assert_array_equal(np_of(routing["gates"]), exp["gates"])
    np.testing.assert_array_equal(np_of(routing["logits"]), exp["logits"])
    err = rel_fro(np_of(out), exp["out"])
    assert err <= TOL_FP32, f"{name}: rel-err {err:.3e}"


def test_block_full_width_bf16():
    """bf16 block at full width (d=2048, E=64, h=1344), 512px x 2: the fused
    prologue (fp32 math, bf16 storage) matches the numpy chain to a bf16 ulp;
    routing of the produced x_norm is bit-exact with the oracle router; the
    residual output matches h + tanh(ff_gate) * oracle layer(x_norm, x_mod)."""
    from oracle.workloads import bf16_round, make_block_inputs
    from paper_2604_12163_b200 import block as BK
    from paper_2604_12163_b200 import moe as M
    from paper_2604_12163_b200 import router as R
    B, S, d, E, h, C, layer = 2, 1024, 2048, 64, 1344, 4.0, 17
    inp = make_block_inputs(71, B, S, d, E, h, mode="bf16")
    bf = torch.bfloat16
    T = lambda k, dt=None: torch.from_numpy(inp[k]).cuda().to(dt or torch.float32)
    cfg = R.RouterConfig(d_model=d, n_experts=E, capacity_factor=C)
    bank = M.ExpertBank(*(T(k, bf) for k in ("w1", "w3", "w2", "sw1", "sw3", "sw2")))
    out, dec, routing, mid = BK.moe_block_forward(
        T("x", bf), T("sa_gate"), T("r_attn", bf), T("ff_scale"), T("ff_gate"), T("t_vec"), layer,
        cfg, bank, T("w_r"), return_routing=True, return_intermediates=True)
    # prologue chain in numpy (f64 ops, bf16 storage rounding)
    f64 = np.float64
    hh = bf16_round((inp["x"].astype(f64) + np.tanh(inp["sa_gate"].astype(f64))[:, None, :]
                     * inp["r_attn"].astype(f64)).astype(np.float32))
    ms = (hh.astype(f64) ** 2).mean(axis=-1, keepdims=True) + 1e-6
    xn0 = bf16_round((hh.astype(f64) / np.sqrt(ms)).astype(np.float32))
    sc = float(bf16_round(np.array([1.0 / np.sqrt(layer + 1)], np.float32))[0])
    xn = bf16_round((xn0.astype(f64) * sc).astype(np.float32))
    onep = (inp["ff_scale"].astype(f64) + 1.0).astype(np.float32).astype(f64)[:, None, :]
    xm = bf16_round((xn.astype(f64) * onep).astype(np.float32))
    for k, ref_v in (("h", hh), ("x_norm", xn), ("x_mod", xm)):
        got = np_of(mid[k])
        # fp32 vs f64 intermediates: <= 2 bf16 ulps (two chained roundings)
        np.testing.assert_allclose(got, ref_v, rtol=2 ** -6, atol=1e-6, err_msg=k)
    xn = np_of(mid["x_norm"])                           # route / layer on what the GPU produced
    xm = np_of(mid["x_mod"])
    hh = np_of(mid["h"])
    r = O.route_full(xn, inp["t_vec"], inp["w_r"], n_experts=E, capacity_factor=C)
    np.testing.assert_array_equal(routing["token_flat"].cpu().numpy(), r["token_flat"])
    w = {k: inp[k] for k in ("w1", "w3", "w2", "sw1", "sw3", "sw2")}
    moe = O.moe_forward(xn, xm, inp["t_vec"], inp["w_r"], w["w1"], w["w3"], w["w2"],
                        w["sw1"], w["sw3"], w["sw2"], capacity_factor=C)
    want = hh.astype(f64) + np.tanh(inp["ff_gate"].astype(f64))[:, None, :] * moe
    got = np_of(out)
    errs = [rel_fro(got[b], want[b]) for b in range(B)]
    assert max(errs) <= TOL_BF16, f"block bf16 per-sample rel-err {errs}"


@pytest.mark.parametrize("B,S,d,E,h,C", [(1, 40, 256, 8, 128, 1.0), (3, 56, 512, 8, 192, 2.0),
                                         (2, 72, 256, 8, 64, 2.0)])
def test_ragged_routed_rows_tcgen05(B, S, d, E, h, C):
    """tcgen05 shapes whose routed row count is not a multiple of the 32-row
    background-gather sub-block or the 256-row pair tile (40 = 8 x 5 rows;
    336 = 8 x 3 x 14; 288): the gather inside GEMM1 and its flags at the
    edges; h = 192 and 64 also end every GEMM1 row block with a half-width
    tile (h = 64: the only one)."""
    from paper_2604_12163_b200 import moe as M
    from paper_2604_12163_b200 import router as R
    inp = make_layer_inputs(61, B, S, d, E, h, mode="bf16")
    g = to_gpu(inp, "bf16")
    cfg = R.RouterConfig(d_model=d, n_experts=E, capacity_factor=C)
    out, _, routing = M.moe_forward(g["x_mod"], g["x_norm"], g["x_mod"], g["t_emb"], cfg, bank_of(g),
                                    g["w_r"], return_routing=True)
    ref_out, ref = O.moe_forward(inp["x_norm"], inp["x_mod"], inp["t_emb"], inp["w_r"], inp["w1"],
                                 inp["w3"], inp["w2"], inp["sw1"], inp["sw3"], inp["sw2"],
                                 capacity_factor=C, return_routing=True)
    np.testing.assert_array_equal(routing["token_flat"].cpu().numpy(), ref["token_flat"])
    assert rel_fro(np_of(out), ref_out) <= TOL_BF16


# ---------------------------------------------------------------- dtypes
def test_router_reads_x_norm_in_its_own_dtype():
    """fp32 x_norm with bf16 x_mod: the routing is computed on the fp32 x_norm
    values (router.py:120-122), bit-exact with the oracle's fp32 routing --
    not on a bf16-rounded copy; the experts run bf16 on x_mod."""
    from paper_2604_12163_b200 import moe as M
    from paper_2604_12163_b200 import router as R
    B, S, d, E, h, C = 2, 1024, 2048, 64, 1344, 4.0
    inp = make_layer_inputs(43, B, S, d, E, h, layer=17, mode="fp32")
    g = to_gpu(inp, "bf16")
    xn32 = torch.from_numpy(inp["x_norm"]).cuda()           # fp32, not bf16-representable
    assert not torch.equal(xn32, xn32.to(torch.bfloat16).float())
    cfg = R.RouterConfig(d_model=d, n_experts=E, capacity_factor=C)
    out, dec, routing = M.moe_forward(g["x_mod"], xn32, g["x_mod"], g["t_emb"], cfg, bank_of(g),
                                      g["w_r"], return_routing=True)
    assert out.dtype == torch.bfloat16
    r = O.route_full(inp["x_norm"], inp["t_emb"], inp["w_r"], n_experts=E, capacity_factor=C)
    np.testing.assert_array_equal(np_of(routing["logits"]), r["logits"])
    np.testing.assert_array_equal(routing["token_flat"].cpu().numpy(), r["token_flat"])
    np.testing.assert_array_equal(np_of(routing["gates"]), r["gates"])
    # the bf16-rounded router input would have routed differently
    r16 = O.route_full(np_of(xn32.to(torch.bfloat16)), inp["t_emb"], inp["w_r"], n_experts=E,
                       capacity_factor=C)
    assert not np.array_equal(r16["logits"], r["logits"])
    xm_np = np_of(g["x_mod"])
    w_np = [np_of(g[k]) for k in ("w1", "w3", "w2", "sw1", "sw3", "sw2")]
    o_ref = O.moe_forward(inp["x_norm"], xm_np, inp["t_emb"], inp["w_r"], *w_np, capacity_factor=C)
    assert rel_fro(np_of(out), o_ref) <= TOL_BF16
    # and route_full / route alone take the fp32 x_norm the same way
    dec2, rt2 = R.route_full(xn32, g["t_emb"], g["w_r"], cfg)
    np.testing.assert_array_equal(np_of(rt2["logits"]), r["logits"])


@pytest.mark.parametrize("B,S,d,E,h,C,gs", [(2, 256, 256, 8, 168, 2.0, 1.0),
                                            (3, 37, 24, 5, 20, 1.7, 1.7),
                                            (1, 1024, 2048, 64, 1344, 4.0, 1.0)])
def test_f64_mode_layer_vs_oracle(B, S, d, E, h, C, gs):
    """The reference's f64 storage mode (tensor.py:39-47): f64 activations with
    the backbone's fp32 weights promote the whole layer to f64 (routing,
    experts, combine, output). Against the oracle in f64: selections equal,
    f64 values to summation-order level."""
    from paper_2604_12163_b200 import moe as M
    from paper_2604_12163_b200 import router as R
    inp = make_layer_inputs(51, B, S, d, E, h, layer=5, mode="fp32")
    f64 = np.float64
    x64 = {k: inp[k].astype(f64) for k in ("x_norm", "x_mod", "t_emb")}
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    ws = [T(inp[k]) for k in ("w1", "w3", "w2", "sw1", "sw3", "sw2")]      # fp32 weights
    cfg = R.RouterConfig(d_model=d, n_experts=E, capacity_factor=C, gate_scale=gs)
    out, dec, routing = M.moe_forward(T(x64["x_mod"]), T(x64["x_norm"]), T(x64["x_mod"]),
                                      T(x64["t_emb"]), cfg, M.ExpertBank(*ws), T(inp["w_r"]),
                                      return_routing=True)
    assert out.dtype == torch.float64 and routing["gates"].dtype == torch.float64
    ref_out, ref = O.moe_forward(x64["x_norm"], x64["x_mod"], x64["t_emb"], inp["w_r"], inp["w1"],
                                 inp["w3"], inp["w2"], inp["sw1"], inp["sw3"], inp["sw2"],
                                 capacity_factor=C, gate_scale=gs, return_routing=True)
    assert ref_out.dtype == f64
    np.testing.assert_array_equal(routing["token_flat"].cpu().numpy(), ref["token_flat"])
    assert rel_fro(routing["logits"].cpu().numpy(), ref["logits"]) < 1e-14
    assert rel_fro(routing["gates"].cpu().numpy(), ref["gates"]) < 1e-14
    assert rel_fro(out.cpu().numpy(), ref_out) < 1e-12
    # grouped_forward / swiglu take the same f64 path
    y = M.swiglu(T(x64["x_mod"][0]), ws[3], ws[4], ws[5])
    y_ref = O.swiglu_arrays(x64["x_mod"][0], inp["sw1"], inp["sw3"], inp["sw2"])
    assert y.dtype == torch.float64 and rel_fro(y.cpu().numpy(), y_ref) < 1e-13


def test_f64_mode_is_forward_only():
    from paper_2604_12163_b200 import moe as M
    from paper_2604_12163_b200 import router as R
    from paper_2604_12163_b200.errors import ConfigError
    inp = make_layer_inputs(52, 1, 64, 64, 4, 64, mode="fp32")
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    xn = T(inp["x_norm"].astype(np.float64)).requires_grad_(True)
    bank = M.ExpertBank(*(T(inp[k]) for k in ("w1", "w3", "w2", "sw1", "sw3", "sw2")))
    cfg = R.RouterConfig(d_model=64, n_experts=4, capacity_factor=2.0)
    with pytest.raises(ConfigError):
        M.moe_forward(T(inp["x_mod"]), xn, T(inp["x_mod"]), T(inp["t_emb"]), cfg, bank,
                      T(inp["w_r"]))


@pytest.mark.parametrize("B,S,d,E,h,C", [(2, 192, 256, 8, 128, 2.0), (3, 100, 512, 16, 192, 1.7)])
def test_fp32_mode_tensor_core_split(B, S, d, E, h, C):
    """fp32 layers whose widths tile the pair kernels run on the bf16 tensor
    cores with split operands (bf16x3, csrc/split_kernels.cu): routing
    bit-exact, layer and swiglu within the fp32 bar against the oracle."""
    from paper_2604_12163_b200 import _lib as L
    from paper_2604_12163_b200 import moe as M
    from paper_2604_12163_b200 import router as R
    f = L.FfnDesc(n_rows=B * S, n_shared_rows=B * S, d=d, h=h, h_shared=h, n_experts=E,
                  act_dtype=L.NIMG_F32, nseg=E)
    import ctypes as C_
    p, y = C_.c_int32(), C_.c_int32()
    L.lib.nimg_ffn_path(C_.byref(f), C_.byref(p), C_.byref(y))
    assert p.value == L.NIMG_PATH_TCGEN05 and y.value == L.NIMG_F32
    inp = make_layer_inputs(91, B, S, d, E, h, mode="fp32")
    g = to_gpu(inp, "fp32")
    cfg = R.RouterConfig(d_model=d, n_experts=E, capacity_factor=C)
    out, _, routing = M.moe_forward(g["x_mod"], g["x_norm"], g["x_mod"], g["t_emb"], cfg, bank_of(g),
                                    g["w_r"], return_routing=True)
    ref_out, ref = O.moe_forward(inp["x_norm"], inp["x_mod"], inp["t_emb"], inp["w_r"], inp["w1"],
                                 inp["w3"], inp["w2"], inp["sw1"], inp["sw3"], inp["sw2"],
                                 capacity_factor=C, return_routing=True)
    assert out.dtype == torch.float32
    np.testing.assert_array_equal(routing["token_flat"].cpu().numpy(), ref["token_flat"])
    np.testing.assert_array_equal(np_of(routing["gates"]), ref["gates"])
    err = rel_fro(np_of(out), ref_out)
    assert err <= TOL_FP32, f"fp32 (tensor-core split) rel-err {err:.3e}"
    ys = M.swiglu(g["x_mod"][0], g["sw1"], g["sw3"], g["sw2"])
    ys_ref = O.swiglu_arrays(inp["x_mod"][0], inp["sw1"], inp["sw3"], inp["sw2"])
    assert rel_fro(np_of(ys), ys_ref) <= TOL_FP32
