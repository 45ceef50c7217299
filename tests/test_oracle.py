"""Pin the CPU oracle (oracle/nimg_oracle.py) to the reference.

1. Bit-exact against golden vectors written by the real reference
   (tests/golden/make_golden.py) -- runs everywhere, including the GPU box.
2. Bit-exact against the live reference on seeded random instances shaped
   like the reference's own tests (test_moe.py:179-191, test_router.py:78-95)
   -- only where /root/reference is mounted.
3. The reference's known-answer tests restated against the oracle
   (test_router.py:15-75, test_moe.py:19-33, :147-176).
"""

import numpy as np
import pytest

from oracle import nimg_oracle as O
from tests import golden_cases as G
from tests.refimport import load_reference, reference_available


@pytest.mark.parametrize("name", G.names("block"))
def test_oracle_block_matches_reference_golden(name):
    """backbone.py:583-606 (MoE branch around the layer) composed from the
    reference's own functions vs the oracle restatement: bit-exact."""
    kind, p, inp, exp = G.case(name)
    res, r = O.moe_block_forward(inp["x"], inp["sa_gate"], inp["r_attn"], inp["ff_scale"],
                                 inp["ff_gate"], inp["t_vec"], p["layer"], inp["w_r"], inp["w1"],
                                 inp["w3"], inp["w2"], inp["sw1"], inp["sw3"], inp["sw2"],
                                 capacity_factor=p["C"], return_routing=True)
    for k in ("h", "x_norm", "x_mod", "moe", "out"):
        np.testing.assert_array_equal(res[k], exp[k], err_msg=k)
    np.testing.assert_array_equal(r["token_flat"], exp["token_flat"])
    np.testing.assert_array_equal(r["gates"], exp["gates"])


@pytest.mark.parametrize("name", G.names("moe") + G.names("route"))
def test_oracle_matches_reference_golden(name):
    kind, p, inp, exp = G.case(name)
    kw = dict(capacity_factor=p["C"], gate_scale=p.get("gate_scale", 1.0))
    if kind == "moe":
        out, r = O.moe_forward(inp["x_norm"], inp["x_mod"], inp["t_emb"], inp["w_r"],
                               inp["w1"], inp["w3"], inp["w2"], inp["sw1"], inp["sw3"],
                               inp["sw2"], return_routing=True, **kw)
        np.testing.assert_array_equal(out, exp["out"])
        assert out.dtype == exp["out"].dtype
    else:
        r = O.route_full(inp["x_norm"], inp["t_emb"], inp["w_r"], n_experts=p["E"], **kw)
    assert r["capacity"] == int(exp["capacity"])
    np.testing.assert_array_equal(r["logits"], exp["logits"])
    np.testing.assert_array_equal(r["token_flat"], exp["token_flat"])
    np.testing.assert_array_equal(r["gates"], exp["gates"])
    np.testing.assert_array_equal(r["top"], exp["top"])
    dec = O.decisions_from(r)
    np.testing.assert_array_equal(np.stack([d["affinity"] for d in dec]), exp["affinity"])


@pytest.mark.skipif(not reference_available(), reason="reference tree not mounted")
def test_oracle_matches_live_reference_random():
    ref = load_reference()
    T = ref.tensor.Tensor
    rng = np.random.default_rng(123)
    for trial in range(12):
        B = int(rng.integers(1, 4))
        S = int(rng.integers(2, 40))
        E = int(rng.integers(1, 9))
        C = float(rng.uniform(0.5, 8.0))
        d = int(rng.integers(2, 12))
        h = int(rng.integers(2, 10))
        dt = np.float32 if trial % 2 == 0 else np.float64
        mk = lambda *s: rng.normal(size=s).astype(dt)
        xn, xm, te, wr = mk(B, S, d), mk(B, S, d), mk(B, d), mk(2 * d, E)
        w1, w3, w2 = mk(E, h, d), mk(E, h, d), mk(E, d, h)
        s1, s3, s2 = mk(h, d), mk(h, d), mk(d, h)
        alpha = float(rng.uniform(0.5, 2.0))
        cfg = ref.router.RouterConfig(d_model=d, n_experts=E, capacity_factor=C, gate_scale=alpha)
        bank = ref.moe.ExpertBank(*(T(a, dtype=dt) for a in (w1, w3, w2, s1, s3, s2)))
        with ref.tensor.no_grad():
            out, dec, routing = ref.moe.moe_forward(T(xm, dtype=dt), T(xn, dtype=dt), T(xm, dtype=dt),
                                                    T(te, dtype=dt), cfg, bank, T(wr, dtype=dt),
                                                    return_routing=True)
        o_out, r = O.moe_forward(xn, xm, te, wr, w1, w3, w2, s1, s3, s2, capacity_factor=C,
                                 gate_scale=alpha, return_routing=True)
        np.testing.assert_array_equal(o_out, out.data, err_msg=f"trial {trial}")
        np.testing.assert_array_equal(r["token_flat"], routing["token_flat"])
        np.testing.assert_array_equal(r["gates"], routing["gates"].data)
        np.testing.assert_array_equal(r["logits"], routing["logits"].data)
        for b, d_ in enumerate(O.decisions_from(r)):
            np.testing.assert_array_equal(d_["top_indices"], dec[b].top_indices)
            np.testing.assert_array_equal(d_["gates"], dec[b].gates)
            np.testing.assert_array_equal(d_["affinity"], dec[b].affinity)


@pytest.mark.skipif(not reference_available(), reason="reference tree not mounted")
def test_oracle_grouped_forward_matches_reference():
    ref = load_reference()
    T = ref.tensor.Tensor
    rng = np.random.default_rng(5)
    E, h, d = 3, 4, 5
    counts = [2, 0, 3]
    w1, w3, w2 = rng.normal(size=(E, h, d)), rng.normal(size=(E, h, d)), rng.normal(size=(E, d, h))
    toks = rng.normal(size=(sum(counts), d))
    off = np.concatenate([[0], np.cumsum(counts)])
    bank = ref.moe.ExpertBank(T(w1, dtype=np.float64), T(w3, dtype=np.float64), T(w2, dtype=np.float64),
                              T(w1[0], dtype=np.float64), T(w3[0], dtype=np.float64), T(w2[0], dtype=np.float64))
    with ref.tensor.no_grad():
        want = ref.moe.grouped_forward(ref.moe.GroupedBatch(T(toks, dtype=np.float64), off), bank).data
    np.testing.assert_array_equal(O.grouped_forward(toks, off, w1, w3, w2), want)


# --- the reference's known-answer tests, restated on the oracle -------------

def test_capacity_kats():                                    # test_router.py:15-28
    assert O.capacity_for(256, 64, 8.0) == 32
    assert O.capacity_for(1024, 64, 4.0) == 64
    assert O.capacity_for(5, 64, 8.0) == 1
    assert O.capacity_for(4, 2, 100.0) == 4
    with pytest.raises(O.ConfigError):
        O.capacity_for(0, 2, 1.0)
    with pytest.raises(O.ConfigError):
        O.capacity_for(4, 2, 0.0)


def test_capacity_schedule_anchors():                        # test_router.py:32-45
    S = O.StageId
    assert O.capacity_schedule(3, S.S1024) == 4.0
    assert O.capacity_schedule(4, S.S1024) == 4.0
    assert O.capacity_schedule(5, S.S1024) == 2.0
    assert O.capacity_schedule(31, S.S1024) == 2.0
    assert O.capacity_schedule(17, S.S256) == 8.0
    assert O.capacity_schedule(17, S.S512) == 4.0
    assert O.capacity_schedule(0, S.S256) is O.DENSE
    with pytest.raises(IndexError):
        O.capacity_schedule(32, S.S256)


def test_uniform_logits_tie_break():                         # test_router.py:48-58
    rng = np.random.default_rng(0)
    r = O.route_full(rng.normal(size=(1, 6, 4)), rng.normal(size=(1, 4)), np.zeros((8, 2)),
                     n_experts=2, capacity_factor=1.0)
    cap = O.capacity_for(6, 2, 1.0)
    for e in range(2):
        np.testing.assert_array_equal(r["top"][0, e], np.arange(cap))
    np.testing.assert_allclose(O.decisions_from(r)[0]["affinity"], 0.5, atol=1e-12)


def test_full_capacity_gates_sum_to_one():                   # test_router.py:61-75
    rng = np.random.default_rng(1)
    wr = rng.normal(size=(8, 2))
    r = O.route_full(rng.normal(size=(1, 4, 4)), rng.normal(size=(1, 4)), wr,
                     n_experts=2, capacity_factor=2.0)
    dec = O.decisions_from(r)[0]
    per_tok = np.zeros(4)
    np.add.at(per_tok, dec["top_indices"].reshape(-1), dec["gates"].reshape(-1))
    np.testing.assert_allclose(per_tok, 1.0, atol=1e-5)


def test_swiglu_scalar_reduction():                          # test_moe.py:28-33
    one = np.ones((1, 1))
    for x in (-1.3, 0.0, 0.7, 2.5):
        out = O.swiglu_arrays(np.array([[x]]), one, one, one)
        np.testing.assert_allclose(out[0, 0], x / (1 + np.exp(-x)) * x, rtol=1e-12)


def test_single_expert_full_capacity():                      # test_moe.py:157-176
    rng = np.random.default_rng(7)
    d, S, h, alpha = 3, 4, 5, 1.7
    w1, w3, w2 = rng.normal(size=(1, h, d)), rng.normal(size=(1, h, d)), rng.normal(size=(1, d, h))
    s1, s3, s2 = rng.normal(size=(h, d)), rng.normal(size=(h, d)), rng.normal(size=(d, h))
    wr = rng.normal(size=(2 * d, 1))
    xm, xn, te = rng.normal(size=(1, S, d)), rng.normal(size=(1, S, d)), rng.normal(size=(1, d))
    out = O.moe_forward(xn, xm, te, wr, w1, w3, w2, s1, s3, s2, capacity_factor=1.0,
                        gate_scale=alpha)
    flat = xm.reshape(-1, d)
    expect = O.swiglu_arrays(flat, s1, s3, s2) + alpha / (1 + 1e-6) * O.swiglu_arrays(
        flat, w1[0], w3[0], w2[0])
    np.testing.assert_allclose(out.reshape(-1, d), expect, rtol=1e-9)


def test_zero_w2_gives_shared_only():                        # test_moe.py:147-154
    rng = np.random.default_rng(6)
    d, E, h = 4, 2, 4
    w1, w3 = rng.normal(size=(E, h, d)), rng.normal(size=(E, h, d))
    w2 = np.zeros((E, d, h))
    s1, s3, s2 = rng.normal(size=(h, d)), rng.normal(size=(h, d)), rng.normal(size=(d, h))
    xm = rng.normal(size=(1, 6, d))
    out = O.moe_forward(rng.normal(size=(1, 6, d)), xm, rng.normal(size=(1, d)),
                        rng.normal(size=(2 * d, E)), w1, w3, w2, s1, s3, s2, capacity_factor=1.0)
    np.testing.assert_array_equal(out.reshape(-1, d), O.swiglu_arrays(xm.reshape(-1, d), s1, s3, s2))


# ------------------------------------------------------------------ backward
GRAD_NAMES = ("x_norm", "x_mod", "t_emb", "w_r", "w1", "w3", "w2", "sw1", "sw3", "sw2")


@pytest.mark.parametrize("name", G.names("moe_bwd"))
def test_oracle_backward_matches_reference_golden(name):
    """Reference Tape + backward through moe_forward (tensor.py:590-628) vs
    the oracle's restated pullbacks: bit-exact f64 gradients."""
    kind, p, inp, exp = G.case(name)
    g = O.moe_backward(*(inp[k] for k in GRAD_NAMES), inp["g_out"], capacity_factor=p["C"],
                       gate_scale=p.get("gate_scale", 1.0))
    for k in GRAD_NAMES:
        np.testing.assert_array_equal(g[k], exp[f"grad_{k}"], err_msg=k)


def test_oracle_backward_vs_finite_differences():
    """test_moe.py:220-236 restated on the oracle: central differences of the
    oracle forward against the oracle backward (f64 inputs)."""
    rng = np.random.default_rng(11)
    B, S, d, E, C, h = 1, 5, 3, 2, 1.5, 4
    a = {"x_norm": rng.normal(size=(B, S, d)), "x_mod": rng.normal(size=(B, S, d)),
         "t_emb": rng.normal(size=(B, d)), "w_r": rng.normal(size=(2 * d, E)),
         "w1": rng.normal(size=(E, h, d)), "w3": rng.normal(size=(E, h, d)),
         "w2": rng.normal(size=(E, d, h)), "sw1": rng.normal(size=(h, d)),
         "sw3": rng.normal(size=(h, d)), "sw2": rng.normal(size=(d, h))}

    def loss(v):
        out = O.moe_forward(v["x_norm"], v["x_mod"], v["t_emb"], v["w_r"], v["w1"], v["w3"],
                            v["w2"], v["sw1"], v["sw3"], v["sw2"], capacity_factor=C)
        return float((out * out).sum())

    out = O.moe_forward(*(a[k] for k in GRAD_NAMES), capacity_factor=C)
    g = O.moe_backward(*(a[k] for k in GRAD_NAMES), 2.0 * out, capacity_factor=C)
    hstep = 1e-5
    for k in ("x_mod", "w_r", "w1", "w3", "w2", "sw1"):
        flat = a[k].reshape(-1)
        num = np.zeros_like(flat)
        for i in range(flat.size):
            keep = flat[i]
            flat[i] = keep + hstep
            fp = loss(a)
            flat[i] = keep - hstep
            fm = loss(a)
            flat[i] = keep
            num[i] = (fp - fm) / (2 * hstep)
        an = g[k].reshape(-1)
        rel = np.abs(an - num) / np.maximum(1e-8, np.abs(an) + np.abs(num))
        assert rel.max() <= 1e-5, (k, rel.max())


@pytest.mark.skipif(not reference_available(), reason="reference tree not mounted")
@pytest.mark.parametrize("seed,B,S,d,E,h,C,gs", [(31, 2, 9, 6, 3, 5, 1.5, 1.0),
                                                 (32, 1, 16, 8, 4, 8, 4.0, 0.5)])
def test_oracle_backward_matches_live_reference(seed, B, S, d, E, h, C, gs):
    ref = load_reference()
    nt = ref.tensor
    rng = np.random.default_rng(seed)
    a = {"x_norm": rng.normal(size=(B, S, d)), "x_mod": rng.normal(size=(B, S, d)),
         "t_emb": rng.normal(size=(B, d)), "w_r": rng.normal(size=(2 * d, E)),
         "w1": rng.normal(size=(E, h, d)), "w3": rng.normal(size=(E, h, d)),
         "w2": rng.normal(size=(E, d, h)), "sw1": rng.normal(size=(h, d)),
         "sw3": rng.normal(size=(h, d)), "sw2": rng.normal(size=(d, h))}
    a = {k: v.astype(np.float32) for k, v in a.items()}
    gout = rng.normal(size=(B, S, d)).astype(np.float32)
    ts = {k: nt.Tensor(v, requires_grad=True, dtype=np.float32) for k, v in a.items()}
    cfg = ref.router.RouterConfig(d_model=d, n_experts=E, capacity_factor=C, gate_scale=gs)
    bank = ref.moe.ExpertBank(ts["w1"], ts["w3"], ts["w2"], ts["sw1"], ts["sw3"], ts["sw2"])
    with nt.Tape() as tape:
        out = ref.moe.moe_forward(ts["x_mod"], ts["x_norm"], ts["x_mod"], ts["t_emb"], cfg, bank,
                                  ts["w_r"])
        loss = nt.sum(nt.mul(out, nt.Tensor(gout, dtype=np.float32)))
    nt.backward(tape, loss)
    g = O.moe_backward(*(a[k] for k in GRAD_NAMES), gout, capacity_factor=C, gate_scale=gs)
    for k in GRAD_NAMES:
        np.testing.assert_array_equal(g[k], ts[k].grad, err_msg=k)
