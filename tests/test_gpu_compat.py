"""The drop-in inside the reference's OWN MoE block caller.

`compat.install(bb)` rebinds the name the reference backbone calls
(backbone.py:24, :595-597); the reference's `MoEDiT.forward` then runs with the
B200 layer in place of its numpy MoE, and everything around it (attention,
modulation, `fused_gated_residual` at backbone.py:47-51, the aux bookkeeping at
backbone.py:598-605) is the reference's own code. The backbone hands the MoE
float64 inputs (backbone.py:259-261), so this exercises the f64 mode.

Checked against the golden velocity and routing the stock reference wrote
(tests/golden/make_golden.py) and against the stock reference run here.
The reference is loaded from $NIMG_REF, /root/reference or the offline
install under baseline/_ref (tests/refimport.py)."""

import numpy as np
import pytest
import torch

from oracle.workloads import DIT_PROMPTS, make_bwd_inputs, make_layer_inputs, perturb_modulation
from tests import golden_cases as G
from tests.gpu_helpers import TOL_FP32, rel_fro
from tests.refimport import load_reference, reference_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not reference_available(), reason="reference package not found")]


def _model(ref, p):
    bb = ref.backbone
    model = bb.MoEDiT(bb.ModelConfig(**p["model"]))
    params = {k: v.data for k, v in model.named_parameters().items()}
    perturb_modulation(params, p["mod_seed"])
    ctx = model.precompute_text_kv(list(DIT_PROMPTS[:p["B"]]))
    return model, ctx


def _forward(ref, model, ctx, inp, p):
    import importlib
    nt = ref.tensor
    rt = importlib.import_module("nimg_ref.router")
    with nt.no_grad():
        return model.forward(nt.Tensor(inp["z"], dtype=np.float32), inp["t"], ctx,
                             rt.StageId[p["stage"]])


@pytest.mark.parametrize("name", G.names("dit"))
def test_reference_moedit_forward_with_dropin(name):
    from paper_2604_12163_b200 import compat
    ref = load_reference()
    bb = ref.backbone
    _, p, inp, exp = G.case(name)
    model, ctx = _model(ref, p)
    stock = bb.moe_forward
    fn = compat.install(bb)
    try:
        assert bb.moe_forward is fn and compat.install(bb) is fn   # idempotent
        vel, aux = _forward(ref, model, ctx, inp, p)
    finally:
        compat.uninstall(bb)
    assert bb.moe_forward is stock
    # the reference's own types came back through the drop-in
    assert isinstance(vel, ref.tensor.Tensor) and vel.data.dtype == exp["vel"].dtype
    assert len(aux["decisions"]) == len([k for k in exp if k.startswith("top_")])
    for j, (layer, decs) in enumerate(aux["decisions"]):
        assert all(isinstance(d, ref.router.RouterDecision) for d in decs)
        np.testing.assert_array_equal(np.stack([d.top_indices for d in decs]), exp[f"top_{layer}"])
        lg = aux["router_logits"][j]
        assert isinstance(lg, ref.tensor.Tensor) and lg.data.dtype == np.float64   # f64 mode
        assert rel_fro(lg.data, exp[f"logits_{layer}"]) < 1e-13
    # MoE in f64 on the GPU vs numpy f64: only the summation order differs
    err = rel_fro(vel.data, exp["vel"])
    # the stock reference, run on this host, against its golden (written on
    # another CPU: OpenBLAS kernels differ in the last f64 bits)
    vel_stock, _ = _forward(ref, model, ctx, inp, p)
    err_stock = rel_fro(vel_stock.data, exp["vel"])
    print(f"{name}: drop-in vs golden {err:.3e}, stock vs golden {err_stock:.3e}, "
          f"drop-in vs stock {rel_fro(vel.data, vel_stock.data):.3e}")
    assert err_stock < 1e-12
    assert err < 1e-12       # measured 2.2e-16 (dit_cfg1), 6.0e-17 (dit_small)


@pytest.mark.parametrize("name", ["cfg1_fp32", "ragged_fp32"])
def test_dropin_layer_fp32_reference_types(name):
    """moe_forward through the adapter on the reference's fp32 Tensors /
    RouterConfig / ExpertBank: routing bit-exact, out within the fp32 bar."""
    from paper_2604_12163_b200 import compat
    ref = load_reference()
    nt, rt, rm = ref.tensor, ref.router, ref.moe
    _, p, inp, exp = G.case(name)
    T = lambda a: nt.Tensor(a, dtype=np.float32)
    cfg = rt.RouterConfig(d_model=p["d"], n_experts=p["E"], capacity_factor=p["C"],
                          gate_scale=p.get("gate_scale", 1.0))
    bank = rm.ExpertBank(*(T(inp[k]) for k in ("w1", "w3", "w2", "sw1", "sw3", "sw2")))
    fn = compat.make_moe_forward(ref.backbone)
    out, decs, routing = fn(T(inp["x_mod"]), T(inp["x_norm"]), T(inp["x_mod"]), T(inp["t_emb"]),
                            cfg, bank, T(inp["w_r"]), return_routing=True)
    assert isinstance(out, nt.Tensor) and out.data.dtype == np.float32
    np.testing.assert_array_equal(routing["token_flat"], exp["token_flat"])
    np.testing.assert_array_equal(routing["gates"].data, exp["gates"])
    np.testing.assert_array_equal(routing["logits"].data, exp["logits"])
    assert routing["capacity"] == int(exp["capacity"])
    assert all(isinstance(d, rt.RouterDecision) for d in decs)
    assert rel_fro(out.data, exp["out"]) <= TOL_FP32
    # the reference's exception types cross the boundary
    with pytest.raises(rt.ConfigError):
        fn(T(inp["x_mod"]), T(inp["x_norm"]), T(inp["x_mod"]), T(inp["t_emb"]), cfg, bank,
           T(inp["w_r"][:-1]))


def test_dropin_records_one_tape_node_fp32():
    """Under the reference's Tape the adapter is one node whose pullback is
    nimg_moe_backward: gradients match the reference's own tape (golden)."""
    from paper_2604_12163_b200 import compat
    ref = load_reference()
    nt, rt, rm = ref.tensor, ref.router, ref.moe
    _, p, inp, exp = G.case("bwd_small_fp32")
    names = ("x_norm", "x_mod", "t_emb", "w_r", "w1", "w3", "w2", "sw1", "sw3", "sw2")
    ts = {k: nt.Tensor(inp[k], requires_grad=True, dtype=np.float32) for k in names}
    cfg = rt.RouterConfig(d_model=inp["x_mod"].shape[-1], n_experts=p["E"],
                          capacity_factor=p["C"], gate_scale=p.get("gate_scale", 1.0))
    bank = rm.ExpertBank(ts["w1"], ts["w3"], ts["w2"], ts["sw1"], ts["sw3"], ts["sw2"])
    fn = compat.make_moe_forward(ref.backbone)
    with nt.Tape() as tape:
        out = fn(ts["x_mod"], ts["x_norm"], ts["x_mod"], ts["t_emb"], cfg, bank, ts["w_r"])
        loss = nt.sum(nt.mul(out, nt.Tensor(inp["g_out"], dtype=np.float32)))
    assert sum(n.op == "moe_forward_b200" for n in tape.nodes) == 1
    nt.backward(tape, loss)
    assert rel_fro(out.data, exp["out"]) <= TOL_FP32
    for k in names:
        assert rel_fro(ts[k].grad, exp[f"grad_{k}"]) <= TOL_FP32, k


def test_dropin_f64_layer_vs_reference():
    """The reference's f64 storage mode (tensor.py:39-47) at the layer: the
    stock reference moe_forward vs the adapter on the same f64 Tensors."""
    from paper_2604_12163_b200 import compat
    ref = load_reference()
    nt, rt, rm = ref.tensor, ref.router, ref.moe
    inp = make_layer_inputs(31, 2, 192, 256, 8, 168, layer=5, mode="fp32")
    T = lambda a: nt.Tensor(np.asarray(a, dtype=np.float64), dtype=np.float64)
    cfg = rt.RouterConfig(d_model=256, n_experts=8, capacity_factor=2.0)
    bank = rm.ExpertBank(*(T(inp[k]) for k in ("w1", "w3", "w2", "sw1", "sw3", "sw2")))
    args = (T(inp["x_mod"]), T(inp["x_norm"]), T(inp["x_mod"]), T(inp["t_emb"]), cfg, bank,
            T(inp["w_r"]))
    with nt.no_grad():
        o_ref, d_ref, r_ref = rm.moe_forward(*args, return_routing=True)
    o, d, r = compat.make_moe_forward(ref.backbone)(*args, return_routing=True)
    assert o.data.dtype == np.float64 and r["gates"].data.dtype == np.float64
    np.testing.assert_array_equal(r["token_flat"], r_ref["token_flat"])
    assert rel_fro(r["logits"].data, r_ref["logits"].data) < 1e-14
    assert rel_fro(r["gates"].data, r_ref["gates"].data) < 1e-14
    assert rel_fro(o.data, o_ref.data) < 1e-12
    for a, b in zip(d, d_ref):
        np.testing.assert_array_equal(a.top_indices, b.top_indices)
