"""Generate golden vectors from the REAL reference (run in the build container).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Imports /root/reference/pkg/src/nimg under the alias ``nimg_ref`` (it cannot
travel to the GPU box) and runs its own public API -- router.route_full and
moe.moe_forward (router.py:104-162, moe.py:138-164) -- on the seeded inputs
of ``oracle.workloads``. Inputs are NOT stored (they are regenerated from the
seed, and their sha256 is stored to detect drift); outputs are stored as
compressed .npz fixtures in this directory.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.workloads import (DIT_PROMPTS, digest, make_block_inputs,  # noqa: E402
                              make_bwd_inputs,
                              make_latent, make_layer_inputs, make_router_inputs,
                              perturb_modulation)
from tests.refimport import load_reference  # noqa: E402

# name -> (kind, params). kind "moe" = full layer, "route" = router only.
CASES = {
    # d=256, E=8, h=168, C=2, S=256, B=2, fp32.
    "cfg1_fp32": ("moe", dict(seed=0, B=2, S=256, d=256, E=8, h=168, C=2.0, mode="fp32")),
    "cfg1_bf16": ("moe", dict(seed=1, B=2, S=256, d=256, E=8, h=168, C=2.0, mode="bf16")),
    # non-multiple-of-tile shapes and gate_scale != 1
    "ragged_fp32": ("moe", dict(seed=2, B=3, S=37, d=24, E=5, h=20, C=1.7, mode="fp32",
                                gate_scale=1.7)),
    "mid_bf16": ("moe", dict(seed=3, B=2, S=192, d=512, E=16, h=336, C=4.0, mode="bf16",
                             layer=7)),
    # full-width router (d=2048, E=64) on a cfg2 sub-batch: the f64-grade
    # router accumulation is what must reproduce the fp32 logits bit-exactly.
    "cfg2_route_fp32": ("route", dict(seed=4, B=2, S=1024, d=2048, E=64, C=4.0, mode="fp32",
                                      layer=17)),
    "cfg2_route_bf16": ("route", dict(seed=5, B=1, S=1024, d=2048, E=64, C=4.0, mode="bf16",
                                      layer=17)),
    # 1024px column length, C=2 (cap 128), one sample
    "s4096_route_bf16": ("route", dict(seed=6, B=1, S=4096, d=2048, E=64, C=2.0, mode="bf16",
                                       layer=17)),
    # the backbone's MoE branch around the layer (backbone.py:583-606), fp32
    "block_fp32": ("block", dict(seed=7, B=2, S=128, d=256, E=8, h=112, C=2.0, mode="fp32",
                                 layer=5)),
    "block_ragged_fp32": ("block", dict(seed=8, B=2, S=40, d=24, E=4, h=20, C=1.5, mode="fp32",
                                        layer=3)),
    # the denoising-step stack (MoEDiT.forward, backbone.py:548-619), SURVEY 8(d)
    # cfg1 block variant: 3 dense + 1 MoE layer, d=256, GQA 4:1, text context
    "dit_cfg1": ("dit", dict(seed=9, B=2, H=32, W=32, stage="S256", mod_seed=11,
                             model=dict(n_layers=4, d_model=256, n_q_heads=4, n_kv_heads=1,
                                        head_dim=64, n_experts=8, expert_hidden=168,
                                        dense_layers=3, latent_channels=16, patch=2,
                                        capacity_override=2.0, dtype="float32", seed=0))),
    # 2 MoE layers on the stage schedule (S256: C=8), GQA 2:1, ragged prompts
    "dit_small": ("dit", dict(seed=10, B=3, H=16, W=16, stage="S256", mod_seed=12,
                              model=dict(n_layers=5, d_model=128, n_q_heads=4, n_kv_heads=2,
                                         head_dim=32, n_experts=4, expert_hidden=64,
                                         dense_layers=3, latent_channels=4, patch=2,
                                         dtype="float32", seed=3))),
    # backward of the layer: reference tape gradients of
    # sum(moe_forward(...) * g_out) for a seeded upstream gradient g_out
    "bwd_small_fp32": ("moe_bwd", dict(seed=20, B=2, S=64, d=64, E=4, h=64, C=2.0, mode="fp32")),
    "bwd_ragged_fp32": ("moe_bwd", dict(seed=21, B=3, S=37, d=24, E=5, h=20, C=1.7, mode="fp32",
                                        gate_scale=1.7)),
    "bwd_tc_bf16": ("moe_bwd", dict(seed=22, B=2, S=128, d=128, E=4, h=64, C=2.0, mode="bf16")),
}

GRAD_NAMES = ("x_norm", "x_mod", "t_emb", "w_r", "w1", "w3", "w2", "sw1", "sw3", "sw2")


def inputs_for(kind, p):
    if kind == "dit":
        z, t = dit_inputs(p)
        return {"z": z, "t": t}
    if kind == "block":
        return make_block_inputs(p["seed"], p["B"], p["S"], p["d"], p["E"], p["h"], mode=p["mode"])
    if kind == "moe_bwd":
        return make_bwd_inputs(p)
    if kind == "moe":
        return make_layer_inputs(p["seed"], p["B"], p["S"], p["d"], p["E"], p["h"],
                                 layer=p.get("layer", 3), mode=p["mode"])
    return make_router_inputs(p["seed"], p["B"], p["S"], p["d"], p["E"],
                              layer=p.get("layer", 3), mode=p["mode"])


def run_reference_block(ref, p, inp):
    """backbone.py:583-606 composed from the reference's own functions."""
    import math
    import importlib
    bb = importlib.import_module("nimg_ref.backbone")
    nt = ref.tensor
    T, f32 = nt.Tensor, np.float32
    B, S, d = inp["x"].shape
    cfg = ref.router.RouterConfig(d_model=d, n_experts=p["E"], capacity_factor=p["C"])
    bank = ref.moe.ExpertBank(*(T(inp[k], dtype=f32) for k in ("w1", "w3", "w2", "sw1", "sw3", "sw2")))
    x, r_attn = T(inp["x"], dtype=f32), T(inp["r_attn"], dtype=f32)
    sa_gate, ff_scale, ff_gate = (T(inp[k], dtype=f32) for k in ("sa_gate", "ff_scale", "ff_gate"))
    t_vec, w_r = T(inp["t_vec"], dtype=f32), T(inp["w_r"], dtype=f32)
    with nt.no_grad():
        h = bb.fused_gated_residual(x, sa_gate, r_attn)
        scale = 1.0 / math.sqrt(p["layer"] + 1)
        x_norm = nt.mul(nt.rmsnorm(h), scale)
        x_mod = nt.mul(x_norm, nt.add(nt.broadcast_to(nt.reshape(ff_scale, (B, 1, -1)), h.shape), 1.0))
        moe_out, decisions, routing = ref.moe.moe_forward(h, x_norm, x_mod, t_vec, cfg, bank, w_r,
                                                          return_routing=True)
        out = bb.fused_gated_residual(h, ff_gate, moe_out)
    return {"out": out.data, "h": h.data, "x_norm": x_norm.data, "x_mod": x_mod.data,
            "moe": moe_out.data, "logits": routing["logits"].data,
            "token_flat": np.asarray(routing["token_flat"], dtype=np.int64),
            "gates": routing["gates"].data, "capacity": np.int64(routing["capacity"])}


def dit_inputs(p):
    return make_latent(p["seed"], p["B"], p["model"]["latent_channels"], p["H"], p["W"])


def run_reference_dit(p):
    """MoEDiT.forward (backbone.py:548-619) of the reference, modulation
    perturbed so the blocks are not identities."""
    import importlib
    bb = importlib.import_module("nimg_ref.backbone")
    rt = importlib.import_module("nimg_ref.router")
    nt = importlib.import_module("nimg_ref.tensor")
    cfg = bb.ModelConfig(**p["model"])
    model = bb.MoEDiT(cfg)
    params = {k: v.data for k, v in model.named_parameters().items()}
    perturb_modulation(params, p["mod_seed"])
    z, t = dit_inputs(p)
    ctx = model.precompute_text_kv(list(DIT_PROMPTS[:p["B"]]))
    with nt.no_grad():
        vel, aux = model.forward(nt.Tensor(z, dtype=np.float32), t, ctx, rt.StageId[p["stage"]])
    res = {"vel": vel.data, "param_digest": np.array(digest(params))}
    for j, (layer, decs) in enumerate(aux["decisions"]):
        res[f"logits_{layer}"] = aux["router_logits"][j].data
        res[f"top_{layer}"] = np.stack([dd.top_indices for dd in decs])
    return res


def run_reference_bwd(ref, p, inp):
    """Reference Tape + backward (tensor.py:590-628) through moe_forward."""
    nt = ref.tensor
    T, f32 = nt.Tensor, np.float32
    B, S, d = inp["x_mod"].shape
    ts = {k: T(inp[k], requires_grad=True, dtype=f32) for k in GRAD_NAMES}
    cfg = ref.router.RouterConfig(d_model=d, n_experts=p["E"], capacity_factor=p["C"],
                                  gate_scale=p.get("gate_scale", 1.0))
    bank = ref.moe.ExpertBank(ts["w1"], ts["w3"], ts["w2"], ts["sw1"], ts["sw3"], ts["sw2"])
    with nt.Tape() as tape:
        out = ref.moe.moe_forward(ts["x_mod"], ts["x_norm"], ts["x_mod"], ts["t_emb"], cfg, bank,
                                  ts["w_r"])
        loss = nt.sum(nt.mul(out, T(inp["g_out"], dtype=f32)))
    nt.backward(tape, loss)
    res = {f"grad_{k}": ts[k].grad for k in GRAD_NAMES}
    res["out"] = out.data
    return res


def run_reference(ref, kind, p, inp):
    if kind == "moe_bwd":
        return run_reference_bwd(ref, p, inp)
    if kind == "dit":
        return run_reference_dit(p)
    if kind == "block":
        return run_reference_block(ref, p, inp)
    T = ref.tensor.Tensor
    f32 = np.float32
    cfg = ref.router.RouterConfig(d_model=p["d"], n_experts=p["E"], capacity_factor=p["C"],
                                  gate_scale=p.get("gate_scale", 1.0))
    with ref.tensor.no_grad():
        if kind == "route":
            decisions, routing = ref.router.route_full(
                T(inp["x_norm"], dtype=f32), T(inp["t_emb"], dtype=f32),
                T(inp["w_r"], dtype=f32), cfg)
            out = None
        else:
            bank = ref.moe.ExpertBank(
                w1=T(inp["w1"], dtype=f32), w3=T(inp["w3"], dtype=f32), w2=T(inp["w2"], dtype=f32),
                shared_w1=T(inp["sw1"], dtype=f32), shared_w3=T(inp["sw3"], dtype=f32),
                shared_w2=T(inp["sw2"], dtype=f32))
            xm = T(inp["x_mod"], dtype=f32)
            out, decisions, routing = ref.moe.moe_forward(
                xm, T(inp["x_norm"], dtype=f32), xm, T(inp["t_emb"], dtype=f32), cfg, bank,
                T(inp["w_r"], dtype=f32), return_routing=True)
    res = {
        "logits": routing["logits"].data,
        "token_flat": np.asarray(routing["token_flat"], dtype=np.int64),
        "gates": routing["gates"].data,
        "top": np.stack([d.top_indices for d in decisions]),
        "affinity": np.stack([d.affinity for d in decisions]),
        "capacity": np.int64(routing["capacity"]),
    }
    if out is not None:
        res["out"] = out.data
    return res


def main():
    ref = load_reference()
    only = set(sys.argv[1:])
    mpath = os.path.join(HERE, "manifest.json")
    manifest = json.load(open(mpath)) if only and os.path.exists(mpath) else {}
    for name, (kind, p) in CASES.items():
        if only and name not in only:
            continue
        inp = inputs_for(kind, p)
        res = run_reference(ref, kind, p, inp)
        res["input_digest"] = np.array(digest(inp))
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **res)
        manifest[name] = {"kind": kind, "params": p, "input_digest": digest(inp)}
        print(name, {k: getattr(v, "shape", None) for k, v in res.items()})
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
