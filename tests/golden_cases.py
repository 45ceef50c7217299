"""Load committed golden fixtures (made by tests/golden/make_golden.py from the
real reference) and regenerate their seeded inputs."""

from __future__ import annotations

import json
import os

import numpy as np

from oracle.workloads import (digest, make_block_inputs, make_bwd_inputs, make_latent, make_layer_inputs,
                              make_router_inputs)

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def manifest() -> dict:
    with open(os.path.join(GOLDEN_DIR, "manifest.json")) as f:
        return json.load(f)


def case(name: str):
    """Returns (kind, params, inputs, expected) for a golden case."""
    m = manifest()[name]
    kind, p = m["kind"], m["params"]
    if kind == "dit":
        z, t = make_latent(p["seed"], p["B"], p["model"]["latent_channels"], p["H"], p["W"])
        inp = {"z": z, "t": t}
    elif kind == "block":
        inp = make_block_inputs(p["seed"], p["B"], p["S"], p["d"], p["E"], p["h"], mode=p["mode"])
    elif kind == "moe_bwd":
        inp = make_bwd_inputs(p)
    elif kind == "moe":
        inp = make_layer_inputs(p["seed"], p["B"], p["S"], p["d"], p["E"], p["h"],
                                layer=p.get("layer", 3), mode=p["mode"])
    else:
        inp = make_router_inputs(p["seed"], p["B"], p["S"], p["d"], p["E"],
                                 layer=p.get("layer", 3), mode=p["mode"])
    with np.load(os.path.join(GOLDEN_DIR, f"{name}.npz")) as z:
        exp = {k: z[k] for k in z.files}
    assert str(exp["input_digest"]) == digest(inp), f"input generator drifted for {name}"
    return kind, p, inp, exp


def names(kind: str | None = None):
    return [n for n, m in manifest().items() if kind is None or m["kind"] == kind]
