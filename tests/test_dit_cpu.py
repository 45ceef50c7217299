"""The denoising-step stack (paper_2604_12163_b200.dit) on
CPU: model init, text encoder and the PyTorch parts of MoEDiT.forward,
pinned against golden vectors written by the reference's own MoEDiT
(tests/golden/make_golden.py, backbone.py:447-635).

The MoE blocks and dense FFNs run through the oracle test double in f64
(tests/dit_oracle_backend.py); the CUDA path is covered by test_gpu_dit.py."""

import numpy as np
import pytest
import torch

from oracle.workloads import DIT_PROMPTS, digest, perturb_modulation
from paper_2604_12163_b200 import dit as D
from paper_2604_12163_b200.errors import ConfigError, DomainError, ShapeError
from paper_2604_12163_b200.router import StageId
from tests import golden_cases as G
from tests.dit_oracle_backend import OracleBackend
from tests.refimport import load_reference, reference_available


def _model(p, device, compute_dtype, backend):
    cfg = D.ModelConfig(**p["model"])
    params = perturb_modulation(D.init_parameters(cfg), p["mod_seed"])
    return cfg, params, D.MoEDiT(cfg, params, compute_dtype=compute_dtype, backend=backend,
                                 device=device)


@pytest.mark.parametrize("name", G.names("dit"))
def test_init_matches_reference_parameters(name):
    """Same names, shapes, dtypes and values as the reference model for the
    same seed (backbone.py:391-465 draw order), after the fixture's
    modulation perturbation."""
    _, p, _, exp = G.case(name)
    params = perturb_modulation(D.init_parameters(D.ModelConfig(**p["model"])), p["mod_seed"])
    assert digest(params) == str(exp["param_digest"])


@pytest.mark.parametrize("name", G.names("dit"))
def test_stack_f64_matches_reference(name):
    """MoEDiT.forward with the MoE stage in f64 (oracle double): the PyTorch
    embedding / modulation / attention / RoPE / text-KV parts reproduce the
    reference's float64 forward to rounding level."""
    _, p, inp, exp = G.case(name)
    cfg, _, m = _model(p, torch.device("cpu"), torch.float64, OracleBackend())
    ctx = m.precompute_text_kv(list(DIT_PROMPTS[:p["B"]]))
    vel, aux = m.forward(inp["z"], inp["t"], ctx, StageId[p["stage"]])
    v = vel.numpy()
    ref = exp["vel"]
    rel = np.linalg.norm(v - ref) / np.linalg.norm(ref)
    assert rel < 1e-12, rel
    for layer, decs in aux["decisions"]:
        np.testing.assert_array_equal(np.stack([d.top_indices for d in decs]), exp[f"top_{layer}"])
    for j, (layer, _) in enumerate(aux["decisions"]):
        np.testing.assert_allclose(aux["router_logits"][j], exp[f"logits_{layer}"], rtol=1e-10,
                                   atol=1e-13)


def test_blocks_are_identities_at_init():
    """Zero-initialised modulation gates every branch off (backbone.py:1-6):
    the stack reduces to patch embed -> LN -> final projection."""
    cfg = D.ModelConfig(n_layers=4, d_model=32, n_q_heads=4, n_kv_heads=2, head_dim=8,
                        n_experts=4, expert_hidden=16, dense_layers=3, latent_channels=4)
    m = D.MoEDiT(cfg, compute_dtype=torch.float64, backend=OracleBackend(),
                 device=torch.device("cpu"))
    z = np.random.default_rng(0).standard_normal((2, 4, 8, 8))
    vel, _ = m.forward(z, 0.5, None, StageId.S256)
    m0 = D.MoEDiT(D.ModelConfig(**{**cfg.__dict__, "n_layers": 0}), compute_dtype=torch.float64,
                  backend=OracleBackend(), device=torch.device("cpu"))
    m0.w["patch_embed.weight"] = m.w["patch_embed.weight"]
    m0.w["final_proj.weight"] = m.w["final_proj.weight"]
    vel0, _ = m0.forward(z, 0.5, None, StageId.S256)
    torch.testing.assert_close(vel, vel0, rtol=0, atol=0)


def test_config_and_domain_errors():
    with pytest.raises(ConfigError):
        D.ModelConfig(n_q_heads=4, n_kv_heads=3)
    with pytest.raises(ConfigError):
        D.ModelConfig(d_model=32, n_q_heads=4, head_dim=6)
    with pytest.raises(ConfigError):
        D.ModelConfig(d_model=24, n_q_heads=4, head_dim=6)
    cfg = D.ModelConfig(n_layers=1, dense_layers=1)
    assert cfg.shared_hidden == cfg.expert_hidden and cfg.dense_hidden == cfg.d_model
    m = D.MoEDiT(cfg, compute_dtype=torch.float64, backend=OracleBackend(),
                 device=torch.device("cpu"))
    with pytest.raises(DomainError):
        m.forward(np.zeros((1, 4, 4, 4)), 1.5, None, StageId.S256)
    with pytest.raises(ShapeError):
        m.forward(np.zeros((1, 4, 5, 4)), 0.5, None, StageId.S256)


def test_capacity_factor_schedule_per_layer():
    """backbone.py:540-546 on the Nucleus-Image layer stack (S1024: layers
    3-4 at C=4, 5-31 at C=2; override wins)."""
    cfg = D.ModelConfig(n_layers=32, d_model=32, n_q_heads=4, head_dim=8, dense_layers=3)
    m = D.MoEDiT.__new__(D.MoEDiT)
    m.cfg = cfg
    assert [m.capacity_factor_for(i, StageId.S1024) for i in (3, 4, 5, 31)] == [4.0, 4.0, 2.0, 2.0]
    assert m.capacity_factor_for(7, StageId.S256) == 8.0
    m.cfg = D.ModelConfig(n_layers=4, d_model=32, n_q_heads=4, head_dim=8, capacity_override=1.5)
    assert m.capacity_factor_for(3, StageId.S1024) == 1.5


@pytest.mark.skipif(not reference_available(), reason="reference tree not mounted")
def test_text_encoder_matches_reference():
    ref = load_reference()
    import importlib
    bb = importlib.import_module("nimg_ref.backbone")
    for prompt in DIT_PROMPTS + ("", "x"):
        np.testing.assert_array_equal(D.encode_prompt(prompt, 48), bb.encode_prompt(prompt, 48))
    assert ref is not None
