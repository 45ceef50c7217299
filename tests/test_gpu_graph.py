"""CUDA-graph replay of the whole layer (moe.MoEPlan.capture): the C ABI is
stream-ordered with no host sync or allocation, so one captured forward --
INT8 router, its f64 fix-up, selection, gates, GEMM1 with the background
gather (device-side flags re-armed by gate_norm on every replay), GEMM2,
combine -- must replay bit-identically to eager calls on new inputs."""

import numpy as np
import pytest
import torch

from oracle.workloads import make_layer_inputs
from tests.gpu_helpers import bank_of, to_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_12163_b200 import _lib as L
    return L


@pytest.mark.parametrize("B,S,d,E,h,Cf", [(4, 512, 1024, 64, 448, 4.0), (2, 256, 256, 8, 128, 2.0)])
def test_graph_replay_matches_eager(B, S, d, E, h, Cf):
    from paper_2604_12163_b200 import moe as M
    from paper_2604_12163_b200 import router as R
    g = to_gpu(make_layer_inputs(31, B, S, d, E, h, mode="bf16"), "bf16")
    cfg = R.RouterConfig(d_model=d, n_experts=E, capacity_factor=Cf)
    plan = M.MoEPlan(cfg, bank_of(g), B, S)
    static = {k: g[k].clone() for k in ("x_norm", "x_mod", "t_emb", "w_r")}
    graph = plan.capture(static["x_norm"], static["x_mod"], static["t_emb"], static["w_r"])
    for seed in (32, 33, 34):
        g2 = to_gpu(make_layer_inputs(seed, B, S, d, E, h, mode="bf16"), "bf16")
        for k in static:
            static[k].copy_(g2[k] if k != "w_r" else g[k])
        graph.replay()
        torch.cuda.synchronize()
        got = plan.out.clone()
        tok = plan.r["token_flat"].clone()
        ref = M.moe_forward(static["x_mod"], static["x_norm"], static["x_mod"], static["t_emb"], cfg,
                            bank_of(g), static["w_r"])
        _, _, routing = M.moe_forward(static["x_mod"], static["x_norm"], static["x_mod"],
                                      static["t_emb"], cfg, bank_of(g), static["w_r"],
                                      return_routing=True)
        torch.cuda.synchronize()
        assert torch.equal(got, ref)
        np.testing.assert_array_equal(tok.cpu().numpy(), routing["token_flat"].cpu().numpy())
