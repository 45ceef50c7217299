"""Two MoE layers in flight at once on two streams (the C ABI takes any
stream). Each persistent grouped GEMM then gets only part of the SMs while the
other holds the rest, so no CTA of GEMM1 may wait on work owned by a CTA that
is not scheduled: the routed-row gather inside GEMM1 claims its 32-row
sub-blocks from a global counter (csrc/grouped_gemm_sm100.cu), so a waiting
producer's own copy warps can always finish the copy. The calls must complete
and give the bits of serial calls."""

import pytest
import torch

from oracle.workloads import make_layer_inputs
from tests.gpu_helpers import bank_of, to_gpu

pytestmark = pytest.mark.gpu


@pytest.mark.timeout(300)
def test_two_layers_concurrently_on_two_streams():
    from paper_2604_12163_b200 import moe as M
    from paper_2604_12163_b200 import router as R
    cases = []
    for seed, (B, S, d, E, h, C) in enumerate([(4, 1024, 1024, 16, 512, 4.0),
                                               (2, 1024, 2048, 64, 1344, 4.0)]):
        g = to_gpu(make_layer_inputs(80 + seed, B, S, d, E, h, layer=9, mode="bf16"), "bf16")
        cfg = R.RouterConfig(d_model=d, n_experts=E, capacity_factor=C)
        plan = M.MoEPlan(cfg, bank_of(g), B, S, torch.bfloat16)
        args = (g["x_norm"], g["x_mod"], g["t_emb"], g["w_r"])
        want = plan.forward(*args).clone()
        cases.append((plan, args, want))
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [[], []]
    for _ in range(12):
        for i, (plan, args, _) in enumerate(cases):
            with torch.cuda.stream(streams[i]):
                outs[i].append(plan.forward(*args).clone())
    torch.cuda.synchronize()
    for i, (_, _, want) in enumerate(cases):
        for o in outs[i]:
            assert torch.equal(o, want)
