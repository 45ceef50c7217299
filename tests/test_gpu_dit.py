"""The denoising-step stack (dit.MoEDiT) on the GPU against the reference's
own MoEDiT.forward (golden vectors, tests/golden/make_golden.py).

* f64 + oracle MoE double: the PyTorch parts on CUDA, rounding-level parity.
* the product path (CudaBackend: fused MoE block kernels, dense FFN through
  the grouped GEMM) in fp32 and bf16. The reference runs its MoE on f64
  activations (the timestep features promote), ours routes on
  fp32 scores, so selections may differ where two f64 scores round to the
  same fp32 value; the bar is the Frobenius rel-err of the velocity plus a
  >= 99% match of the routed (expert, slot) selections."""

import numpy as np
import pytest
import torch

from oracle.workloads import DIT_PROMPTS, perturb_modulation
from paper_2604_12163_b200 import dit as D
from paper_2604_12163_b200.router import StageId
from tests import golden_cases as G
from tests.dit_oracle_backend import OracleBackend
from tests.gpu_helpers import TOL_BF16

pytestmark = pytest.mark.gpu

TOL_STACK_FP32 = 1e-4


def _run(name, compute_dtype, backend):
    _, p, inp, exp = G.case(name)
    cfg = D.ModelConfig(**p["model"])
    params = perturb_modulation(D.init_parameters(cfg), p["mod_seed"])
    m = D.MoEDiT(cfg, params, compute_dtype=compute_dtype, backend=backend)
    ctx = m.precompute_text_kv(list(DIT_PROMPTS[:p["B"]]))
    vel, aux = m.forward(inp["z"], inp["t"], ctx, StageId[p["stage"]])
    torch.cuda.synchronize()
    return vel.double().cpu().numpy(), aux, exp


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("name", G.names("dit"))
def test_stack_f64_on_cuda(name):
    v, aux, exp = _run(name, torch.float64, OracleBackend())
    assert _rel(v, exp["vel"]) < 1e-12
    for layer, decs in aux["decisions"]:
        np.testing.assert_array_equal(np.stack([d.top_indices for d in decs]), exp[f"top_{layer}"])


def _selection_match(aux, exp):
    hit = tot = 0
    for layer, decs in aux["decisions"]:
        ours = np.stack([d.top_indices for d in decs])
        ref = exp[f"top_{layer}"]
        for b in range(ours.shape[0]):
            for e in range(ours.shape[1]):
                hit += len(set(ours[b, e].tolist()) & set(ref[b, e].tolist()))
                tot += ours.shape[2]
    return hit / tot


@pytest.mark.parametrize("name", G.names("dit"))
def test_stack_cuda_fp32(name):
    v, aux, exp = _run(name, torch.float32, D.CudaBackend(torch.float32))
    assert _selection_match(aux, exp) >= 0.99
    assert _rel(v, exp["vel"]) < TOL_STACK_FP32


@pytest.mark.parametrize("name", G.names("dit"))
def test_stack_cuda_bf16(name):
    v, aux, exp = _run(name, torch.bfloat16, D.CudaBackend(torch.bfloat16))
    assert np.isfinite(v).all()
    assert _rel(v, exp["vel"]) < TOL_BF16
