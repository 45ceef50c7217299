"""A small slice of the randomised sweeps (tools/parity_sweep.py,
tools/grad_sweep.py): seeded random layer shapes across the dispatch paths,
routing bit-exact and outputs / gradients within the north-star tolerance."""

import importlib.util
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
TOOLS = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools")


def _load(name):
    spec = importlib.util.spec_from_file_location(name, os.path.join(TOOLS, name + ".py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_random_layer_shapes_vs_oracle():
    ps = _load("parity_sweep")
    rng = np.random.default_rng(31)
    for i in range(16):
        c = ps.draw(rng)
        same, err, tol = ps.run(c, 31 + i)
        assert same and err <= tol, (c, same, err)


def test_random_training_shapes_vs_oracle():
    gs = _load("grad_sweep")
    rng = np.random.default_rng(37)
    for i in range(8):
        c = gs.draw(rng)
        errs, tol = gs.run(c, 37 + 7 * i)
        assert max(errs.values()) <= tol, (c, errs)
