"""The GEMM epilogues store each thread's 32-byte row segment with one 256-bit
store when the address is 32-B aligned and with two 16-B stores otherwise
(common.cuh st_global_32). An output buffer that is only 16-B aligned (what
the C ABI requires) must give the same bits as an aligned one."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ffn(stages, x, off, ex, w1, w3, w2, xs, sw1, sw3, sw2, yr, ys):
    return stages.expert_ffn(x, off, ex, w1, w3, w2, xs, sw1, sw3, sw2, y_routed=yr, y_shared=ys)


def _view16(n, d, dt, dev):
    """(n, d) view whose data pointer is 16 B past a 32-B boundary."""
    es = torch.empty((), dtype=dt).element_size()
    buf = torch.empty(n * d + 32 // es, dtype=dt, device=dev)
    base = buf.data_ptr()
    skip = ((16 - base % 32) % 32) // es
    v = buf[skip:skip + n * d].view(n, d)
    assert v.data_ptr() % 32 == 16
    return v


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float32])
def test_misaligned_expert_outputs_bitwise(dt):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_12163_b200.stages import CudaStages
    st = CudaStages()
    g = torch.Generator(device="cuda").manual_seed(5)
    dev = "cuda"
    E, rows_e, d, h, T = 4, 256, 256, 128, 512
    rn = lambda *s, std=1.0: (torch.randn(*s, generator=g, device=dev) * std).to(dt)
    x, xs = rn(E * rows_e, d), rn(T, d)
    w1, w3, w2 = rn(E, h, d, std=0.05), rn(E, h, d, std=0.05), rn(E, d, h, std=0.05)
    sw1, sw3, sw2 = rn(h, d, std=0.05), rn(h, d, std=0.05), rn(d, h, std=0.05)
    off = np.arange(E + 1, dtype=np.int64) * rows_e
    ex = np.arange(E, dtype=np.int32)
    ydt = st.ffn_y_dtype(dt, d, h, h)
    ya, ysa = _ffn(st, x, off, ex, w1, w3, w2, xs, sw1, sw3, sw2, None, None)
    yr, ys = _view16(E * rows_e, d, ydt, dev), _view16(T, d, ydt, dev)
    _ffn(st, x, off, ex, w1, w3, w2, xs, sw1, sw3, sw2, yr, ys)
    torch.cuda.synchronize()
    assert torch.equal(ya, yr) and torch.equal(ysa, ys)
