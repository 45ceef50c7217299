"""Time the routing stage (nimg_route: prep + scores + fix-up + select + gates)
at cfg2 through the C ABI, for A/B library builds (NIMG_LIB_PATH)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from oracle.workloads import make_router_inputs  # noqa: E402
from paper_2604_12163_b200 import _lib  # noqa: E402
from paper_2604_12163_b200 import router as R  # noqa: E402
from paper_2604_12163_b200._tensors import ptr, stream_handle, workspace  # noqa: E402

B, S, d, E = int(os.environ.get("B", 16)), int(os.environ.get("S", 1024)), 2048, 64
C_ = float(os.environ.get("C", 4.0))
inp = make_router_inputs(2, B, S, d, E, layer=17, mode="bf16")
x = torch.from_numpy(inp["x_norm"]).cuda().to(torch.bfloat16)
t = torch.from_numpy(inp["t_emb"]).cuda()
w = torch.from_numpy(inp["w_r"]).cuda()
cfg = R.RouterConfig(d_model=d, n_experts=E, capacity_factor=C_)
cap = R.capacity_for(S, E, C_)
desc = R.make_desc(B, S, d, E, cap, 1, 1, cfg, torch.bfloat16)
n = C.c_size_t()
_lib.check(_lib.lib.nimg_route_workspace_bytes(C.byref(desc), C.byref(n)))
ws = workspace(n.value)
r = R.alloc_route_out(B, S, E, cap, x.device)
ro = R.route_struct(r)
evs = [torch.cuda.Event(enable_timing=True) for _ in range(8)]


def once(prof=False):
    if prof:
        arr = (C.c_void_p * 7)(*[e.cuda_event for e in evs[:7]])
        _lib.check(_lib.lib.nimg_profile_events(arr, 7))
    _lib.check(_lib.lib.nimg_route(C.byref(desc), ptr(x), ptr(t), ptr(w), C.byref(ro), ptr(ws),
                                   ws.numel(), stream_handle()))
    if prof:
        _lib.check(_lib.lib.nimg_profile_events(None, 0))


for e in evs:
    e.record()
for _ in range(5):
    once()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
N = 50
a.record()
for _ in range(N):
    once()
b.record()
torch.cuda.synchronize()
tot = a.elapsed_time(b) / N * 1e3
sc = 0.0
for _ in range(10):
    evs[0].record()
    once(prof=True)
    torch.cuda.synchronize()
    sc += evs[0].elapsed_time(evs[6]) * 1e3 / 10
print(f"{os.path.basename(_lib.LIB_PATH)}: route {tot:.1f} us (scores incl. prep ~{sc:.1f} us)")
