"""Probe: time the router stage alone at cfg2 (B=16, S=1024, d=2048, E=64, bf16)
for the INT8 and FP64 routers; under ncu it gives the per-kernel split."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle.workloads import make_router_inputs
from paper_2604_12163_b200 import router as R

B, S, d, E = int(os.environ.get("B", 16)), int(os.environ.get("S", 1024)), 2048, 64
inp = make_router_inputs(2, B, S, d, E, layer=17, mode="bf16")
x = torch.from_numpy(inp["x_norm"]).cuda().to(torch.bfloat16)
t = torch.from_numpy(inp["t_emb"]).cuda()
w = torch.from_numpy(inp["w_r"]).cuda()
cfg = R.RouterConfig(d_model=d, n_experts=E, capacity_factor=4.0)
n = int(os.environ.get("N", 20))
for router in ("i8", "dmma"):
    os.environ["NIMG_ROUTER"] = router
    for _ in range(3):
        R.route_full(x, t, w, cfg)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        R.route_full(x, t, w, cfg)
    b.record(); torch.cuda.synchronize()
    print(router, "route_full %.1f us" % (a.elapsed_time(b) / n * 1e3))
