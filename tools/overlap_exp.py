"""Experiment: can the FP64 (DMMA) router overlap the shared-expert tcgen05
GEMMs? Times route alone, shared FFN alone, and both on two streams."""
import sys, os, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import CFG2, make_inputs
from paper_2604_12163_b200 import router as R
from paper_2604_12163_b200.stages import CudaStages

c = CFG2
inp = make_inputs(c, torch.device("cuda"))
st = CudaStages()
cfg = R.RouterConfig(d_model=c["d"], n_experts=c["E"], capacity_factor=c["C"])
cap = R.capacity_for(c["S"], c["E"], c["C"])
T = c["B"] * c["S"]
xm = inp["x_mod"].view(T, -1)
route = lambda: st.route(inp["x_norm"], inp["t_emb"], inp["w_r"], cfg, cap)
shared = lambda: st.expert_ffn(None, None, None, None, None, None, xm, inp["sw1"], inp["sw3"], inp["sw2"])
s2 = torch.cuda.Stream()

def timeit(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n

def both(order):
    def f():
        s2.wait_stream(torch.cuda.current_stream())
        if order == "route_first":
            route()
            with torch.cuda.stream(s2): shared()
        else:
            with torch.cuda.stream(s2): shared()
            route()
        torch.cuda.current_stream().wait_stream(s2)
    return f

print("stages", os.environ.get("NIMG_GEMM_STAGES", "6"))
print("route alone  %.3f ms" % timeit(route))
print("shared alone %.3f ms" % timeit(shared))
print("sequential   %.3f ms" % timeit(lambda: (route(), shared())))
print("concurrent route-first  %.3f ms" % timeit(both("route_first")))
print("concurrent shared-first %.3f ms" % timeit(both("shared_first")))
