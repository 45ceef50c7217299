"""Debug: INT8 router logits WITHOUT the f64 fix-up vs the oracle (which
tokens would be flagged, and how far the raw int8-path logits are off)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import nimg_oracle as O
from oracle.workloads import make_router_inputs
from paper_2604_12163_b200 import router as R
B, S, d, E = 2, 1024, int(os.environ.get("D", 2048)), 64
inp = make_router_inputs(2, B, S, d, E, layer=17, mode="bf16")
ref = O.route_full(inp["x_norm"], inp["t_emb"], inp["w_r"], n_experts=E, capacity_factor=4.0)
cfg = R.RouterConfig(d_model=d, n_experts=E, capacity_factor=4.0)
os.environ["NIMG_ROUTER_I8_NOFIX"] = "1"
_, rt = R.route_full(torch.from_numpy(inp["x_norm"]).cuda().to(torch.bfloat16),
                     torch.from_numpy(inp["t_emb"]).cuda(), torch.from_numpy(inp["w_r"]).cuda(), cfg)
lg = rt["logits"].float().cpu().numpy()
rl = ref["logits"]
bad = lg != rl
print("mismatch frac", bad.mean(), "rows", bad.any(-1).sum(), "of", B * S)
idx = np.argwhere(bad)[:10]
for i in idx:
    print(tuple(i), lg[tuple(i)], rl[tuple(i)])
# x-half only check: subtract t-bias
tb = (inp["t_emb"].astype(np.float64) @ inp["w_r"][d:].astype(np.float64))
xh = inp["x_norm"].astype(np.float64) @ inp["w_r"][:d].astype(np.float64)
ratio = (lg.astype(np.float64) - tb[:, None, :]) / xh
print("ratio (gpu - tb)/x-half: median", np.median(ratio), "p1", np.percentile(ratio, 1), "p99", np.percentile(ratio, 99))
print("corr", np.corrcoef((lg - tb[:, None, :]).ravel(), xh.ravel())[0, 1])
