"""Kernel-level profile of the stack's PyTorch parts (full width, 4 layers)."""
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
from paper_2604_12163_b200 import dit as D
from paper_2604_12163_b200.router import StageId
dev = torch.device("cuda", 0)
cfg = D.ModelConfig(**{**D.NUCLEUS_IMAGE, "n_layers": 4})
m = D.MoEDiT(cfg, D.random_parameters(cfg, dev), compute_dtype=torch.bfloat16)
B = 4
ctx = m.precompute_text_kv([" ".join(f"tok{i}" for i in range(256))] * B)
z = torch.randn(B, 16, 128, 128, device=dev)
t = np.linspace(0.2, 0.8, B)
f = lambda: m.forward(z, t, ctx, StageId.S1024, return_aux=False)
for _ in range(3): f()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3): f()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30, max_name_column_width=70))
