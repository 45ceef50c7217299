"""Which SDPA path is fast on B200 for the stack's joint attention shape."""
import torch, torch.nn.functional as F
from torch.nn.attention import sdpa_kernel, SDPBackend
B, H, Hkv, S, St, D = 4, 16, 4, 4096, 256, 128
dev = "cuda"
q = torch.randn(B, H, S, D, device=dev, dtype=torch.bfloat16)
k = torch.randn(B, Hkv, S + St, D, device=dev, dtype=torch.bfloat16)
v = torch.randn_like(k)
mask = torch.ones(B, 1, 1, S + St, dtype=torch.bool, device=dev)
mask[1, ..., S + 100:] = False
kr, vr = k.repeat_interleave(H // Hkv, 1), v.repeat_interleave(H // Hkv, 1)
def t(name, f):
    try:
        for _ in range(3): f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): f()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        fl = 4 * B * H * S * (S + St) * D
        print(f"{name:40s} {ms:8.3f} ms  {fl / ms / 1e9:7.0f} TF/s")
    except Exception as ex:
        print(f"{name:40s} failed: {type(ex).__name__}: {str(ex)[:100]}")
t("default repeat nomask", lambda: F.scaled_dot_product_attention(q, kr, vr))
t("default repeat boolmask", lambda: F.scaled_dot_product_attention(q, kr, vr, attn_mask=mask))
t("default gqa nomask", lambda: F.scaled_dot_product_attention(q, k, v, enable_gqa=True))
t("default gqa boolmask", lambda: F.scaled_dot_product_attention(q, k, v, attn_mask=mask, enable_gqa=True))
for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION, SDPBackend.EFFICIENT_ATTENTION, SDPBackend.MATH):
    with sdpa_kernel([be]):
        t(f"{be.name} repeat nomask", lambda: F.scaled_dot_product_attention(q, kr, vr))
        t(f"{be.name} repeat boolmask", lambda: F.scaled_dot_product_attention(q, kr, vr, attn_mask=mask))
        t(f"{be.name} gqa nomask", lambda: F.scaled_dot_product_attention(q, k, v, enable_gqa=True))
try:
    import flash_attn
    from flash_attn import flash_attn_func
    qq, kk, vv = q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2)
    t("flash_attn pkg gqa", lambda: flash_attn_func(qq, kk, vv))
except Exception as ex:
    print("flash_attn import failed", ex)
