"""B200-native (sm_100a) expert-choice MoE layer of Nucleus-Image (arXiv 2604.12163).

Drop-in for the reference's operator API (`nimg.router`, `nimg.moe`):

    from paper_2604_12163_b200 import router, moe
    out = moe.moe_forward(x, x_norm, x_mod, t_emb, cfg, bank, w_r)

All compute runs in libnimg_moe.so (hand-written CUDA for sm_100a, C ABI in
include/nimg_moe.h). Importing the operator modules requires that library.
"""

__version__ = "0.1.0"
