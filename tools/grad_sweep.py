"""Randomised sweep of the layer's training path (reference-style Tape / backward
over moe_forward, as in tests/test_gpu_backward.py) against the oracle's
pullbacks (oracle.moe_backward): every gradient -- x_norm, x_mod, t_emb, W_r,
routed and shared expert weights -- within the north-star tolerance
(Frobenius rel. error 2e-2 bf16, 1e-4 fp32). One line per case, a summary,
exit code 1 on any failure.

usage: python tools/grad_sweep.py [N] [seed]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import nimg_oracle as O  # noqa: E402
from oracle.workloads import bf16_round, make_layer_inputs  # noqa: E402
from tests.gpu_helpers import TOL_BF16, TOL_FP32, np_of, rel_fro, to_gpu  # noqa: E402

GRADS = ("x_norm", "x_mod", "t_emb", "w_r", "w1", "w3", "w2", "sw1", "sw3", "sw2")


def draw(rng):
    mode = "bf16" if rng.random() < 0.75 else "fp32"
    d = int(rng.choice([128, 256, 384, 512]))
    E = int(rng.choice([4, 8, 16, 64]))
    h = int(rng.choice([64, 128, 192, 256, 80]))
    hs = int(rng.choice([h, 64, 128]))
    B = int(rng.integers(1, 4))
    S = int(rng.choice([32, 64, 100, 256]))
    C = float(rng.choice([1.0, 2.0, 4.0]))
    return dict(mode=mode, d=d, E=E, h=h, hs=hs, B=B, S=S, C=C)


def run(c, seed):
    from paper_2604_12163_b200 import moe as M
    from paper_2604_12163_b200 import router as R
    from paper_2604_12163_b200 import tensor as nt
    inp = make_layer_inputs(seed, c["B"], c["S"], c["d"], c["E"], c["h"], h_shared=c["hs"], mode=c["mode"])
    g_out = bf16_round(np.random.default_rng(seed + 1).standard_normal((c["B"], c["S"], c["d"])).astype(np.float32))
    g = to_gpu(inp, c["mode"])
    for k in GRADS:
        g[k].requires_grad_(True)
    cfg = R.RouterConfig(d_model=c["d"], n_experts=c["E"], capacity_factor=c["C"])
    bank = M.ExpertBank(g["w1"], g["w3"], g["w2"], g["sw1"], g["sw3"], g["sw2"])
    act = torch.bfloat16 if c["mode"] == "bf16" else torch.float32
    gt = torch.from_numpy(g_out).cuda().to(act)
    with nt.Tape() as tape:
        out = M.moe_forward(g["x_mod"], g["x_norm"], g["x_mod"], g["t_emb"], cfg, bank, g["w_r"])
        loss = (out.float() * gt.float()).sum()
    nt.backward(tape, loss)
    torch.cuda.synchronize()
    ref = O.moe_backward(*(inp[k] for k in GRADS), g_out, capacity_factor=c["C"])
    errs = {k: rel_fro(np_of(g[k].grad), ref[k]) for k in GRADS}
    tol = TOL_BF16 if c["mode"] == "bf16" else TOL_FP32
    return errs, tol


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 11
    rng = np.random.default_rng(seed)
    fails, worst = 0, {"bf16": 0.0, "fp32": 0.0}
    t0 = time.time()
    for i in range(n):
        c = draw(rng)
        errs, tol = run(c, seed + 7 * i)
        w = max(errs.values())
        ok = w <= tol
        fails += not ok
        worst[c["mode"]] = max(worst[c["mode"]], w)
        bad = {k: f"{v:.2e}" for k, v in errs.items() if v > tol}
        print(f"{i:3d} {'ok  ' if ok else 'FAIL'} {c} worst grad rel-err {w:.3e} (tol {tol:g}) {bad or ''}",
              flush=True)
    print(f"summary: {n - fails}/{n} passed, worst grad rel-err bf16 {worst['bf16']:.3e} "
          f"fp32 {worst['fp32']:.3e}, {time.time() - t0:.0f} s")
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
