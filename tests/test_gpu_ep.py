"""Expert parallel on GPUs over NCCL: EP(R) must equal the 1-GPU layer bitwise
(the returned rows land in the 1-GPU expert-major layout and
the combine is deterministic). R = 1 (loopback through the EP code path)
always runs; R = 2 runs when two GPUs are visible."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs(B, S, d, E, h, seed, dev):
    g = torch.Generator(device=dev).manual_seed(seed)
    rn = lambda *s, std=1.0: torch.randn(*s, generator=g, device=dev) * std
    tn = lambda *s, std: torch.clamp(rn(*s, std=std), -2 * std, 2 * std)
    x = rn(B, S, d)
    xn = (x * torch.rsqrt((x * x).mean(-1, keepdim=True) + 1e-6) / 4.0).to(torch.bfloat16)
    xm = (xn.float() * (1 + 0.1 * rn(B, 1, d))).to(torch.bfloat16)
    bf = torch.bfloat16
    return dict(x_norm=xn, x_mod=xm, t_emb=rn(B, d), w_r=tn(2 * d, E, std=0.006),
                w1=tn(E, h, d, std=0.02).to(bf), w3=tn(E, h, d, std=0.02).to(bf),
                w2=tn(E, d, h, std=0.02).to(bf), sw1=tn(h, d, std=0.02).to(bf),
                sw3=tn(h, d, std=0.02).to(bf), sw2=tn(d, h, std=0.02).to(bf))


def _worker(rank, world, port, q, shape, modes=("plain", "nccl", "ce"), oracle=False):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    ngpu = torch.cuda.device_count()
    dev_idx = rank % ngpu
    torch.cuda.set_device(dev_idx)
    if world > ngpu:
        # oversubscribed (several ranks per GPU): NCCL refuses duplicate
        # devices, the copy-engine transport only needs a CPU control plane
        dist.init_process_group("gloo", rank=rank, world_size=world)
    else:
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", dev_idx))
    try:
        from paper_2604_12163_b200 import moe as M
        from paper_2604_12163_b200 import router as R
        from paper_2604_12163_b200.ep import EPContext, ep_moe_forward, shard_bank
        B, S, d, E, h, C = shape
        dev = torch.device("cuda", dev_idx)
        a = _inputs(B, S, d, E, h, 7, dev)
        cfg = R.RouterConfig(d_model=d, n_experts=E, capacity_factor=C)
        bank = M.ExpertBank(a["w1"], a["w3"], a["w2"], a["sw1"], a["sw3"], a["sw2"])
        full = M.moe_forward(a["x_mod"], a["x_norm"], a["x_mod"], a["t_emb"], cfg, bank, a["w_r"])
        bl = B // world
        sl = slice(rank * bl, (rank + 1) * bl)
        local = shard_bank(bank, rank, world)
        res = {}
        for mode in modes:
            ctx = EPContext(overlap=mode != "plain", transport="nccl" if mode == "nccl" else "ce")
            ok = True
            for _ in range(3):   # several steps: exercises the per-step flag epochs
                out = ep_moe_forward(a["x_norm"][sl].contiguous(), a["x_mod"][sl].contiguous(),
                                     a["t_emb"][sl].contiguous(), cfg, local, a["w_r"], ctx)
                torch.cuda.synchronize()
                ok = ok and bool(torch.equal(out, full[sl]))
            res[mode] = ok
        if oracle:
            # this rank's samples of the EP output against the CPU oracle
            # (moe.py:138-164 restated), per sample
            from oracle import nimg_oracle as O
            f = lambda t: t.float().cpu().numpy()
            ref = O.moe_forward(f(a["x_norm"][sl]), f(a["x_mod"][sl]), f(a["t_emb"][sl]), f(a["w_r"]),
                                *(f(a[k]) for k in ("w1", "w3", "w2", "sw1", "sw3", "sw2")),
                                capacity_factor=C)
            o = f(out)
            res["oracle_rel_err"] = [float(np.linalg.norm(o[i] - ref[i]) / np.linalg.norm(ref[i]))
                                     for i in range(o.shape[0])]
        q.put((rank, res))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _run(world, shape, modes=("plain", "nccl", "ce"), oracle=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, shape, modes, oracle))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    import queue as _q
    import time as _t
    deadline = _t.time() + 600
    while len(res) < world:
        try:
            r, v = q.get(timeout=5)
            res[r] = v
        except _q.Empty:
            dead = [p for p in procs if p.exitcode not in (None, 0)]
            if dead or _t.time() > deadline:
                for p in procs:
                    p.kill()
                raise AssertionError(f"EP worker failed (exit codes {[p.exitcode for p in procs]})")
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("shape", [(2, 1024, 2048, 64, 1344, 4.0), (2, 256, 256, 8, 112, 2.0)])
def test_ep_loopback_bitwise(shape):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    res = _run(1, shape)
    assert res[0] == {"plain": True, "nccl": True, "ce": True}


def test_ep_two_gpus_bitwise():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    res = _run(2, (4, 1024, 2048, 64, 1344, 4.0), oracle=True)
    print("EP2 per-sample rel-err vs oracle:", {r: res[r]["oracle_rel_err"] for r in res})
    for r in range(2):
        errs = res[r].pop("oracle_rel_err")
        assert max(errs) <= 2e-2, errs
        assert res[r] == {"plain": True, "nccl": True, "ce": True}, res


def test_ep_four_gpus_bitwise():
    if torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    res = _run(4, (4, 1024, 2048, 64, 1344, 4.0), modes=("ce", "nccl"), oracle=True)
    print("EP4 per-sample rel-err vs oracle:", {r: res[r]["oracle_rel_err"] for r in res})
    for r in range(4):
        errs = res[r].pop("oracle_rel_err")
        assert max(errs) <= 2e-2, errs
        assert res[r] == {"ce": True, "nccl": True}, res


@pytest.mark.parametrize("world", [4, 8])
def test_ep_oversubscribed_ce_bitwise(world):
    """R ranks on fewer GPUs (rank % n_gpus): exercises the R-peer copy-engine
    schedule, segment tables and flag epochs at R = 4 and 8 on any box
    (an 8-GPU node is not available to the test runner)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if torch.cuda.device_count() >= world:
        pytest.skip("covered by the one-rank-per-GPU runs")
    res = _run(world, (world, 512, 2048, 64, 1344, 4.0), modes=("ce",))
    for r in range(world):
        assert res[r] == {"ce": True}, res


def _stack_worker(rank, world, port, q, dtype_name):
    """MoEDiT with expert-parallel MoE blocks vs the 1-GPU stack on the same
    samples: bitwise (same prologue / combine kernels, EP layer == 1-GPU)."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    ngpu = torch.cuda.device_count()
    torch.cuda.set_device(rank % ngpu)
    if world > ngpu:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    else:
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", rank % ngpu))
    try:
        from paper_2604_12163_b200 import dit as D
        from paper_2604_12163_b200.ep import EPContext
        from paper_2604_12163_b200.router import StageId
        dt = getattr(torch, dtype_name)
        # S1024 schedule: layers 3-4 at C=4, layer 5 at C=2 -> the EP chunk size
        # changes inside a step and back at the next (transport slot reuse)
        cfg = D.ModelConfig(n_layers=6, d_model=256, n_q_heads=4, n_kv_heads=1, head_dim=64,
                            n_experts=8, expert_hidden=112, dense_layers=3, latent_channels=16,
                            patch=2, dtype="float32", seed=1)
        params = D.init_parameters(cfg)
        rng = np.random.default_rng(4)
        for k in params:   # non-identity blocks
            if "mod." in k:
                params[k][...] = rng.standard_normal(params[k].shape) * 0.1
        B = 2 * world
        z = np.random.default_rng(5).standard_normal((B, 16, 32, 32)).astype(np.float32)
        t = np.linspace(0.1, 0.9, B)
        prompts = ["a cat", "two dogs on a beach", "sky", "red car at night"] * world
        sl = slice(2 * rank, 2 * rank + 2)
        single = D.MoEDiT(cfg, params, compute_dtype=dt, backend=D.CudaBackend(dt))
        ctx1 = single.precompute_text_kv(prompts[sl])
        ref, _ = single.forward(z[sl], t[sl], ctx1, StageId.S1024, return_aux=False)
        ep = D.MoEDiT(cfg, params, compute_dtype=dt, backend=D.CudaBackend(dt, ep=EPContext()))
        ctx2 = ep.precompute_text_kv(prompts[sl])
        ok = True
        for _ in range(3):
            out, _ = ep.forward(z[sl], t[sl], ctx2, StageId.S1024, return_aux=False)
            torch.cuda.synchronize()
            ok = ok and bool(torch.equal(out, ref))
        q.put((rank, {"stack": ok}))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _run_stack(world, dtype_name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_stack_worker, args=(r, world, port, q, dtype_name))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    import queue as _q
    import time as _t
    deadline = _t.time() + 600
    while len(res) < world:
        try:
            r, v = q.get(timeout=5)
            res[r] = v
        except _q.Empty:
            if any(p.exitcode not in (None, 0) for p in procs) or _t.time() > deadline:
                for p in procs:
                    p.kill()
                raise AssertionError(f"EP stack worker failed ({[p.exitcode for p in procs]})")
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("dtype_name", ["bfloat16", "float32"])
def test_ep_stack_matches_single_gpu(dtype_name):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    world = 2
    res = _run_stack(world, dtype_name)
    for r in range(world):
        assert res[r] == {"stack": True}, res
