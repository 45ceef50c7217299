"""Expert-parallel host logic on CPU: the exchange plan (pure arithmetic) and a
world_size-2 gloo run of ep_moe_forward with the oracle test double standing
in for the CUDA stages. The distributed result must equal the single-process
oracle layer (the EP layout is the 1-GPU expert-major layout)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import nimg_oracle as O
from oracle.workloads import make_layer_inputs


def test_plan_layout():
    from paper_2604_12163_b200.ep import EPPlan
    p = EPPlan(world=4, rank=1, n_experts=64, b_local=8, seq=4096, cap=128)
    assert p.experts_per_rank == 16
    assert p.block_rows == 1024 and p.chunk_rows == 16 * 1024
    off, ex = p.recv_segments()
    assert len(off) == 65 and off[-1] == 4 * 16 * 1024
    assert list(ex[:17]) == list(range(16)) + [0]
    assert list(p.local_experts()) == list(range(16, 32))
    for s in range(1, 4):
        to, frm = p.step_peers(s)
        # the peer we send to at step s receives from us at the same step
        assert EPPlan(4, to, 64, 8, 4096, 128).step_peers(s)[1] == 1
    from paper_2604_12163_b200.errors import ConfigError
    with pytest.raises(ConfigError):
        EPPlan(world=3, rank=0, n_experts=64, b_local=1, seq=8, cap=1)


def test_chunk_groups_and_skip_segments():
    from paper_2604_12163_b200.ep import EPPlan
    # cfg2 weak-scaled at 8 ranks: chunks of 8192 rows run in pairs
    p = EPPlan(world=8, rank=1, n_experts=64, b_local=16, seq=1024, cap=64)
    assert p.chunk_rows == 8192
    groups = p.chunk_groups(12288)
    assert groups == [[0, 7], [6, 5], [4, 3], [2]]           # arrival order, sizes 2,2,2,1
    assert sorted(sum(groups, [])) == [0, 2, 3, 4, 5, 6, 7]
    off, ex = p.group_segments([0, 7])                      # wraps around the buffer
    n, blk = p.chunk_rows, p.block_rows
    assert off[0] == 0 and off[-1] == 8 * n and np.all(np.diff(off) >= 0)
    assert list(ex) == list(range(8)) + [-1] + list(range(8))
    assert off[8] == n and off[9] == 7 * n and off[10] == 7 * n + blk
    # 4 ranks: chunks already >= the threshold, one per launch
    q = EPPlan(world=4, rank=2, n_experts=64, b_local=16, seq=1024, cap=64)
    assert q.chunk_groups(12288) == [[1], [0], [3]]
    # cfg4 strong at 8 ranks (4096-row chunks): groups of 3,2,2
    r = EPPlan(world=8, rank=0, n_experts=64, b_local=4, seq=4096, cap=128)
    assert [len(g) for g in r.chunk_groups(12288)] == [3, 2, 2]
    assert EPPlan(world=1, rank=0, n_experts=8, b_local=2, seq=16, cap=4).chunk_groups(12288) == []
    # every computed row is covered exactly once, skipped chunks not at all
    off, ex = r.group_segments([7, 6, 5])
    cover = np.zeros(8 * r.chunk_rows, np.int32)
    for i, e in enumerate(ex):
        if e >= 0:
            cover[off[i]:off[i + 1]] += 1
    assert cover.reshape(8, -1).all(axis=1).tolist() == [False] * 5 + [True] * 3
    assert cover.max() == 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_12163_b200.ep import EPContext, ep_moe_forward, shard_bank
        from paper_2604_12163_b200.moe import ExpertBank
        from paper_2604_12163_b200.router import RouterConfig
        from tests.ep_cpu_stages import OracleStages
        B, S, d, E, h, C = 4, 24, 16, 8, 12, 2.0
        inp = make_layer_inputs(21, B, S, d, E, h)
        T = {k: torch.from_numpy(v) for k, v in inp.items()}
        bl = B // world
        sl = slice(rank * bl, (rank + 1) * bl)
        bank = shard_bank(ExpertBank(T["w1"], T["w3"], T["w2"], T["sw1"], T["sw3"], T["sw2"]),
                          rank, world)
        cfg = RouterConfig(d_model=d, n_experts=E, capacity_factor=C)
        ctx = EPContext(overlap=False)
        out = ep_moe_forward(T["x_norm"][sl], T["x_mod"][sl], T["t_emb"][sl], cfg, bank, T["w_r"],
                             ctx, stages=OracleStages())
        q.put((rank, out.numpy()))
    finally:
        dist.destroy_process_group()


def test_ep_world2_gloo_matches_single_process_oracle():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = np.concatenate([res[r] for r in range(world)], axis=0)
    B, S, d, E, h, C = 4, 24, 16, 8, 12, 2.0
    inp = make_layer_inputs(21, B, S, d, E, h)
    want = O.moe_forward(inp["x_norm"], inp["x_mod"], inp["t_emb"], inp["w_r"], inp["w1"],
                         inp["w3"], inp["w2"], inp["sw1"], inp["sw3"], inp["sw2"], capacity_factor=C)
    np.testing.assert_allclose(got, want, rtol=1e-6, atol=1e-7)
