"""Expert-parallel MoE layer over NCCL (spec'd as epsim in
/root/reference/SPEC.md:698-766, not shipped by the reference).

Layout. Rank r owns samples [r*B_l, (r+1)*B_l) and experts
[r*El, (r+1)*El) with El = E / R. Routing is per sample (router.py:127), so
router, select, gates, gather, shared expert and combine are rank-local.
Expert-choice counts are static -- every (source rank, expert) pair carries
exactly B_l*cap rows -- so the counts all-to-all of the paper
is unnecessary and both exchanges are uniform all-to-alls:

  dispatch  xg[e, b, slot] (local expert-major gather, router.py:131-133) is
            split by destination rank (contiguous expert ranges) -> recv laid
            out [src][el][b][slot]; segment (src, el) is B_l*cap rows of local
            expert el.
  return    y_recv goes back along the same split, so y_back lands in the
            sender's own [e][b][slot] order -- the same row numbering as the
            1-GPU layout -- and the deterministic combine runs unchanged.
            Hence EP(R) == 1-GPU bitwise (tested).

Overlap (default): the dispatch all-to-all runs on a comm stream while the
compute stream runs the shared expert and the rank's own chunk; remote chunks
are then computed one source rank at a time and each finished chunk is sent
back on a second communicator while the next chunk computes.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from .errors import ConfigError
from .moe import ExpertBank
from .router import RouterConfig, build_routing, capacity_for


@dataclass(frozen=True)
class EPPlan:
    """Static exchange plan for one rank (pure host arithmetic)."""
    world: int
    rank: int
    n_experts: int
    b_local: int
    seq: int
    cap: int

    def __post_init__(self):
        if self.n_experts % self.world:
            raise ConfigError(f"n_experts {self.n_experts} not divisible by world {self.world}")

    @property
    def experts_per_rank(self) -> int:
        return self.n_experts // self.world

    @property
    def block_rows(self) -> int:
        """Rows per (source rank, expert) block: B_l * cap."""
        return self.b_local * self.cap

    @property
    def chunk_rows(self) -> int:
        """Rows exchanged with one peer in one direction."""
        return self.experts_per_rank * self.block_rows

    def local_experts(self) -> range:
        El = self.experts_per_rank
        return range(self.rank * El, (self.rank + 1) * El)

    def recv_segments(self):
        """(offsets, local expert ids) over the whole receive buffer."""
        El = self.experts_per_rank
        off = np.arange(self.world * El + 1, dtype=np.int64) * self.block_rows
        ex = np.tile(np.arange(El, dtype=np.int32), self.world)
        return off, ex

    def chunk_segments(self):
        """(offsets, local expert ids) of one source chunk."""
        El = self.experts_per_rank
        return (np.arange(El + 1, dtype=np.int64) * self.block_rows,
                np.arange(El, dtype=np.int32))

    def step_peers(self, s: int):
        """Pairwise step s (1..R-1): (send-to, receive-from) for the dispatch;
        the return of step s uses the reverse pair."""
        return (self.rank + s) % self.world, (self.rank - s) % self.world


def shard_bank(bank: ExpertBank, rank: int, world: int) -> ExpertBank:
    """Local expert slice + replicated shared expert."""
    E = bank.n_experts
    if E % world:
        raise ConfigError(f"n_experts {E} not divisible by world {world}")
    El = E // world
    sl = slice(rank * El, (rank + 1) * El)
    return ExpertBank(bank.w1[sl], bank.w3[sl], bank.w2[sl], bank.shared_w1, bank.shared_w3,
                      bank.shared_w2)


class EPContext:
    """Process groups and streams for one expert-parallel layer."""

    def __init__(self, group=None, overlap: bool = True):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.overlap = overlap and self.world > 1
        self._ret_group = None
        self._streams = None

    @property
    def ret_group(self):
        # a second communicator so returns overlap with the dispatch's stream
        if self._ret_group is None:
            ranks = list(range(self.world)) if self.group is None else dist.get_process_group_ranks(self.group)
            self._ret_group = dist.new_group(ranks) if self.overlap else self.group
        return self._ret_group

    def streams(self):
        if self._streams is None:
            self._streams = (torch.cuda.Stream(), torch.cuda.Stream())
        return self._streams


def ep_moe_forward(x_norm, x_mod, t_emb, cfg: RouterConfig, bank_local: ExpertBank, w_r,
                   ctx: EPContext, stages=None, return_routing: bool = False):
    """Expert-parallel moe_forward (moe.py:138-164) for this rank's samples.

    x_norm, x_mod: (B_l, S, d) local samples; bank_local: this rank's El
    experts (shard_bank) + the shared expert; w_r, t_emb as in moe_forward.
    """
    if stages is None:
        from .stages import CudaStages
        stages = CudaStages()
    B_l, S, d = x_mod.shape
    E = cfg.n_experts
    cap = capacity_for(S, E, cfg.capacity_factor)
    plan = EPPlan(ctx.world, ctx.rank, E, B_l, S, cap)
    if bank_local.w1.shape[0] != plan.experts_per_rank:
        raise ConfigError(f"local bank has {bank_local.w1.shape[0]} experts, plan needs "
                          f"{plan.experts_per_rank}")
    act = x_mod.dtype
    T = B_l * S
    xm = x_mod.reshape(T, d)
    w = bank_local

    r = stages.route(x_norm, t_emb, w_r, cfg, cap)
    xg = stages.gather(xm, r["token_flat"])                       # (E*B_l*cap, d)

    if not ctx.overlap:
        recv = torch.empty_like(xg)
        if ctx.world > 1:
            dist.all_to_all_single(recv, xg, group=ctx.group)
        else:
            recv.copy_(xg)
        off, ex = plan.recv_segments()
        y_recv, y_sh = stages.expert_ffn(recv, off, ex, w.w1, w.w3, w.w2, xm, w.shared_w1,
                                         w.shared_w3, w.shared_w2)
        y_back = torch.empty_like(y_recv)
        if ctx.world > 1:
            dist.all_to_all_single(y_back, y_recv, group=ctx.group)
        else:
            y_back.copy_(y_recv)
    else:
        y_back, y_sh = _overlapped_exchange(plan, ctx, stages, xg, xm, w)

    out = stages.combine(y_back, y_sh, r, act).view(B_l, S, d)
    if return_routing:
        decisions, routing = build_routing(r, B_l, S, E, cap)
        return out, decisions, routing
    return out


def _overlapped_exchange(plan: EPPlan, ctx: EPContext, stages, xg, xm, w):
    R, me, n = plan.world, plan.rank, plan.chunk_rows
    comp = torch.cuda.current_stream()
    s_disp, s_ret = ctx.streams()
    recv = torch.empty_like(xg)
    xg_c = xg.view(R, n, -1)
    recv_c = recv.view(R, n, -1)
    coff, cex = plan.chunk_segments()

    # dispatch on its own stream (after the gather)
    s_disp.wait_stream(comp)
    with torch.cuda.stream(s_disp):
        dist.all_to_all_single(recv, xg, group=ctx.group)
        disp_done = torch.cuda.Event()
        disp_done.record(s_disp)

    # meanwhile: shared expert (all local tokens) + this rank's own chunk,
    # written straight into its final place in y_back
    d = xg.shape[1]
    ydt = stages.ffn_y_dtype(xg.dtype, d, w.w1.shape[1], w.shared_w1.shape[0])
    y_recv = torch.empty((R, n, d), dtype=ydt, device=xg.device)
    y_back = torch.empty((R, n, d), dtype=ydt, device=xg.device)
    _, y_sh = stages.expert_ffn(xg_c[me], coff, cex, w.w1, w.w3, w.w2, xm, w.shared_w1,
                                w.shared_w3, w.shared_w2, y_routed=y_back[me])

    comp.wait_event(disp_done)
    ret_group = ctx.ret_group
    for s in range(1, R):
        send_to, recv_from = plan.step_peers(s)           # dispatch pairing of step s
        # chunk that arrived from `recv_from` -> compute -> send back to it
        stages.expert_ffn(recv_c[recv_from], coff, cex, w.w1, w.w3, w.w2, None, None, None, None,
                          y_routed=y_recv[recv_from])
        s_ret.wait_stream(comp)
        with torch.cuda.stream(s_ret):
            ops = [dist.P2POp(dist.isend, y_recv[recv_from], recv_from, group=ret_group),
                   dist.P2POp(dist.irecv, y_back[send_to], send_to, group=ret_group)]
            for wk in dist.batch_isend_irecv(ops):
                wk.wait()
    comp.wait_stream(s_ret)
    return y_back.view(R * n, -1), y_sh
