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

Transports.
  "ce" (default): copy engines over NVLink. Receive and return buffers are
      CUDA-IPC shared between the ranks; every chunk moves with one
      cudaMemcpyAsync straight into the peer's buffer on a per-peer stream, and
      per-step 32-bit flags (cuStreamWriteValue32 into the peer's flag array /
      cuStreamWaitValue32 locally) order producer and consumer. No SMs are
      used, so transfers overlap the persistent tensor-core GEMMs, which hold
      every SM and would otherwise starve NCCL's copy kernels.
  "nccl": all_to_all for the dispatch on a comm stream (overlapping the shared
      expert and the rank's own chunk), per-chunk P2P returns on a second
      communicator. Kept for comparison.
  overlap=False: two blocking all_to_alls.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

import ctypes as C

from . import _lib
from ._tensors import stream_handle
from .errors import ConfigError
from .moe import ExpertBank
from .router import RouterConfig, build_routing, capacity_for


import os as _os

_DISPATCH_SERIAL = _os.environ.get("NIMG_EP_DISPATCH", "parallel") == "serial"
# remote chunks are computed in groups of at least this many rows per launch
_GROUP_ROWS = int(_os.environ.get("NIMG_EP_GROUP_ROWS", "12288"))
# expert slices of the last remote chunk, each returned as soon as computed
_RET_SPLIT = int(_os.environ.get("NIMG_EP_RET_SPLIT", "1"))
# own experts computed before the remote chunks (-1: half)
_OWN_A = int(_os.environ.get("NIMG_EP_OWN_A", "-1"))
# NIMG_EP_BG_GATHER=1: the rank-local gather runs inside the first grouped
# launch (background warps; the dispatch copies wait on per-chunk completion
# counters). Off by default: measured equal at EP2 (1.280 vs 1.290 ms weak)
# and slower at EP4 (1.53 vs 1.39 ms weak): inside the GEMM the gather runs on
# 2 warps per CTA, so the remote chunks -- and their dispatch copies -- finish
# later than with the dedicated gather kernel.
_BG_GATHER = _os.environ.get("NIMG_EP_BG_GATHER", "0") == "1"
# NIMG_EP_OWN_BG=1: only the rank's own chunk is gathered on the first grouped
# launch's background warps; the remote chunks by the gather kernel first
_BG_OWN = _os.environ.get("NIMG_EP_OWN_BG", "0") == "1"
# the rank-local combine forms the gates (no gate kernel; nimg_route_for_combine
# / nimg_combine_routed); NIMG_EP_FUSE_GATES=0 keeps the gate kernel
_FUSE_GATES = _os.environ.get("NIMG_EP_FUSE_GATES", "1") != "0"
_MAX_CHUNKS = 64


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

    def chunk_groups(self, min_rows: int):
        """Remote source ranks in arrival order (src = rank-1, rank-2, ...: the
        sender at distance s dispatches to this rank at its step s), split
        into consecutive groups of ~min_rows rows each, one grouped launch per
        group: small chunks alone would run partial waves on every launch.
        Group sizes are non-increasing, so the last group's return (which
        the rank's own second half must hide) is the smallest."""
        srcs = [(self.rank - s) % self.world for s in range(1, self.world)]
        if not srcs:
            return []
        g = max(1, -(-min_rows // max(1, self.chunk_rows)))
        ng = -(-len(srcs) // g)
        base, extra = divmod(len(srcs), ng)
        out, i = [], 0
        for j in range(ng):
            k = base + (1 if j < extra else 0)
            out.append(srcs[i:i + k])
            i += k
        return out

    def group_segments(self, srcs):
        """(offsets, expert ids) over the whole receive buffer computing only
        the chunks of `srcs`; other chunks are skip segments (expert -1, one
        per run of skipped chunks)."""
        El, blk, n = self.experts_per_rank, self.block_rows, self.chunk_rows
        want = set(srcs)
        off, ex = [0], []
        for src in range(self.world):
            if src in want:
                for el in range(El):
                    off.append(src * n + (el + 1) * blk)
                    ex.append(el)
            elif ex and ex[-1] == -1:
                off[-1] = (src + 1) * n
            else:
                off.append((src + 1) * n)
                ex.append(-1)
        return np.asarray(off, dtype=np.int64), np.asarray(ex, dtype=np.int32)

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


class _CAI:
    """__cuda_array_interface__ over a raw device pointer (no ownership)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3}


def _view(ptr: int, shape, dtype: torch.dtype, device) -> torch.Tensor:
    n = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
    return torch.as_tensor(_CAI(ptr, n), device=device).view(dtype).view(shape)


class PeerBuffer:
    """A device buffer per rank, mapped into every other rank of the group
    (CUDA IPC; ranks of one node)."""

    def __init__(self, nbytes: int, group, rank: int, world: int):
        own = C.c_void_p()
        handle = (C.c_uint8 * 64)()
        _lib.check(_lib.lib.nimg_ipc_alloc(nbytes, C.byref(own), handle))
        handles = [None] * world
        dist.all_gather_object(handles, bytes(handle), group=group)
        self.ptrs, self._opened = [], []
        for q in range(world):
            if q == rank:
                self.ptrs.append(own.value)
                continue
            p = C.c_void_p()
            _lib.check(_lib.lib.nimg_ipc_open((C.c_uint8 * 64).from_buffer_copy(handles[q]),
                                              C.byref(p)))
            self.ptrs.append(p.value)
            self._opened.append(p.value)
        self.own = own.value
        self.nbytes = nbytes

    def close(self):
        for p in self._opened:
            _lib.lib.nimg_ipc_close(p)
        _lib.lib.nimg_free(self.own)
        self._opened, self.ptrs = [], []


class CETransport:
    """Copy-engine exchange state: peer-shared receive / return buffers (grow
    only) and the per-step flags. One transport serves every EP layer of a
    model whatever its shape: each call views the buffers as (world, n, d) of
    its own chunk size, and the per-call epochs order the reuse of every slot
    across calls (a peer writes my receive slot for call k only after I
    returned its chunk of call k-1, my return slot only after I combined k-1)."""

    def __init__(self, group, rank, world, x_bytes, y_bytes, device):
        self.rank, self.world, self.device = rank, world, device
        self.x_cap, self.y_cap = x_bytes, y_bytes
        self.recv = PeerBuffer(world * x_bytes, group, rank, world)
        self.yback = PeerBuffer(world * y_bytes, group, rank, world)
        self.flags = PeerBuffer(3 * world * 4, group, rank, world)   # disp | ret | comb
        self.streams = [torch.cuda.Stream(device) for _ in range(world)]   # returns, per peer
        self.disp_stream = torch.cuda.Stream(device)
        # gather progress per destination chunk (written by the first grouped
        # launch's background gather, never reset): the dispatch copy of chunk
        # q waits until chunk_done[q] reaches the running total chunk_expect[q]
        self.chunk_done = torch.zeros(_MAX_CHUNKS, dtype=torch.int32, device=device)
        self.chunk_expect = [0] * _MAX_CHUNKS
        self.epoch = 0
        self.key = None
        self.reshaped = False
        dist.barrier(group=group)   # every buffer zeroed and mapped before first use

    def set_shape(self, chunk_rows, d, act, ydt):
        key = (chunk_rows, d, act, ydt)
        # A new chunk size moves the slot boundaries in the receive buffer: my
        # next chunk for q may overlap slots q has not consumed yet, which
        # q's RET flag (it consumed MY chunk) does not cover. The next
        # dispatch therefore also waits for q's COMB flag of the previous call
        # (q has combined, so it consumed its whole receive buffer).
        self.reshaped = self.key is not None and key != self.key
        if key != self.key:
            self.chunk_rows, self.d = chunk_rows, d
            self.act_es = torch.empty((), dtype=act).element_size()
            self.y_es = torch.empty((), dtype=ydt).element_size()
            self.recv_t = _view(self.recv.own, (self.world, chunk_rows, d), act, self.device)
            self.yback_t = _view(self.yback.own, (self.world, chunk_rows, d), ydt, self.device)
            self.key = key
        return self

    def flag(self, owner: int, kind: int, idx: int) -> int:
        return self.flags.ptrs[owner] + 4 * (kind * self.world + idx)

    def close(self):
        for b in (self.recv, self.yback, self.flags):
            b.close()


class _Ring:
    """Two persistent buffers of one shape, handed out alternately. Before a
    slot is reused, the current stream waits for the side-stream readers of
    its previous use (events the caller records with reader_done). Replaces
    per-step allocations whose record_stream() deferred frees would keep the
    caching allocator growing -- each new segment a cudaMalloc that must also
    map into every IPC peer, stalling the host for tens of ms mid-run."""

    def __init__(self, shape, dtype, device):
        self.bufs = [torch.empty(shape, dtype=dtype, device=device) for _ in range(2)]
        self.events = [[], []]
        self.k = 0

    def next(self):
        s = self.k % 2
        self.k += 1
        cur = torch.cuda.current_stream()
        for ev in self.events[s]:
            cur.wait_event(ev)
        self.events[s] = []
        return s, self.bufs[s]

    def reader_done(self, slot: int, stream) -> None:
        ev = torch.cuda.Event()
        ev.record(stream)
        self.events[slot].append(ev)


class EPContext:
    """Process groups, streams and transport state of one expert-parallel layer."""

    def __init__(self, group=None, overlap: bool = True, transport: str = "ce"):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.overlap = overlap and self.world > 1
        if transport not in ("ce", "nccl"):
            raise ConfigError(f"unknown EP transport {transport!r}")
        self.transport = transport
        self._ce = None
        self._ret_group = None
        self._streams = None
        self._rings = {}

    def ring(self, name: str, shape, dtype, device) -> _Ring:
        key = (name, tuple(shape), dtype, str(device))
        r = self._rings.get(key)
        if r is None:
            r = self._rings[key] = _Ring(shape, dtype, device)
        return r

    def ce(self, chunk_rows, d, act, ydt, device) -> CETransport:
        """The transport, grown (collectively: every rank makes the same calls)
        only when a call needs larger chunks than any before."""
        xb = chunk_rows * d * torch.empty((), dtype=act).element_size()
        yb = chunk_rows * d * torch.empty((), dtype=ydt).element_size()
        tp = self._ce
        if tp is None or xb > tp.x_cap or yb > tp.y_cap:
            if tp is not None:
                xb, yb = max(xb, tp.x_cap), max(yb, tp.y_cap)
                torch.cuda.synchronize()
                dist.barrier(group=self.group)   # no peer still copies into the old buffers
                tp.close()
            self._ce = tp = CETransport(self.group, self.rank, self.world, xb, yb, device)
        return tp.set_shape(chunk_rows, d, act, ydt)

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


_TRACE = _os.environ.get("NIMG_EP_TRACE") == "1"


def _mark(timeline, name):
    if _TRACE:
        import sys as _sys
        print(f"[ep rank {dist.get_rank()}] {name}", file=_sys.stderr, flush=True)
    if timeline is not None:
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        timeline.append((name, ev))


def ep_moe_block_forward(x, sa_gate, r_attn, ff_scale, ff_gate, t_vec, layer: int,
                         cfg: RouterConfig, bank_local: ExpertBank, w_r, ctx: "EPContext",
                         return_routing: bool = False):
    """Expert-parallel MoE branch of the backbone (backbone.py:583-606) for
    this rank's samples: the 1-GPU block's prologue kernels, the EP layer, and
    the gated residual in the combine epilogue -- the same kernels as
    block.moe_block_forward, so the result equals the 1-GPU block."""
    from .block import moe_block_prologue
    h, x_norm, x_mod, th_ff = moe_block_prologue(x, sa_gate, r_attn, ff_scale, ff_gate, layer, cfg)
    return ep_moe_forward(x_norm, x_mod, t_vec, cfg, bank_local, w_r, ctx,
                          return_routing=return_routing, residual=(h, th_ff))


def ep_moe_forward(x_norm, x_mod, t_emb, cfg: RouterConfig, bank_local: ExpertBank, w_r,
                   ctx: EPContext, stages=None, return_routing: bool = False, timeline=None,
                   residual=None):
    """Expert-parallel moe_forward (moe.py:138-164) for this rank's samples.

    x_norm, x_mod: (B_l, S, d) local samples; bank_local: this rank's El
    experts (shard_bank) + the shared expert; w_r, t_emb as in moe_forward.
    residual = (h, th_ff): the combine adds backbone.py:606 in its epilogue.
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
    if act == torch.float64 or x_norm.dtype == torch.float64:
        raise ConfigError("expert parallel runs the fp32 / bf16 modes (the f64 mode is 1-GPU)")
    T = B_l * S
    xm = x_mod.reshape(T, d)
    w = bank_local

    _mark(timeline, "start")
    r = stages.route(x_norm, t_emb, w_r, cfg, cap, for_combine=_FUSE_GATES)
    _mark(timeline, "routed")
    xring = None
    bg = None
    if ctx.overlap and ctx.transport == "ce":
        # persistent double buffer (read by the dispatch copy streams)
        xring = ctx.ring("xg", (E * B_l * cap, d), act, x_mod.device)
        xslot, xg = xring.next()
        flags = (stages.bg_flags(r) if (_BG_GATHER or _BG_OWN) and ctx.world > 1
                 and ctx.world <= _MAX_CHUNKS and hasattr(stages, "bg_flags") else 0)
        if flags and _BG_GATHER:
            # the first grouped launch gathers every chunk while it runs
            bg = {"src": xm, "idx": r["token_flat"], "dst": xg, "flags": flags}
        elif flags:
            # the remote chunks first (the dispatch copies wait for them), then
            # the own chunk on the first grouped launch's background warps
            n, me, tf = plan.chunk_rows, plan.rank, r["token_flat"]
            if me > 0:
                stages.gather(xm, tf[:me * n], out=xg[:me * n])
            if me < ctx.world - 1:
                stages.gather(xm, tf[(me + 1) * n:], out=xg[(me + 1) * n:])
            bg = {"src": xm, "idx": tf[me * n:(me + 1) * n], "dst": xg[me * n:(me + 1) * n],
                  "flags": flags, "own": True}
        else:
            stages.gather(xm, r["token_flat"], out=xg)
    else:
        xg = stages.gather(xm, r["token_flat"])                   # (E*B_l*cap, d)
    _mark(timeline, "gathered")

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
    elif ctx.transport == "ce":
        y_back, y_sh = _ce_exchange(plan, ctx, stages, xg, xm, w, timeline, (xring, xslot), bg)
    else:
        y_back, y_sh = _overlapped_exchange(plan, ctx, stages, xg, xm, w, timeline)
    _mark(timeline, "returned")
    out = (stages.combine(y_back, y_sh, r, act) if residual is None else
           stages.combine(y_back, y_sh, r, act, residual=residual)).view(B_l, S, d)
    if ctx.overlap and ctx.transport == "ce":
        ce_after_combine(ctx)
    _mark(timeline, "combined")
    if return_routing:
        decisions, routing = build_routing(r, B_l, S, E, cap)
        return out, decisions, routing
    return out


def _overlapped_exchange(plan: EPPlan, ctx: EPContext, stages, xg, xm, w, timeline=None):
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
    _mark(timeline, "own+shared")

    comp.wait_event(disp_done)
    _mark(timeline, "dispatched")
    ret_group = ctx.ret_group
    for s in range(1, R):
        send_to, recv_from = plan.step_peers(s)           # dispatch pairing of step s
        # chunk that arrived from `recv_from` -> compute -> send back to it
        stages.expert_ffn(recv_c[recv_from], coff, cex, w.w1, w.w3, w.w2, None, None, None, None,
                          y_routed=y_recv[recv_from])
        _mark(timeline, f"chunk{s}")
        s_ret.wait_stream(comp)
        with torch.cuda.stream(s_ret):
            ops = [dist.P2POp(dist.isend, y_recv[recv_from], recv_from, group=ret_group),
                   dist.P2POp(dist.irecv, y_back[send_to], send_to, group=ret_group)]
            for wk in dist.batch_isend_irecv(ops):
                wk.wait()
    comp.wait_stream(s_ret)
    return y_back.view(R * n, -1), y_sh


def _ce_exchange(plan: EPPlan, ctx: EPContext, stages, xg, xm, w, timeline=None, xring=None,
                 bg=None):
    """Copy-engine dispatch / return with per-step flags (see module doc).

    Flags in rank r's array: disp[src] (src's chunk for r has landed in r's
    recv), ret[q] (q's results for r have landed in r's y_back; also: q has
    consumed r's previous chunk), comb[src] (src combined the previous step, so
    its y_back slot for r may be overwritten)."""
    L = _lib.lib
    R, me, n = plan.world, plan.rank, plan.chunk_rows
    d = xg.shape[1]
    dev = xg.device
    ydt = stages.ffn_y_dtype(xg.dtype, d, w.w1.shape[1], w.shared_w1.shape[0])
    tp = ctx.ce(n, d, xg.dtype, ydt, dev)
    tp.epoch += 1
    k = tp.epoch
    DISP, RET, COMB = 0, 1, 2
    comp = torch.cuda.current_stream()
    xbytes, ybytes = n * d * tp.act_es, n * d * tp.y_es
    coff, cex = plan.chunk_segments()

    own_bg = bg is not None and bg.get("own", False)
    if own_bg:   # the own chunk only: no dispatch copy waits on it
        bg = {k: v for k, v in bg.items() if k != "own"}
    elif bg is not None:
        # sub-blocks of 32 gathered rows overlapping each chunk: the running
        # totals the dispatch copies wait for
        bg = dict(bg, row_off=me * n, chunk_rows=n, chunk_done=tp.chunk_done.data_ptr())
        for q in range(R):
            tp.chunk_expect[q] += ((q + 1) * n - 1) // 32 - (q * n) // 32 + 1
    # The rank's own chunk needs no exchange: its first half of experts runs
    # right after the shared expert (together they cover the dispatch copies),
    # its second half last (covers the final return copy).
    El = plan.experts_per_rank
    half = (min(El, max(0, _OWN_A)) if _OWN_A >= 0 else El // 2) if R > 1 else El
    blk = plan.block_rows
    own_x = xg[me * n:(me + 1) * n]

    def own_part(e0, e1, shared=False, gather=None):
        xs = (xm, w.shared_w1, w.shared_w3, w.shared_w2) if shared else (None,) * 4
        if e1 <= e0:
            return stages.expert_ffn(None, None, None, None, None, None, *xs,
                                     gather=gather) if shared else None
        off = (np.arange(e0, e1 + 1, dtype=np.int64) - e0) * blk
        return stages.expert_ffn(own_x[e0 * blk:e1 * blk], off, np.arange(e0, e1, dtype=np.int32),
                                 w.w1, w.w3, w.w2, *xs, y_routed=tp.yback_t[me, e0 * blk:e1 * blk],
                                 gather=gather)

    # shared expert + first half of the own chunk in one grouped launch (with
    # bg: that launch also gathers every chunk, the dispatch copies start as
    # their chunks complete). It is enqueued BEFORE the dispatch copies: a
    # peer copy may block the host until it runs, and with bg it waits on this
    # launch's progress (GPU-side the copies only wait on x_ready + chunk_done).
    x_ready = torch.cuda.Event()
    x_ready.record(comp)
    _, y_sh = own_part(0, half, shared=True, gather=bg)
    _mark(timeline, "shared+own_a")

    # dispatch: one copy per destination rank, straight into its recv slot.
    # "parallel" (default): one stream per destination; "serial"
    # (NIMG_EP_DISPATCH=serial): one stream, in the order destinations consume
    # the chunks (destination me+s uses it at its step s).
    serial = _DISPATCH_SERIAL
    for s in range(1, R):
        q = (me + s) % R
        st = tp.disp_stream if serial else tp.streams[q]
        if not serial or s == 1:
            st.wait_event(x_ready)
        sh = st.cuda_stream
        if bg is not None and not own_bg:   # chunk q gathered by the first grouped launch
            _lib.check(L.nimg_stream_wait_geq_u32(tp.chunk_done.data_ptr() + 4 * q,
                                                  tp.chunk_expect[q] & 0xFFFFFFFF, sh))
        if k > 1:   # q consumed my previous chunk
            _lib.check(L.nimg_stream_wait_geq_u32(tp.flag(me, RET, q), k - 1, sh))
            if tp.reshaped:   # ... and, after a chunk-size change, every chunk (see set_shape)
                _lib.check(L.nimg_stream_wait_geq_u32(tp.flag(me, COMB, q), k - 1, sh))
        if timeline is not None:
            ev0 = torch.cuda.Event(enable_timing=True)
            ev0.record(st)
        _lib.check(L.nimg_copy_async(tp.recv.ptrs[q] + me * xbytes, xg[q * n:(q + 1) * n].data_ptr(),
                                     xbytes, sh))
        if timeline is not None:
            ev1 = torch.cuda.Event(enable_timing=True)
            ev1.record(st)
            timeline.append((f"copy_start_q{q}", ev0))
            timeline.append((f"copy_end_q{q}", ev1))
        _lib.check(L.nimg_stream_write_u32(tp.flag(q, DISP, me), k, sh))
        if xring is not None and xring[0] is not None:
            xring[0].reader_done(xring[1], st)
        else:
            xg.record_stream(st)

    yring = ctx.ring("y_recv", (R, n, d), ydt, dev)
    yslot, y_recv = yring.next()
    recv_all = tp.recv_t.view(R * n, d)
    y_all = y_recv.view(R * n, d)
    groups = plan.chunk_groups(_GROUP_ROWS)
    for gi, grp in enumerate(groups):
        for src in grp:
            _lib.check(L.nimg_stream_wait_geq_u32(tp.flag(me, DISP, src), k, comp.cuda_stream))
        if len(grp) == 1 and gi == len(groups) - 1 and _RET_SPLIT > 1:
            # the last remote chunk in expert slices, each returned as soon as
            # it is computed: only the last slice's copy is left for the own
            # second half to hide
            src = grp[0]
            st = tp.streams[src]
            sh = st.cuda_stream
            cuts = [El * i // _RET_SPLIT for i in range(_RET_SPLIT + 1)]
            for i in range(_RET_SPLIT):
                e0, e1 = cuts[i], cuts[i + 1]
                if e1 <= e0:
                    continue
                r0, r1 = e0 * blk, e1 * blk
                stages.expert_ffn(tp.recv_t[src][r0:r1], coff[e0:e1 + 1] - coff[e0], cex[e0:e1],
                                  w.w1, w.w3, w.w2, None, None, None, None, y_routed=y_recv[src][r0:r1])
                done = torch.cuda.Event()
                done.record(comp)
                st.wait_event(done)
                if k > 1 and i == 0:   # src has combined the previous step: its y_back slot is free
                    _lib.check(L.nimg_stream_wait_geq_u32(tp.flag(me, COMB, src), k - 1, sh))
                _lib.check(L.nimg_copy_async(tp.yback.ptrs[src] + me * ybytes + r0 * d * tp.y_es,
                                             y_recv[src][r0:r1].data_ptr(), (r1 - r0) * d * tp.y_es, sh))
            _lib.check(L.nimg_stream_write_u32(tp.flag(src, RET, me), k, sh))
            _mark(timeline, f"group{gi + 1}")
            continue
        if len(grp) == 1:
            src = grp[0]
            stages.expert_ffn(tp.recv_t[src], coff, cex, w.w1, w.w3, w.w2, None, None, None, None,
                              y_routed=y_recv[src])
        else:
            goff, gex = plan.group_segments(grp)
            stages.expert_ffn(recv_all, goff, gex, w.w1, w.w3, w.w2, None, None, None, None,
                              y_routed=y_all)
        _mark(timeline, f"group{gi + 1}")
        done = torch.cuda.Event()
        done.record(comp)
        for src in grp:
            st = tp.streams[src]
            st.wait_event(done)
            sh = st.cuda_stream
            if k > 1:   # src has combined the previous step: its y_back slot is free
                _lib.check(L.nimg_stream_wait_geq_u32(tp.flag(me, COMB, src), k - 1, sh))
            _lib.check(L.nimg_copy_async(tp.yback.ptrs[src] + me * ybytes, y_recv[src].data_ptr(),
                                         ybytes, sh))
            _lib.check(L.nimg_stream_write_u32(tp.flag(src, RET, me), k, sh))
    for st in tp.streams:
        yring.reader_done(yslot, st)

    own_part(half, El)
    _mark(timeline, "own_b")

    for q in range(R):
        if q != me:
            _lib.check(L.nimg_stream_wait_geq_u32(tp.flag(me, RET, q), k, comp.cuda_stream))
    return tp.yback_t.view(R * n, d), y_sh


def ce_after_combine(ctx: EPContext):
    """Tell every peer that this rank's y_back slots are free again."""
    tp = ctx._ce
    if tp is None:
        return
    done = torch.cuda.Event()
    done.record(torch.cuda.current_stream())
    for q in range(tp.world):
        if q == tp.rank:
            continue
        st = tp.streams[q]
        st.wait_event(done)
        _lib.check(_lib.lib.nimg_stream_write_u32(tp.flag(q, 2, tp.rank), tp.epoch, st.cuda_stream))
