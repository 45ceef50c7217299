"""Does enqueueing a peer copy / stream wait block the host? (2 ranks, torchrun)
A stream is made to wait behind a ~100 ms sleep kernel; we time the host cost
of enqueueing ops behind it."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

rank = int(os.environ["RANK"])
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
from paper_2604_12163_b200 import _lib
from paper_2604_12163_b200.ep import PeerBuffer

L = _lib.lib
nb = 64 << 20
buf = PeerBuffer(nb, None, rank, 2)
flags = PeerBuffer(64, None, rank, 2)
src = torch.empty(nb, dtype=torch.uint8, device="cuda")
peer = 1 - rank
dist.barrier()
if rank == 0:
    def hold(st):
        with torch.cuda.stream(st):
            torch.cuda._sleep(200_000_000)   # ~100 ms
    for what in ("copy_local", "copy_peer", "wait_value", "wait_then_copy_peer", "write_value_peer"):
        st = torch.cuda.Stream()
        hold(st)
        t0 = time.perf_counter()
        h = st.cuda_stream
        if what == "copy_local":
            _lib.check(L.nimg_copy_async(buf.own, src.data_ptr(), nb, h))
        elif what == "copy_peer":
            _lib.check(L.nimg_copy_async(buf.ptrs[peer], src.data_ptr(), nb, h))
        elif what == "wait_value":
            _lib.check(L.nimg_stream_wait_geq_u32(flags.own, 0, h))
        elif what == "wait_then_copy_peer":
            _lib.check(L.nimg_stream_wait_geq_u32(flags.own, 0, h))
            _lib.check(L.nimg_copy_async(buf.ptrs[peer], src.data_ptr(), nb, h))
        elif what == "write_value_peer":
            _lib.check(L.nimg_stream_write_u32(flags.ptrs[peer], 1, h))
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"{what:22s}: host enqueue {1e3 * (t1 - t0):8.3f} ms (stream drained after {1e3 * (t2 - t0):.1f} ms)",
              flush=True)
dist.barrier()
