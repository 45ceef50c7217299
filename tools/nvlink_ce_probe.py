"""NVLink hardware-counter evidence for the copy-engine exchange (ep.py).

One process drives two GPUs and moves the EP exchange's chunks peer to peer
with the same copy-engine path ep.py uses (cudaMemcpyAsync between peer
buffers, both directions at once, as dispatch and return overlap). Under
`ncu --replay-mode range --profile-from-start off --metrics
nvltx__bytes.sum,nvlrx__bytes.sum,gpu__time_duration.sum` the region between
cudaProfilerStart/Stop is one profiled range, so ncu reports the NVLink TX/RX
bytes the copies put on the links (ep.py's CE copies are not kernels, so a
per-kernel ncu capture of the EP step cannot see them). Without ncu it
prints the CUDA-event bandwidth of the same copies.

  python tools/nvlink_ce_probe.py [chunk_MB ...]
"""
import sys

import torch

sizes = [int(a) for a in sys.argv[1:]] or [134, 67]
torch.cuda.set_device(0)
for dev in (0, 1):
    with torch.cuda.device(dev):
        torch.zeros(1, device=dev)
a0 = {s: torch.empty(s << 20, dtype=torch.uint8, device="cuda:0") for s in sizes}
a1 = {s: torch.empty(s << 20, dtype=torch.uint8, device="cuda:1") for s in sizes}
b0 = {s: torch.empty(s << 20, dtype=torch.uint8, device="cuda:0") for s in sizes}
b1 = {s: torch.empty(s << 20, dtype=torch.uint8, device="cuda:1") for s in sizes}
s0 = torch.cuda.Stream(device=0)
tick = torch.zeros(16, device="cuda:0")
s1 = torch.cuda.Stream(device=1)
for s in sizes:   # warm (peer mappings, copy engines)
    with torch.cuda.stream(s0):
        a1[s].copy_(a0[s], non_blocking=True)
    with torch.cuda.stream(s1):
        b0[s].copy_(b1[s], non_blocking=True)
torch.cuda.synchronize(0)
torch.cuda.synchronize(1)
for s in sizes:
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.profiler.start()
    with torch.cuda.stream(s0):
        tick.add_(1)       # range replay needs a kernel in the range
    ev[0].record(s0)
    s1.wait_event(ev[0])
    with torch.cuda.stream(s0):
        a1[s].copy_(a0[s], non_blocking=True)     # GPU0 -> GPU1 (dispatch direction)
    with torch.cuda.stream(s1):
        b0[s].copy_(b1[s], non_blocking=True)     # GPU1 -> GPU0 (return direction)
    done1 = torch.cuda.Event()
    done1.record(s1)
    s0.wait_event(done1)
    with torch.cuda.stream(s0):
        tick.add_(1)
    ev[1].record(s0)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    torch.cuda.profiler.stop()
    ms = ev[0].elapsed_time(ev[1])
    nbytes = s << 20
    print(f"chunk {s} MB each way: {ms:.3f} ms, {nbytes / ms / 1e6:.1f} GB/s per direction "
          f"(GPU0 egress {nbytes} B, ingress {nbytes} B)", flush=True)
