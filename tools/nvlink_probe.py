"""Probe which NVLink traffic counters this driver exposes (run on a >=2-GPU box)."""
import subprocess
import pynvml as N
import torch

N.nvmlInit()
h = N.nvmlDeviceGetHandleByIndex(0)
links = [l for l in range(18) if N.nvmlDeviceGetNvLinkState(h, l) == N.NVML_FEATURE_ENABLED]
print("active links", links)
for f in (138, 139, 140, 141, 201, 202, 203, 204):
    try:
        v = N.nvmlDeviceGetFieldValues(h, [(f, links[0])])[0]
        v2 = N.nvmlDeviceGetFieldValues(h, [f])[0]
        print("field", f, "scoped ret", v.nvmlReturn, "val", v.value.ullVal, "| unscoped ret", v2.nvmlReturn, v2.value.ullVal)
    except Exception as e:
        print("field", f, "exc", e)
for name in ("nvmlDeviceGetNvLinkUtilizationCounter",):
    try:
        ctrl = N.c_nvmlNvLinkUtilizationControl_t()
        ctrl.units = N.NVML_NVLINK_COUNTER_UNIT_BYTES
        ctrl.pktfilter = N.NVML_NVLINK_COUNTER_PKTFILTER_ALL
        for l in links:
            N.nvmlDeviceSetNvLinkUtilizationControl(h, l, 0, ctrl, True)
        print("util control set")
    except Exception as e:
        print("set util control exc", e)
    try:
        print("util counter link0", N.nvmlDeviceGetNvLinkUtilizationCounter(h, links[0], 0))
    except Exception as e:
        print("util counter exc", e)
# traffic: 2 GB GPU0 -> GPU1
a = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:0")
b = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:1")
def snap():
    out = {}
    for f in (138, 139, 202, 204):
        vals = N.nvmlDeviceGetFieldValues(h, [(f, l) for l in links])
        out[f] = sum(v.value.ullVal for v in vals if v.nvmlReturn == 0), sum(v.nvmlReturn != 0 for v in vals)
    try:
        out["util"] = sum(N.nvmlDeviceGetNvLinkUtilizationCounter(h, l, 0)[1] for l in links)
    except Exception as e:
        out["util"] = str(e)
    return out
s0 = snap()
for _ in range(4):
    b.copy_(a)
torch.cuda.synchronize()
s1 = snap()
print("before", s0)
print("after ", s1)
print(subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", "0"], capture_output=True, text=True).stdout[:800])
print(subprocess.run(["nvidia-smi", "nvlink", "-s", "-i", "0"], capture_output=True, text=True).stdout[:600])
