"""NVLink traffic counters (NVML) for the expert-parallel exchange.

The copy-engine exchange (ep.py) moves its chunks with cudaMemcpyAsync over
NVLink, so no kernel carries the traffic and ncu cannot attribute it. NVML's
per-link hardware counters can: `NvLinkCounters(dev)` snapshots the device's
transmitted / received data bytes summed over its active links, and the
difference of two snapshots around a timed region gives the bytes the GPU put
on (and took off) NVLink in that region. Instrumentation only -- nothing on
the data path depends on it; if NVML or the counters are unavailable the
snapshot is None.

Fields (nvml.h): NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX (138 / 139, KiB,
data payload) and NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES / RCV_BYTES (202 / 204,
bytes), per link (scopeId = link index); whichever the driver supports.
"""

from __future__ import annotations

import time

_FIELDS = ((138, 139, 1024), (202, 204, 1))   # (tx, rx, bytes per unit)
_MAX_LINKS = 18


class NvLinkCounters:
    def __init__(self, device_index: int):
        self.ok = False
        self.err = None
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(device_index)
            self.links = []
            for l in range(_MAX_LINKS):
                try:
                    if N.nvmlDeviceGetNvLinkState(self.h, l) == N.NVML_FEATURE_ENABLED:
                        self.links.append(l)
                except N.NVMLError:
                    break
            self.field = None
            for tx, rx, unit in _FIELDS:
                vals = self._read(tx, rx)
                if vals is not None:
                    self.field = (tx, rx, unit)
                    break
            self.ok = self.field is not None and bool(self.links)
            if not self.ok:
                self.err = f"no NVLink counter field readable on {len(self.links)} active links"
        except Exception as e:  # NVML absent / no permission: instrumentation is optional
            self.err = f"{type(e).__name__}: {e}"

    def _read(self, tx, rx):
        N = self.N
        req = [(f, l) for l in self.links for f in (tx, rx)]
        if not req:
            return None
        try:
            vals = N.nvmlDeviceGetFieldValues(self.h, req)
        except N.NVMLError:
            return None
        t = r = 0
        for i, v in enumerate(vals):
            if v.nvmlReturn != 0:
                return None
            x = v.value.ullVal if v.valueType == N.NVML_VALUE_TYPE_UNSIGNED_LONG_LONG else v.value.ulVal
            if i % 2 == 0:
                t += x
            else:
                r += x
        return t, r

    def snapshot(self):
        """(time_s, tx_bytes, rx_bytes) summed over the active links, or None."""
        if not self.ok:
            return None
        v = self._read(self.field[0], self.field[1])
        if v is None:
            return None
        return (time.perf_counter(), v[0] * self.field[2], v[1] * self.field[2])

    @staticmethod
    def delta(a, b, device_seconds: float | None = None) -> dict | None:
        """Bytes moved between two snapshots; GB/s over `device_seconds` (the
        CUDA-event time of the region) or, failing that, the host interval."""
        if a is None or b is None:
            return None
        secs = device_seconds if device_seconds else (b[0] - a[0])
        tx, rx = b[1] - a[1], b[2] - a[2]
        return {"tx_bytes": tx, "rx_bytes": rx, "seconds": secs,
                "tx_gbs": tx / secs / 1e9 if secs > 0 else None,
                "rx_gbs": rx / secs / 1e9 if secs > 0 else None}
