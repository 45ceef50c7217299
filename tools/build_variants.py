"""Build A/B variants of the library (timing probes NIMG_BWD_PROBE, tile configurations) next
to the default one; tools/gpu_bwd_probe.sh times each with bench.py (A/B only: probe results are wrong)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2604_12163_b200 import _build  # noqa: E402

VARIANTS = {"probe1": ("NIMG_BWD_PROBE=1",), "probe2": ("NIMG_BWD_PROBE=2",), "staged": ("NIMG_W_SECTOR=0",), "st128": ("NIMG_ST256=0",), "cbminb1": ("NIMG_CB_MINB=1",), "d2nostage": ("NIMG_D2_HSTAGE=0",), "cbb4m4": ("NIMG_CB_BATCH=4", "NIMG_CB_MINB=4"),
            "g1bn112": ("NIMG_G1_BN=112",), "b128": ("NIMG_I8_B256=0",),
            "trace": ("NIMG_I8_TRACE=1",), "trace_nomma": ("NIMG_I8_TRACE=1", "NIMG_I8_PROBE=2"),
            "trace_noconv": ("NIMG_I8_TRACE=1", "NIMG_I8_PROBE=1"), "lx3": ("NIMG_I8_LX=3",),
            "lx3_trace": ("NIMG_I8_LX=3", "NIMG_I8_TRACE=1"),
            "kb128": ("NIMG_I8_KB=128",), "intconv": ("NIMG_I8_FCONV=0",), "noconv": ("NIMG_I8_PROBE=1",),
            "nomma": ("NIMG_I8_PROBE=2",), "noepi": ("NIMG_I8_PROBE=3",)}
for tag in (sys.argv[1:] or VARIANTS):
    defs = VARIANTS[tag]
    out = os.path.join(os.path.dirname(_build.LIB), f"libnimg_moe_{tag}.so")
    print(_build.build(out=out, defines=defs))
