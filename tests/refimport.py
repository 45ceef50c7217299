"""Import the read-only reference package under the alias ``nimg_ref``.

Location: $NIMG_REF, else /root/reference/pkg/src/nimg (build container),
else the offline pip install of the reference under baseline/_ref/nimg (the
one copy that travels to the GPU box; git-ignored, built by
`pip install --no-index --target baseline/_ref`).
"""

from __future__ import annotations

import importlib.util
import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_CANDIDATES = [os.environ.get("NIMG_REF"), "/root/reference/pkg/src/nimg",
               os.path.join(_ROOT, "baseline", "_ref", "nimg")]
REF_DIR = next((c for c in _CANDIDATES if c and os.path.isfile(os.path.join(c, "__init__.py"))),
               _CANDIDATES[1])


def reference_available() -> bool:
    return os.path.isfile(os.path.join(REF_DIR, "__init__.py"))


def load_reference():
    """Return the reference package (modules: tensor, router, moe)."""
    if "nimg_ref" in sys.modules:
        return sys.modules["nimg_ref"]
    sys.dont_write_bytecode = True  # the tree is read-only
    spec = importlib.util.spec_from_file_location(
        "nimg_ref", os.path.join(REF_DIR, "__init__.py"),
        submodule_search_locations=[REF_DIR])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["nimg_ref"] = mod
    spec.loader.exec_module(mod)
    import importlib as il
    for sub in ("tensor", "router", "moe", "backbone"):
        setattr(mod, sub, il.import_module(f"nimg_ref.{sub}"))
    return mod
