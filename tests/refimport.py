"""Import the read-only reference package under the alias ``nimg_ref``.

Only usable in the build container (the reference tree does not travel to
the GPU box). Location: $NIMG_REF, else /root/reference/pkg/src/nimg.
"""

from __future__ import annotations

import importlib.util
import os
import sys

REF_DIR = os.environ.get("NIMG_REF", "/root/reference/pkg/src/nimg")


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
