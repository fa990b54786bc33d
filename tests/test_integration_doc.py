"""The reference-side ctypes binding shown in INTEGRATION.md matches the library's layout
(CPU only: struct sizes and field names against include/wfst_b200.h and _native)."""
import os
import re

import numpy as np

from paper_1808_00687_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _stub_namespace():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = re.search(r"```python\n# lsd_wfst/b200.py.*?```", text, re.S).group(0)
    code = code.strip("`").split("\n", 1)[1]
    # keep the layout definitions only (the stub imports the reference package)
    keep = code.split("def upload")[0]
    keep = "\n".join(l for l in keep.splitlines()
                     if not l.startswith("from .") and "CDLL" not in l)
    ns = {}
    exec(keep, ns)
    return ns


def test_integration_stub_layouts_match_library():
    ns = _stub_namespace()
    assert ns["RESULT"].itemsize == N.UTT_RESULT_DTYPE.itemsize
    assert list(ns["RESULT"].names) == list(N.UTT_RESULT_DTYPE.names)
    import ctypes as C
    assert C.sizeof(ns["Config"]) == C.sizeof(N.Config)
    assert C.sizeof(ns["GraphDesc"]) == C.sizeof(N.GraphDesc)
