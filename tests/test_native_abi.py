"""The C ABI library loads and exports every symbol include/wfst_b200.h declares (CPU-only:
no compute calls), and the host shim maps status codes to the reference's exceptions."""
import ctypes
import os
import re

import pytest

from paper_1808_00687_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "wfst_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(wb_\w+)\s*\(", text, re.M)))


def test_header_declares_the_abi():
    names = declared_functions()
    assert set(names) == set(N.EXPORTED), names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(N.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_library_is_sm100a():
    """The shared library carries sm_100a SASS (cross-compiled here, run on the B200)."""
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "--list-elf", N.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_version_and_error_string():
    lib = N.load()
    assert lib.wb_version() >= 1
    assert isinstance(lib.wb_last_error(), bytes)


def test_status_mapping():
    from paper_1808_00687_b200.lattice import LatticeError
    from paper_1808_00687_b200.wfst import WfstError
    N.check(N.WB_OK)
    with pytest.raises(ValueError):
        N.check(N.WB_ERR_VALUE)
    with pytest.raises(WfstError):
        N.check(N.WB_ERR_WFST)
    with pytest.raises(LatticeError):
        N.check(N.WB_ERR_LATTICE)
    with pytest.raises(N.CapacityError):
        N.check(N.WB_ERR_CAPACITY)
    with pytest.raises(N.NativeError):
        N.check(N.WB_ERR_CUDA)


def test_utt_result_layout_matches_header():
    """numpy record layout == sizeof(wb_utt_result) in the header (8-byte aligned fields)."""
    text = open(HEADER).read()
    body = text[text.index("typedef struct {\n    double total_cost;"):]
    body = body[:body.index("} wb_utt_result;")]
    fields = re.findall(r"^\s*(double|int64_t|int32_t)\s+(\w+)(?:\[(\d+)\])?;", body, re.M)
    assert [f[1] for f in fields] == list(N.UTT_RESULT_DTYPE.names)
    size = {"double": 8, "int64_t": 8, "int32_t": 4}
    assert sum(size[t] * int(n or 1) for t, _, n in fields) == N.UTT_RESULT_DTYPE.itemsize
