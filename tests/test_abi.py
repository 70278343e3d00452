"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every
entry point include/lc_b200.h declares, and the ctypes layouts match the
header's structs.  No compute calls (there is no GPU in the build container).
"""

from __future__ import annotations

import ctypes as C
import os
import re
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lc_b200.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|int64_t|const char\*)\s+(lc_[a-z0-9_]+)\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2604_17353_b200 import _capi

    lib = C.CDLL(_capi.LIB_PATH)
    missing = [s for s in _declared() if not hasattr(lib, s)]
    assert not missing, missing
    assert len(_declared()) >= 25
    # every declared symbol is also bound with a signature in the ctypes layer
    assert set(_declared()) <= set(_capi._SIGS), set(_declared()) - set(_capi._SIGS)


def test_exports_are_exactly_the_header(tmp_path):
    from paper_2604_17353_b200 import _capi

    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True, text=True).stdout
    exported = sorted({ln.split()[-1] for ln in out.splitlines() if re.search(r" T lc_", ln)})
    assert exported == _declared()


def test_abi_version_and_status_strings():
    from paper_2604_17353_b200 import _capi

    assert _capi.lib.lc_abi_version() == 5
    assert _capi.lib.lc_status_string(6) == b"write-back prefix no longer live"
    assert _capi.lib.lc_status_string(0) == b"ok"
    assert _capi.lib.lc_status_string(1) == b"config error"


def test_struct_layouts_match_header():
    from paper_2604_17353_b200 import _capi

    assert C.sizeof(_capi.LcTask) == 72 == _capi.TASK_DTYPE.itemsize
    assert C.sizeof(_capi.LcDraws) == 64
    assert C.sizeof(_capi.LcCacheConfig) == 48
    assert C.sizeof(_capi.LcCacheStats) == 11 * 8
    src = open(HEADER).read()
    body = src[src.index("typedef struct lc_task {"): src.index("} lc_task;")]
    fields = re.findall(r"^\s+\w+_t\s+(\w+);|^\s+double\s+(\w+);", body, re.M)
    names = [a or b for a, b in fields]
    assert names == [f[0] for f in _capi.LcTask._fields_]
    body = src[src.index("typedef struct lc_decode_step {"): src.index("} lc_decode_step;")]
    names = re.findall(r"^\s+(?:const\s+)?\w+\*?\s+\*?(\w+);", body, re.M)
    assert names == [f[0] for f in _capi.LcDecodeStep._fields_]
    assert C.sizeof(_capi.LcDecodeStep) == 8 + 4 * 4 + 8 * 3 + 8 * 13


def test_workspace_query_needs_no_gpu():
    from paper_2604_17353_b200 import _capi

    b = _capi.lib.lc_resample_workspace_bytes(1024, 32000)
    assert b > 1024 * 8


def test_argument_validation_without_gpu():
    """Entry points reject bad arguments before touching the device."""
    from paper_2604_17353_b200 import _capi

    assert _capi.lib.lc_hash_prefix(None, None, None, -1, None, None) == _capi.LC_E_ARG
    assert _capi.lib.lc_uniforms(None, None, 5, None, None) == _capi.LC_E_ARG
    assert _capi.lib.lc_hash_prefix(None, None, None, 0, None, None) == _capi.LC_OK
    cfg = _capi.LcCacheConfig(0, 0, 1, 1, 1, 1, 0, 0)  # vocab 0 is invalid
    h = C.c_void_p()
    assert _capi.lib.lc_cache_create(C.byref(cfg), C.byref(h)) == _capi.LC_E_CONFIG


def test_make_tasks_layout():
    import paper_2604_17353_b200 as lcb

    t = lcb.make_tasks(row=np.arange(3), temperature=0.6, top_k=None, top_p=0.9)
    assert t.dtype.itemsize == 72
    assert t["draw_end"].tolist() == [1, 2, 3] and t["top_k"].tolist() == [0, 0, 0]
    raw = t.view(np.uint8).reshape(3, 72)
    assert np.frombuffer(raw[1, 0:8].tobytes(), "<i8")[0] == 1
