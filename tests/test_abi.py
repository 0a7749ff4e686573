"""CPU checks of the boundary: libtrail.so builds for sm_100a, loads without a GPU,
exports every symbol include/trail.h declares, and rejects invalid configurations on the
host before touching CUDA.  The binding fails loudly when the library is missing."""
import ctypes
import math
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2410_01035_b200 import _build
from paper_2410_01035_b200 import trail as T


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return T.load_library()


def declared_symbols():
    src = open(_build.HEADER).read()
    return sorted(set(re.findall(r"TRAIL_API\s+[\w\s\*]+?\b(trail_\w+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for name in ("trail_create", "trail_predict_step", "trail_schedule_step", "trail_destroy",
                 "trail_release", "trail_schedule_pack", "trail_schedule_select"):
        assert name in syms


def test_every_declared_symbol_is_exported(lib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", _build.LIB]).decode()
    exported = set(re.findall(r"\bT (trail_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    for s in declared_symbols():
        getattr(lib, s)


def test_built_for_sm100a_only(lib):
    out = subprocess.check_output(["cuobjdump", "--list-elf", _build.LIB]).decode()
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_sass_uses_tcgen05_and_tma(lib):
    sass = subprocess.check_output(["cuobjdump", "-sass", _build.LIB]).decode()
    assert "UTCHMMA" in sass          # tcgen05.mma
    assert "UTMALDG" in sass          # cp.async.bulk.tensor (TMA)
    assert "LDTM" in sass             # tcgen05.ld


def test_abi_version_and_status_strings(lib):
    assert T.trail_abi_version() == 1
    assert lib.trail_status_string(-1) == b"invalid argument"
    assert lib.trail_status_string(1).startswith(b"forced set")


def _cfg(**over):
    k = 10
    edges = np.array([512.0 * i / k for i in range(k + 1)])
    W1 = np.zeros((512, 4096), np.uint16)
    b1 = np.zeros(512, np.float32)
    W2 = np.zeros((k, 512), np.float32)
    b2 = np.zeros(k, np.float32)
    keep = [edges, W1, b1, W2, b2]
    base = dict(d=4096, hidden=512, k=k, dtype=T.TRAIL_BF16, w1=W1.ctypes.data, b1=b1.ctypes.data,
                w2=W2.ctypes.data, b2=b2.ctypes.data, bin_edges=edges.ctypes.data, prior=None,
                c=0.8, max_slots=16, max_requests=16, max_sched=16, world_size=1, id_base=0,
                device=0, l1_mode=0)
    base.update(over)
    return T.trail_config(**base), keep


@pytest.mark.parametrize("over", [
    dict(k=0), dict(k=33), dict(hidden=500), dict(hidden=640), dict(d=100), dict(dtype=7),
    dict(c=-0.5), dict(c=math.nan), dict(max_slots=0), dict(max_requests=0),
    dict(world_size=0), dict(l1_mode=6), dict(l1_mode=-1), dict(w1=None),
])
def test_invalid_configs_rejected_on_host(lib, over):
    cfg, keep = _cfg(**over)
    h = ctypes.c_void_p()
    assert lib.trail_create(ctypes.byref(cfg), ctypes.byref(h)) == T.TRAIL_ERR_INVALID
    assert not h.value


@pytest.mark.parametrize("l1_mode", [T.TRAIL_L1_TF32])
def test_tf32_mode_needs_fp32(lib, l1_mode):
    """TRAIL_L1_TF32 (the 3xTF32 tensor-core layer 1) exists for fp32 handles only."""
    cfg, keep = _cfg(l1_mode=l1_mode)            # a bf16 handle
    h = ctypes.c_void_p()
    assert lib.trail_create(ctypes.byref(cfg), ctypes.byref(h)) == T.TRAIL_ERR_UNSUPPORTED
    assert not h.value


def test_bad_edges_and_prior_rejected(lib):
    for edges in ([0.0, 0.5, 1.0], [0.0, 10.0, 5.0], [-1.0, 10.0, 20.0]):
        e = np.array(edges)
        cfg, keep = _cfg(k=2, bin_edges=e.ctypes.data)
        h = ctypes.c_void_p()
        assert lib.trail_create(ctypes.byref(cfg), ctypes.byref(h)) == T.TRAIL_ERR_INVALID
    pr = np.full(10, 0.2)
    cfg, keep = _cfg(prior=pr.ctypes.data)
    h = ctypes.c_void_p()
    assert lib.trail_create(ctypes.byref(cfg), ctypes.byref(h)) == T.TRAIL_ERR_INVALID


def test_null_handle_calls_are_invalid(lib):
    assert lib.trail_predict_step(None, None, 0, None, None, None, None, 1, None, None, None) == -1
    assert lib.trail_schedule_step(None, None, None, None, None, 0, 0, 0, None, None, None, None,
                                   None) == -1
    assert lib.trail_time_update(None, None, 1, 1, None, None, None) == -1
    assert lib.trail_set_rows_hint(None, 0) == -1
    assert lib.trail_set_threshold_mode(None, 1) == -1
    assert lib.trail_prefill_chunk(None, None, 0, None, None, None, 1, None, 0, None) == -1
    assert lib.trail_destroy(None) == -1


def test_binding_fails_loudly_without_library(monkeypatch, tmp_path):
    monkeypatch.setattr(T, "_LIB", None)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        T.load_library(str(tmp_path / "missing.so"))
