"""Thin ctypes binding of libtrail.so (include/trail.h).  Argument marshalling only: every
step of the predict+schedule path runs in the CUDA kernels behind the C ABI.  There is no
CPU fallback — if the shared library is missing this module raises on import of the
library (`load_library`).

Functions keep the C names (`trail_create`, `trail_predict_step`, ...) and accept torch
tensors (device memory) or raw integer device pointers; `stream` defaults to torch's
current CUDA stream.  `Trail` is a small convenience wrapper that owns a handle.
"""
from __future__ import annotations

import ctypes
import math
import os
from typing import Optional

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libtrail.so")

TRAIL_OK = 0
TRAIL_WARN_OVER_BUDGET = 1
TRAIL_ERR_INVALID = -1
TRAIL_ERR_CUDA = -2
TRAIL_ERR_NOMEM = -3
TRAIL_ERR_CAPACITY = -4
TRAIL_ERR_NCCL = -5
TRAIL_ERR_STATE = -6
TRAIL_ERR_UNSUPPORTED = -7

TRAIL_F32, TRAIL_BF16 = 0, 1
(TRAIL_L1_AUTO, TRAIL_L1_GEMV, TRAIL_L1_UMMA, TRAIL_L1_UMMA_UNFUSED, TRAIL_L1_WIDE,
 TRAIL_L1_TF32) = 0, 1, 2, 3, 4, 5
TRAIL_K = {"pool": 0, "gemv": 1, "umma": 2, "head": 3, "pack": 4, "select": 5, "gather": 6}
TRAIL_DEV_BAD_ID, TRAIL_DEV_BAD_ROWS, TRAIL_DEV_NEG_KV, TRAIL_DEV_NONFIN = 1, 2, 4, 8
RECORD_BYTES = 16


class TrailError(RuntimeError):
    def __init__(self, fn: str, status: int):
        msg = _lib().trail_status_string(status).decode() if _LIB is not None else str(status)
        super().__init__(f"{fn} -> {status} ({msg})")
        self.status = status


class trail_config(ctypes.Structure):
    _fields_ = [
        ("d", ctypes.c_int32), ("hidden", ctypes.c_int32), ("k", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("w1", ctypes.c_void_p), ("b1", ctypes.c_void_p), ("w2", ctypes.c_void_p),
        ("b2", ctypes.c_void_p), ("bin_edges", ctypes.c_void_p), ("prior", ctypes.c_void_p),
        ("c", ctypes.c_double),
        ("max_slots", ctypes.c_int32), ("max_requests", ctypes.c_int32),
        ("max_sched", ctypes.c_int32), ("world_size", ctypes.c_int32),
        ("id_base", ctypes.c_uint32), ("device", ctypes.c_int32), ("l1_mode", ctypes.c_int32),
    ]


_LIB: Optional[ctypes.CDLL] = None

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_SIGS = {
    "trail_abi_version": ([], _I32),
    "trail_status_string": ([_I32], ctypes.c_char_p),
    "trail_create": ([ctypes.POINTER(trail_config), ctypes.POINTER(_P)], _I32),
    "trail_destroy": ([_P], _I32),
    "trail_predict_step": ([_P, _P, _I64, _P, _P, _P, _P, _I32, _P, _P, _P], _I32),
    "trail_predict_step_layers": ([_P, _P, _P, _I32, _I64, _P, _P, _P, _P, _I32, _P, _P, _P],
                                  _I32),
    "trail_schedule_step": ([_P, _P, _P, _P, _P, _I32, _I64, _I32, _P, _P, _P, _P, _P], _I32),
    "trail_schedule_pack": ([_P, _P, _P, _P, _P, _I32, _I32, _P, _P], _I32),
    "trail_schedule_select": ([_P, _P, _I32, _I64, _I32, _P, _P, _P, _P, _P], _I32),
    "trail_release": ([_P, _P, _I32, _P], _I32),
    "trail_read_state": ([_P, _P, _I32, _P, _P, _P, _P, _P, _P], _I32),
    "trail_nccl_unique_id": ([_P], _I32),
    "trail_comm_init": ([_P, _P, _I32, _I32], _I32),
    "trail_device_errors": ([_P, ctypes.POINTER(ctypes.c_uint32), _I32], _I32),
    "trail_profile_enable": ([_P, _I32], _I32),
    "trail_profile_read": ([_P, _I32, ctypes.POINTER(ctypes.c_double),
                            ctypes.POINTER(ctypes.c_int64), _I32], _I32),
    "trail_set_l1_mode": ([_P, _I32], _I32),
    "trail_set_rows_hint": ([_P, _I64], _I32),
    "trail_time_update": ([_P, _P, _I32, _I32, _P, _P, _P], _I32),
    "trail_prefill_chunk": ([_P, _P, _I64, _P, _P, _P, _I32, _P, _I64, _P], _I32),
    "trail_set_threshold_mode": ([_P, _I32], _I32),
    "trail_set_fill_mode": ([_P, _I32], _I32),
    "trail_set_w1_l2_persist": ([_P, _I32], _I32),
    "trail_set_prefill_start": ([_P, _I32], _I32),
    "trail_trace_enable": ([_P, _I32], _I32),
    "trail_trace_read": ([_P, _P, _I32], _I32),
    "trail_plan_l1": ([_P, _I32, ctypes.POINTER(_I32), ctypes.POINTER(_I32)], _I32),
}


def load_library(path: Optional[str] = None) -> ctypes.CDLL:
    """Load libtrail.so (fails loudly if it has not been built)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    p = path or os.environ.get("TRAIL_LIB", LIB_PATH)
    if not os.path.exists(p):
        raise RuntimeError(f"libtrail.so not found at {p}; run __graft_entry__.build() "
                           "(there is no CPU fallback)")
    lib = ctypes.CDLL(p)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _LIB = lib
    return lib


def _lib() -> ctypes.CDLL:
    return _LIB if _LIB is not None else load_library()


def _ptr(x) -> Optional[int]:
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        if not x.is_cuda:
            raise ValueError("device tensor expected")
        if not x.is_contiguous():
            raise ValueError("contiguous tensor expected")
        return x.data_ptr()
    raise TypeError(type(x))


def _stream(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _check(fn: str, st: int, allow_warn: bool = False) -> int:
    if st < 0 or (st > 0 and not allow_warn):
        raise TrailError(fn, st)
    return st


# ------------------------------------------------------------------ C-named functions
def trail_abi_version() -> int:
    return _lib().trail_abi_version()


def trail_create(cfg: trail_config) -> int:
    h = ctypes.c_void_p()
    _check("trail_create", _lib().trail_create(ctypes.byref(cfg), ctypes.byref(h)))
    return h.value


def trail_destroy(h: int) -> None:
    _check("trail_destroy", _lib().trail_destroy(h))


def trail_predict_step(h, emb, emb_ld, row_offsets, request_ids, is_prefill, prior_override,
                       n, posteriors, expected_remaining, stream=None) -> int:
    return _check("trail_predict_step", _lib().trail_predict_step(
        h, _ptr(emb), int(emb_ld), _ptr(row_offsets), _ptr(request_ids), _ptr(is_prefill),
        _ptr(prior_override), int(n), _ptr(posteriors), _ptr(expected_remaining),
        _stream(stream)))


def trail_predict_step_layers(h, embs, layer_weights, emb_ld, row_offsets, request_ids,
                              is_prefill, prior_override, n, posteriors, expected_remaining,
                              stream=None) -> int:
    """Multi-layer weighted embeddings (D-28): `embs` a list of device tensors / pointers,
    `layer_weights` host floats; marshalled into the (host) pointer and weight arrays."""
    L = len(embs)
    ptrs = (ctypes.c_void_p * L)(*[_ptr(e) for e in embs])
    ws = (ctypes.c_float * L)(*[float(x) for x in layer_weights])
    return _check("trail_predict_step_layers", _lib().trail_predict_step_layers(
        h, ctypes.cast(ptrs, ctypes.c_void_p), ctypes.cast(ws, ctypes.c_void_p), L, int(emb_ld),
        _ptr(row_offsets), _ptr(request_ids), _ptr(is_prefill), _ptr(prior_override), int(n),
        _ptr(posteriors), _ptr(expected_remaining), _stream(stream)))


def trail_set_prefill_start(h, first_prefill: int) -> int:
    """Host hint: requests before `first_prefill` are single-row decodes (-1 = unknown)."""
    return _check("trail_set_prefill_start", _lib().trail_set_prefill_start(h, int(first_prefill)))


def trail_set_w1_l2_persist(h, enable: int) -> int:
    """L2-persisting W1 for the layer-1 kernels (device-wide set-aside)."""
    return _check("trail_set_w1_l2_persist", _lib().trail_set_w1_l2_persist(h, int(enable)))


def trail_set_fill_mode(h, mode: int) -> int:
    """0 = strict prefix (D-15), 1 = first-fit."""
    return _check("trail_set_fill_mode", _lib().trail_set_fill_mode(h, int(mode)))


def trail_schedule_step(h, request_ids, arrival_seq, kv_blocks, is_running, n, kv_budget,
                        max_run, run_ids, preempt_ids, admit_ids, counts, stream=None) -> int:
    return _check("trail_schedule_step", _lib().trail_schedule_step(
        h, _ptr(request_ids), _ptr(arrival_seq), _ptr(kv_blocks), _ptr(is_running), int(n),
        int(kv_budget), int(max_run), _ptr(run_ids), _ptr(preempt_ids), _ptr(admit_ids),
        _ptr(counts), _stream(stream)))


def trail_schedule_pack(h, request_ids, arrival_seq, kv_blocks, is_running, n, capacity,
                        records, stream=None) -> int:
    return _check("trail_schedule_pack", _lib().trail_schedule_pack(
        h, _ptr(request_ids), _ptr(arrival_seq), _ptr(kv_blocks), _ptr(is_running), int(n),
        int(capacity), _ptr(records), _stream(stream)))


def trail_schedule_select(h, records, n_records, kv_budget, max_run, run_ids, preempt_ids,
                          admit_ids, counts, stream=None) -> int:
    return _check("trail_schedule_select", _lib().trail_schedule_select(
        h, _ptr(records), int(n_records), int(kv_budget), int(max_run), _ptr(run_ids),
        _ptr(preempt_ids), _ptr(admit_ids), _ptr(counts), _stream(stream)))


def trail_release(h, request_ids, n, stream=None) -> int:
    return _check("trail_release", _lib().trail_release(h, _ptr(request_ids), int(n),
                                                        _stream(stream)))


def trail_read_state(h, request_ids, n, L=None, age=None, threshold=None, seen=None,
                     posterior=None, stream=None) -> int:
    return _check("trail_read_state", _lib().trail_read_state(
        h, _ptr(request_ids), int(n), _ptr(L), _ptr(age), _ptr(threshold), _ptr(seen),
        _ptr(posterior), _stream(stream)))


def trail_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check("trail_nccl_unique_id", _lib().trail_nccl_unique_id(buf))
    return buf.raw


def trail_comm_init(h, uid: bytes, rank: int, world_size: int) -> int:
    buf = ctypes.create_string_buffer(bytes(uid), 128)
    return _check("trail_comm_init", _lib().trail_comm_init(h, buf, int(rank), int(world_size)))


def trail_device_errors(h, clear: bool = False) -> int:
    bits = ctypes.c_uint32(0)
    _check("trail_device_errors", _lib().trail_device_errors(h, ctypes.byref(bits), int(clear)))
    return int(bits.value)


def trail_profile_enable(h, enable: bool = True) -> None:
    _check("trail_profile_enable", _lib().trail_profile_enable(h, int(enable)))


def trail_profile_read(h, kernel: str, reset: bool = False):
    ms = ctypes.c_double(0.0)
    cnt = ctypes.c_int64(0)
    _check("trail_profile_read", _lib().trail_profile_read(h, TRAIL_K[kernel], ctypes.byref(ms),
                                                           ctypes.byref(cnt), int(reset)))
    return float(ms.value), int(cnt.value)


def trail_trace_enable(h, max_ctas: int) -> None:
    _check("trail_trace_enable", _lib().trail_trace_enable(h, int(max_ctas)))


def trail_trace_read(h, max_ctas: int) -> np.ndarray:
    out = np.zeros((int(max_ctas), 16), dtype=np.uint64)
    _check("trail_trace_read", _lib().trail_trace_read(h, out.ctypes.data, int(max_ctas)))
    return out


def trail_set_l1_mode(h, mode: int) -> None:
    _check("trail_set_l1_mode", _lib().trail_set_l1_mode(h, int(mode)))


def trail_time_update(h, request_ids, n: int, steps: int, posteriors, expected_remaining,
                      stream=None) -> None:
    _check("trail_time_update", _lib().trail_time_update(
        h, _ptr(request_ids), int(n), int(steps), _ptr(posteriors), _ptr(expected_remaining),
        _stream(stream)))


def trail_prefill_chunk(h, emb, emb_ld: int, row_offsets, request_ids, is_final, n: int,
                        pooled, pooled_ld: int, stream=None) -> None:
    _check("trail_prefill_chunk", _lib().trail_prefill_chunk(
        h, _ptr(emb), int(emb_ld), _ptr(row_offsets), _ptr(request_ids), _ptr(is_final), int(n),
        _ptr(pooled), int(pooled_ld), _stream(stream)))


def trail_set_threshold_mode(h, mode: int) -> None:
    _check("trail_set_threshold_mode", _lib().trail_set_threshold_mode(h, int(mode)))


def trail_set_rows_hint(h, rows: int) -> None:
    _check("trail_set_rows_hint", _lib().trail_set_rows_hint(h, int(rows)))


def trail_plan_l1(h, n: int):
    mode, splits = _I32(0), _I32(0)
    _check("trail_plan_l1", _lib().trail_plan_l1(h, int(n), ctypes.byref(mode), ctypes.byref(splits)))
    return int(mode.value), int(splits.value)


# ------------------------------------------------------------------ convenience wrapper
class Trail:
    """Owns one handle plus preallocated device outputs.

    weights: dict with W1 ([H][d] float32, or uint16 bf16 bits), b1, W2, b2 (float32) and
    'edges' (float64 [k+1]); dtype 'bf16' or 'f32'."""

    def __init__(self, weights: dict, c: float, max_slots: int, max_requests: int,
                 max_sched: int, dtype: str = "bf16", prior=None, device: int = 0,
                 world_size: int = 1, id_base: int = 0, l1_mode: int = TRAIL_L1_AUTO):
        import torch
        self.torch = torch
        W1 = np.ascontiguousarray(weights["W1"])
        H, d = W1.shape
        edges = np.ascontiguousarray(weights["edges"], dtype=np.float64)
        k = edges.shape[0] - 1
        self.d, self.H, self.k, self.dtype = d, H, k, dtype
        self.max_requests, self.max_sched, self.world = max_requests, max_sched, world_size
        self._keep = [W1, np.ascontiguousarray(weights["b1"], np.float32),
                      np.ascontiguousarray(weights["W2"], np.float32),
                      np.ascontiguousarray(weights["b2"], np.float32), edges]
        pr = None
        if prior is not None:
            pr = np.ascontiguousarray(prior, np.float64)
            self._keep.append(pr)
        cfg = trail_config(
            d=d, hidden=H, k=k, dtype=TRAIL_BF16 if dtype == "bf16" else TRAIL_F32,
            w1=self._keep[0].ctypes.data, b1=self._keep[1].ctypes.data,
            w2=self._keep[2].ctypes.data, b2=self._keep[3].ctypes.data,
            bin_edges=edges.ctypes.data, prior=(pr.ctypes.data if pr is not None else None),
            c=float(c) if not math.isinf(c) else math.inf,
            max_slots=max_slots, max_requests=max_requests, max_sched=max_sched,
            world_size=world_size, id_base=id_base, device=device, l1_mode=l1_mode)
        self.device = torch.device("cuda", device)
        self.h = trail_create(cfg)
        cap = max(1, max_sched) * world_size
        dev = self.device
        self.post = torch.empty((max_requests, k), dtype=torch.float32, device=dev)
        self.L = torch.empty((max_requests,), dtype=torch.float32, device=dev)
        self.run_ids = torch.empty((cap,), dtype=torch.int32, device=dev)
        self.preempt_ids = torch.empty((cap,), dtype=torch.int32, device=dev)
        self.admit_ids = torch.empty((cap,), dtype=torch.int32, device=dev)
        self.counts = torch.zeros((4,), dtype=torch.int32, device=dev)

    def close(self):
        if getattr(self, "h", None):
            trail_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def predict(self, emb, row_offsets, request_ids, is_prefill, prior_override=None,
                stream=None, rows=None, prefill_start=None):
        n = int(request_ids.shape[0])
        # host-side row count of the flat batch (selects the pooling kernel variant only)
        rows = int(emb.shape[0]) if rows is None and emb.dim() == 2 else int(rows or 0)
        if rows != getattr(self, "_rows_hint", 0):
            trail_set_rows_hint(self.h, rows)
            self._rows_hint = rows
        # host-side batch layout: index of the first multi-row (prefill) request, if known
        pfs = -1 if prefill_start is None else int(prefill_start)
        if pfs != getattr(self, "_prefill_start", -1):
            trail_set_prefill_start(self.h, pfs)
            self._prefill_start = pfs
        trail_predict_step(self.h, emb, emb.shape[1] if emb.dim() == 2 else self.d, row_offsets,
                           request_ids, is_prefill, prior_override, n, self.post, self.L, stream)
        return self.post[:n], self.L[:n]

    def predict_layers(self, embs, layer_weights, row_offsets, request_ids, is_prefill,
                       prior_override=None, stream=None):
        """Probe on the weighted average of several layers' embeddings."""
        n = int(request_ids.shape[0])
        ld = embs[0].shape[1] if embs[0].dim() == 2 else self.d
        trail_predict_step_layers(self.h, embs, layer_weights, ld, row_offsets, request_ids,
                                  is_prefill, prior_override, n, self.post, self.L, stream)
        return self.post[:n], self.L[:n]

    def time_update(self, request_ids, steps: int, stream=None):
        """Iterations without an observation (predict every K iterations)."""
        n = int(request_ids.shape[0])
        trail_time_update(self.h, request_ids, n, steps, self.post, self.L, stream)
        return self.post[:n], self.L[:n]

    def schedule(self, request_ids, arrival_seq, kv_blocks, is_running, kv_budget: int,
                 max_run: int = 0, stream=None):
        n = int(request_ids.shape[0])
        trail_schedule_step(self.h, request_ids, arrival_seq, kv_blocks, is_running, n,
                            kv_budget, max_run, self.run_ids, self.preempt_ids, self.admit_ids,
                            self.counts, stream)
        return self.run_ids, self.preempt_ids, self.admit_ids, self.counts

    def read_state(self, request_ids):
        torch = self.torch
        n = int(request_ids.shape[0])
        dev = self.device
        L = torch.empty(n, dtype=torch.float32, device=dev)
        age = torch.empty(n, dtype=torch.int32, device=dev)
        thr = torch.empty(n, dtype=torch.int32, device=dev)
        seen = torch.empty(n, dtype=torch.uint8, device=dev)
        post = torch.empty((n, self.k), dtype=torch.float32, device=dev)
        trail_read_state(self.h, request_ids, n, L, age, thr, seen, post)
        return {"L": L, "age": age, "thr": thr, "seen": seen, "post": post}

    def release(self, request_ids, stream=None):
        trail_release(self.h, request_ids, int(request_ids.shape[0]), stream)
