"""TEST INFRASTRUCTURE ONLY — ctypes front-end for oracle/mg1_des.c (M/G/1 DES of the
SPRPT-LP rank policy, App. C, App. D)."""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from typing import Dict

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mg1_des.c")
_BUILD = os.path.join(_HERE, "_build")
_LIB_PATH = os.path.join(_BUILD, "libmg1des.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile mg1_des.c with gcc (plain C, -O2).  Building the checker is not using it."""
    os.makedirs(_BUILD, exist_ok=True)
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-shared", "-fPIC", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            d = ctypes.POINTER(ctypes.c_double)
            lib.mg1_simulate.argtypes = [ctypes.c_int64, d, d, d, ctypes.c_double, ctypes.c_int,
                                         d, d, ctypes.POINTER(ctypes.c_int64), d]
            lib.mg1_simulate.restype = ctypes.c_int
            _lib = lib
    return _lib


def job_stream(n: int, lam: float, predictor: str, seed: int, burst: bool = False):
    """Poisson(lam) arrivals (or all at t=0 for the burst shape), Exp(1) sizes
    (App. D: f(x) = e^{-x}), predictions: 'perfect' r = x, or 'exponential' r ~ Exp(mean x)
    with g(x,y) = e^{-x} (1/x) e^{-y/x} (App. D P:953 with the typo fixed, reading D-19a)."""
    g = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 19, int(lam * 1e6)])))
    arrival = np.zeros(n) if burst else np.cumsum(g.exponential(1.0 / lam, n))
    size = g.exponential(1.0, n)
    if predictor == "perfect":
        pred = size.copy()
    elif predictor == "exponential":
        pred = g.exponential(1.0, n) * size
    else:
        raise ValueError(predictor)
    return arrival, size, pred


def simulate(arrival, size, pred, C: float, zero_plus: bool = False) -> Dict[str, np.ndarray]:
    lib = _load()
    n = int(arrival.shape[0])
    arrival = np.ascontiguousarray(arrival, dtype=np.float64)
    size = np.ascontiguousarray(size, dtype=np.float64)
    pred = np.ascontiguousarray(pred, dtype=np.float64)
    comp = np.empty(n)
    first = np.empty(n)
    npre = ctypes.c_int64(0)
    peak = ctypes.c_double(0.0)
    p = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))  # noqa: E731
    rc = lib.mg1_simulate(n, p(arrival), p(size), p(pred), float(C), int(zero_plus),
                          p(comp), p(first), ctypes.byref(npre), ctypes.byref(peak))
    if rc != 0:
        raise MemoryError("mg1_simulate")
    return {"completion": comp, "first_service": first, "response": comp - arrival,
            "preemptions": int(npre.value), "peak_memory": float(peak.value)}


def mean_response(n: int, lam: float, C: float, predictor: str, seed: int,
                  zero_plus: bool = False, warmup: float = 0.2, nbatch: int = 20):
    """Steady-state mean response time with a batch-means standard error (jobs after the
    first `warmup` fraction, in arrival order, split into `nbatch` batches)."""
    a, s, r = job_stream(n, lam, predictor, seed)
    out = simulate(a, s, r, C, zero_plus)
    resp = out["response"][int(warmup * n):]
    b = resp[: (resp.shape[0] // nbatch) * nbatch].reshape(nbatch, -1).mean(axis=1)
    return float(resp.mean()), float(b.std(ddof=1) / np.sqrt(nbatch)), out
