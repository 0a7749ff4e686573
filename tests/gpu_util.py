"""Helpers for the GPU parity tests: move synth inputs to the device, call the C ABI
through the binding, and compare against the fp64 oracle with the accuracy contract of
DESIGN.md §5 (posteriors 2e-3 abs, L 1e-3 rel, selection bit-exact on GPU keys)."""
from __future__ import annotations

import numpy as np
import torch

from oracle import trail_ref as R
from synth import workload as W

Q_ATOL = 2e-3
L_RTOL = 1e-3


def dev(a: np.ndarray, device="cuda") -> torch.Tensor:
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).to(device)


def make_pair(weights, c, max_slots, max_requests, max_sched, dtype, prior=None, l1_mode=0):
    from paper_2410_01035_b200 import Trail
    t = Trail(weights, c, max_slots, max_requests, max_sched, dtype=dtype, prior=prior,
              l1_mode=l1_mode)
    o = R.TrailOracle(W.decode(weights["W1"], dtype) if dtype == "bf16" else weights["W1"],
                      weights["b1"], weights["W2"], weights["b2"], weights["edges"], c,
                      max_slots, prior=prior, x_dtype=dtype)
    return t, o


def gpu_predict(t, emb, off, ids, pref, prior_override=None):
    e = dev(emb)
    po = dev(prior_override.astype(np.float32)) if prior_override is not None else None
    q, L = t.predict(e, dev(off.astype(np.int32)), dev(ids.astype(np.uint32)),
                     dev(pref.astype(np.uint8)), po)
    torch.cuda.synchronize()
    return q.cpu().numpy().astype(np.float64), L.cpu().numpy().astype(np.float64)


def oracle_predict(o, emb, off, ids, pref, dtype, prior_override=None):
    return o.predict_step(W.decode(emb, dtype), off, ids, pref, prior_override)


def gpu_schedule(t, b, max_run=0):
    run, pre, adm, cnt = t.schedule(dev(b.sched_ids), dev(b.arrival_seq), dev(b.kv_blocks),
                                    dev(b.is_running), b.kv_budget, max_run)
    torch.cuda.synchronize()
    c = cnt.cpu().numpy()
    return (run[:c[0]].cpu().numpy().astype(np.int64), pre[:c[1]].cpu().numpy().astype(np.int64),
            adm[:c[2]].cpu().numpy().astype(np.int64), int(c[3]))


def gpu_state(t, ids):
    s = t.read_state(dev(np.asarray(ids, dtype=np.uint32)))
    torch.cuda.synchronize()
    out = {k: v.cpu().numpy() for k, v in s.items()}
    out["age"] = out["age"].view(np.uint32).astype(np.int64)
    out["thr"] = out["thr"].view(np.uint32).astype(np.int64)
    return out


def gpu_keys_forced(t, ids, is_running, prior_L):
    """The key and forced flag the GPU would pack, rebuilt from its own state."""
    st = gpu_state(t, ids)
    seen = st["seen"] != 0
    key = np.where(seen, st["L"].astype(np.float32), np.float32(prior_L)).astype(np.float64)
    forced = (np.asarray(is_running) != 0) & seen & (st["age"] >= st["thr"])
    return key, forced, st


def assert_predict_close(qg, Lg, qo, Lo, what=""):
    dq = np.abs(qg - qo).max() if qg.size else 0.0
    rl = (np.abs(Lg - Lo) / Lo).max() if Lg.size else 0.0
    assert dq <= Q_ATOL, f"{what}: max|dq| = {dq:.3e}"
    assert rl <= L_RTOL, f"{what}: max rel dL = {rl:.3e}"
    return dq, rl


def top2_gap(q):
    s = np.sort(q, axis=-1)
    return s[..., -1] - s[..., -2]


def report_exemptions(name: str, record: dict) -> None:
    """Write a parity run's near-tie exemptions (the comparator reports every
    exemption) to gpurun_out/parity_exemptions/<name>.json, visible after `-q` runs."""
    import json
    import os
    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "gpurun_out", "parity_exemptions")
    os.makedirs(root, exist_ok=True)
    with open(os.path.join(root, name + ".json"), "w") as f:
        json.dump(record, f, indent=1)
    print(f"{name}: {record.get('key_exempt_steps')} steps with key near-tie exemptions, "
          f"{len(record.get('exemptions', []))} exempted ids")
