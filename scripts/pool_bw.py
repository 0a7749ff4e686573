"""Diagnostic: K1 (pool) bandwidth on the burst-prefill batch, register vs bulk variant,
L2 flushed before each run; plus torch's own copy of the same rows as a streaming floor."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_01035_b200 import Trail  # noqa: E402
from paper_2410_01035_b200.trail import (trail_profile_enable, trail_profile_read,  # noqa: E402
                                         trail_set_rows_hint)
from synth import workload as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
d = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
eng = W.EngineScript(n, d=d, dtype="bf16", seed=1)
w = W.make_weights(d, 512, 10, "bf16", seed=1)
b0 = eng.batch()
dv = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int32) if a.dtype == np.uint32 else np.ascontiguousarray(a)).cuda()  # noqa: E731
x0 = [dv(a) for a in (b0.emb, b0.row_offsets, b0.request_ids, b0.is_prefill)]
rows = int(b0.row_offsets[-1])
byts = (rows + n) * d * 2
t = Trail(w, 0.8, eng.max_slots, eng.max_slots, eng.max_slots, dtype="bf16")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, hint in (("register", 0), ("bulk", rows)):
    trail_profile_enable(t.h, 2)
    ts = []
    for it in range(8):
        flush.zero_()
        trail_set_rows_hint(t.h, hint)
        t._rows_hint = hint
        t.predict(*x0, rows=hint)
        torch.cuda.synchronize()
        ms, _ = trail_profile_read(t.h, "pool")
        if it >= 2:
            ts.append(ms)
    trail_profile_enable(t.h, 0)
    m = statistics.median(ts)
    print(f"{name:9s} pool {m*1e3:8.2f} us  {byts/(m/1e3)/1e9:8.1f} GB/s  (rows {rows})")
e = x0[0]
out = torch.empty_like(e)
ts = []
for it in range(8):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); out.copy_(e); b.record(); torch.cuda.synchronize()
    if it >= 2:
        ts.append(a.elapsed_time(b))
m = statistics.median(ts)
print(f"torch copy {m*1e3:8.2f} us  read {e.numel()*2/(m/1e3)/1e9:8.1f} GB/s  read+write {2*e.numel()*2/(m/1e3)/1e9:8.1f} GB/s")
ts = []
for it in range(8):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); s = e.view(torch.int32).sum(dtype=torch.int64); b.record(); torch.cuda.synchronize()
    if it >= 2:
        ts.append(a.elapsed_time(b))
m = statistics.median(ts)
print(f"torch int sum {m*1e3:8.2f} us  read {e.numel()*2/(m/1e3)/1e9:8.1f} GB/s")
