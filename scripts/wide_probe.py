"""K2d timing probe at configs[3] shape (16 384 requests, d = 8192, k = 20): median per-launch
time of the layer-1 kernel (profile mode: CUDA events around the launch), L2 flushed before
every step.  Knob: TRAIL_WIDE_DIAG (load-skipping probes).  Diagnostic."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_01035_b200 import Trail, trail_profile_enable, trail_profile_read  # noqa: E402
from synth import workload as W  # noqa: E402

n, d = int(sys.argv[1]) if len(sys.argv) > 1 else 16384, 8192
eng = W.EngineScript(n, n // 4, d=d, dtype="bf16", seed=W.MASTER_SEED + 1, burst_start=False)
init = eng.batch(); eng.advance()
b = eng.batch()
w = W.make_weights(d, 512, 20, "bf16", edges=W.paper_bin_edges(20, 1024.0), seed=1)
dv = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int32) if a.dtype == np.uint32 else np.ascontiguousarray(a)).cuda()  # noqa: E731
x0 = [dv(a) for a in (init.emb, init.row_offsets, init.request_ids, init.is_prefill)]
x = [dv(a) for a in (b.emb, b.row_offsets, b.request_ids, b.is_prefill)]
t = Trail(w, 0.8, eng.max_slots, eng.max_slots, eng.max_slots, dtype="bf16")
t.predict(*x0)
for _ in range(3):
    t.predict(*x)
torch.cuda.synchronize()
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
fl2 = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
trail_profile_enable(t.h, 1)
out = {"diag": os.environ.get("TRAIL_WIDE_DIAG", "0")}
for name in ("umma", "pool"):
    trail_profile_read(t.h, name, reset=True)
vals = {"umma": [], "pool": []}
for it in range(12):
    fl.zero_(); fl2.sum()
    torch.cuda.synchronize()
    t.predict(*x)
    torch.cuda.synchronize()
    for name in vals:
        ms, cnt = trail_profile_read(t.h, name, reset=True)
        if cnt:
            vals[name].append(1e3 * ms / cnt)
for name, v in vals.items():
    if v:
        out[name + "_us_med"] = round(float(np.median(v)), 2)
        out[name + "_us_min"] = round(float(np.min(v)), 2)
print(json.dumps(out), flush=True)
