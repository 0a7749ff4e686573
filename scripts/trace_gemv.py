"""Per-CTA phase timeline of the broadcast GEMV K2a at configs[0] (fp32, n = 64, d = 4096):
W1 cp.async issue, PDL wait, X staging issue, operands landed, compute + store.  Diagnostic."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_01035_b200 import Trail, trail_trace_enable, trail_trace_read  # noqa: E402
from synth import workload as W  # noqa: E402

n, d = 64, 4096
w = W.make_weights(d, 512, 10, "f32", seed=1)
emb, off, pref = W.make_step_inputs(n, d, "f32", prefill_frac=0.0, seed=2)
dv = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int32) if a.dtype == np.uint32 else np.ascontiguousarray(a)).cuda()  # noqa: E731
x = [dv(emb), dv(off), dv(np.arange(n, dtype=np.uint32)), dv(pref)]
t = Trail(w, 0.8, n, n, n, dtype="f32")
for _ in range(3):
    t.predict(*x)
torch.cuda.synchronize()
trail_trace_enable(t.h, 4096)
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
names = ["w1_issue+scan", "pdl_wait", "x_issue", "landed", "compute"]
for it in range(4):
    fl.zero_()
    torch.cuda.synchronize()
    t.predict(*x)
    torch.cuda.synchronize()
    tr = trail_trace_read(t.h, 4096).astype(np.int64)
    tr = tr[(tr[:, 0] > 0) & (tr[:, 5] > 0)]
    t0 = tr[:, 0].min()
    ph = {nm: [int(np.median(tr[:, i + 1] - tr[:, i])), int(np.max(tr[:, i + 1] - tr[:, i]))]
          for i, nm in enumerate(names)}
    print(json.dumps({"ctas": int(tr.shape[0]), "span_ns": int(tr[:, 5].max() - t0),
                      "start_skew_ns": int(tr[:, 0].max() - t0), **ph}))
