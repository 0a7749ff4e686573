"""Per-CTA phases of the bulk K1 kernel on a configs[3]-shaped mixed batch (16 384 requests,
~6.6 K prompt rows at d = 8192): prologue (work prefix + search) and streaming.  Diagnostic."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_01035_b200 import Trail, trail_trace_enable, trail_trace_read  # noqa: E402
from synth import workload as W  # noqa: E402

n, d = int(sys.argv[1]) if len(sys.argv) > 1 else 16384, 8192
eng = W.EngineScript(n, n // 4, d=d, dtype="bf16", seed=W.MASTER_SEED + 1, burst_start=False)
init = eng.batch(); eng.advance()
b = eng.batch()
w = W.make_weights(d, 512, 20, "bf16", edges=W.paper_bin_edges(20, 1024.0), seed=1)
dv = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int32) if a.dtype == np.uint32 else np.ascontiguousarray(a)).cuda()  # noqa: E731
x = [dv(a) for a in (b.emb, b.row_offsets, b.request_ids, b.is_prefill)]
t = Trail(w, 0.8, eng.max_slots, eng.max_slots, eng.max_slots, dtype="bf16")
t.predict(*x)
torch.cuda.synchronize()
trail_trace_enable(t.h, 4096 + 160)
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for it in range(3):
    fl.zero_()
    torch.cuda.synchronize()
    t.predict(*x)
    torch.cuda.synchronize()
    tr = trail_trace_read(t.h, 4096 + 160).astype(np.int64)[4096:]
    tr = tr[(tr[:, 0] > 0)]
    t0 = tr[:, 0].min()
    has = tr[:, 2] > 0
    print(json.dumps({"ctas": int(tr.shape[0]), "working": int(has.sum()),
                      "prologue_med_max": [int(np.median(tr[has, 1] - tr[has, 0])), int(np.max(tr[has, 1] - tr[has, 0]))],
                      "stream_med_max": [int(np.median(tr[has, 2] - tr[has, 1])), int(np.max(tr[has, 2] - tr[has, 1]))],
                      "span": int(tr[has, 2].max() - t0), "start_skew": int(tr[:, 0].max() - t0),
                      "rows": int(b.row_offsets[-1])}))
