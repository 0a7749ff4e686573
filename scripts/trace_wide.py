"""Per-CTA phase timeline of the CTA-pair kernel K2d at configs[3] (trail_trace_*), L2
flushed: prologue, K loop (until `done`), layer 2 on the tensor cores, head, teardown —
median / max across CTAs, ns.  TRAIL_WIDE_DIAG=3 skips the loads (timing only).  Diagnostic."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_01035_b200 import Trail, trail_trace_enable, trail_trace_read  # noqa: E402
from synth import workload as W  # noqa: E402

n, d = 16384, 8192
eng = W.EngineScript(n, n // 4, d=d, dtype="bf16", seed=W.MASTER_SEED + 1, burst_start=False)
init = eng.batch(); eng.advance()
b = eng.batch()
w = W.make_weights(d, 512, 20, "bf16", edges=W.paper_bin_edges(20, 1024.0), seed=1)
dv = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int32) if a.dtype == np.uint32 else np.ascontiguousarray(a)).cuda()  # noqa: E731
x0 = [dv(a) for a in (init.emb, init.row_offsets, init.request_ids, init.is_prefill)]
x = [dv(a) for a in (b.emb, b.row_offsets, b.request_ids, b.is_prefill)]
t = Trail(w, 0.8, eng.max_slots, eng.max_slots, eng.max_slots, dtype="bf16")
t.predict(*x0)
for _ in range(2):
    t.predict(*x)
torch.cuda.synchronize()
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for rep in range(3):
    trail_trace_enable(t.h, 160)
    fl.zero_(); torch.cuda.synchronize()
    t.predict(*x)
    torch.cuda.synchronize()
    tr = trail_trace_read(t.h, 160).astype(np.int64)
    trail_trace_enable(t.h, 0)
    tr = tr[(tr[:, 0] > 0) & (tr[:, 5] > 0)]
    t0 = tr[:, 0].min()
    ph = lambda i, j: [int(np.median(tr[:, j] - tr[:, i])), int((tr[:, j] - tr[:, i]).max())]  # noqa: E731
    # CTAs whose 128 rows hold a prompt (their X rows come from K1's xs: they wait for K1)
    pf = np.asarray(b.is_prefill).astype(bool)
    has_p = np.array([pf[128 * c:128 * c + 128].any() for c in range(len(tr))])
    kl = tr[:, 2] - tr[:, 1]
    extra = {"k_loop_prompt_ctas": [int(np.median(kl[has_p])) if has_p.any() else -1, int(has_p.sum())],
             "k_loop_decode_ctas": [int(np.median(kl[~has_p])), int(kl[~has_p].max()), int((~has_p).sum())],
             "start_prompt_ctas": int(np.median(tr[has_p, 0] - t0)) if has_p.any() else -1}
    print(json.dumps(extra), flush=True)
    print(json.dumps({"diag": os.environ.get("TRAIL_WIDE_DIAG", "0"), "ctas": len(tr),
                      "start_skew": int(tr[:, 0].max() - t0), "prologue": ph(0, 1), "k_loop": ph(1, 2),
                      "layer2": ph(2, 3), "head": ph(3, 4), "teardown": ph(4, 5),
                      "span": int(tr[:, 5].max() - t0)}), flush=True)
