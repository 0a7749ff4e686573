"""K1b timing on a configs[3]-shaped mixed batch (16 384 requests, 82 prompts of ~84 rows,
d = 8192) with the prompts (a) scattered among the decode rows (as the engine script places
them) and (b) contiguous at the end of the batch.  Profile-mode events, L2 flushed.  Diagnostic."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_01035_b200 import (Trail, trail_profile_enable, trail_profile_read,  # noqa: E402
                                   trail_trace_enable, trail_trace_read)
from paper_2410_01035_b200.trail import trail_set_rows_hint  # noqa: E402
from synth import workload as W  # noqa: E402

n, d, npr, plen = 16384, 8192, 82, 84
rs = np.random.default_rng(1)
w = W.make_weights(d, 512, 20, "bf16", edges=W.paper_bin_edges(20, 1024.0), seed=1)
t = Trail(w, 0.8, n + 8, n, n, dtype="bf16")
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rows_total = n - npr + npr * plen
emb = torch.randn(rows_total, d, device="cuda").to(torch.bfloat16)
ids = torch.arange(n, dtype=torch.int32, device="cuda")
for layout in ("scattered", "contiguous", "scattered", "contiguous"):
    cnt = np.ones(n, np.int64)
    pos = rs.choice(n, npr, replace=False) if layout == "scattered" else np.arange(n - npr, n)
    cnt[pos] = plen
    off = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int32)
    pref = (cnt > 1).astype(np.uint8)
    o = torch.from_numpy(off).cuda(); p = torch.from_numpy(pref).cuda()
    trail_set_rows_hint(t.h, int(off[-1]))
    for _ in range(2):
        t.predict(emb, o, ids, p)
    torch.cuda.synchronize()
    trail_profile_enable(t.h, 1)
    trail_profile_read(t.h, "pool", reset=True)
    v = []
    for _ in range(8):
        fl.zero_(); torch.cuda.synchronize()
        t.predict(emb, o, ids, p)
        torch.cuda.synchronize()
        ms, c = trail_profile_read(t.h, "pool", reset=True)
        v.append(1e3 * ms / max(c, 1))
    trail_profile_enable(t.h, 0)
    # per-CTA phases (globaltimer, ns): prologue, first stage, streaming, tail, crossings
    trail_trace_enable(t.h, 4096 + 160)
    fl.zero_(); torch.cuda.synchronize()
    t.predict(emb, o, ids, p)
    torch.cuda.synchronize()
    tr = trail_trace_read(t.h, 4096 + 160).astype(np.int64)[4096:]
    tr = tr[(tr[:, 0] > 0) & (tr[:, 2] > 0)]
    trail_trace_enable(t.h, 0)
    med = lambda a: int(np.median(a))  # noqa: E731
    print(json.dumps({"layout": layout, "pool_us_med": round(float(np.median(v)), 2),
                      "rows": int(off[-1]), "prompt_rows": npr * plen, "ctas": len(tr),
                      "prologue": med(tr[:, 1] - tr[:, 0]), "first_stage": med(tr[:, 3] - tr[:, 1]),
                      "stream": med(tr[:, 4] - tr[:, 3]), "stream_max": int((tr[:, 4] - tr[:, 3]).max()),
                      "tail": med(tr[:, 2] - tr[:, 4]), "tail_max": int((tr[:, 2] - tr[:, 4]).max()),
                      "span": int(tr[:, 2].max() - tr[:, 0].min())}), flush=True)
