"""Per-CTA phase timeline of the bucketed selection (B0 samples, B1 histogram, B2 scatter,
B3 rank) on given records (trail_trace_*): start / end of each kernel relative to B0's first
CTA, and median / max per phase across CTAs, ns.  Diagnostic."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_01035_b200 import Trail, trail_schedule_select, trail_trace_enable, trail_trace_read  # noqa: E402
from synth import workload as W  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from select_micro import recs  # noqa: E402

w = W.make_weights(256, 128, 10, "bf16", seed=1)
rs = np.random.default_rng(0)
B3, B0, B1, B2 = 2048, 3072, 3136, 3584
for m in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "20480,81920").split(",")]:
    t = Trail(w, 0.8, 4, 4, m, dtype="bf16")
    rec, budget = recs(m, True, rs)
    for _ in range(3):
        trail_schedule_select(t.h, rec, m, budget, 0, t.run_ids, t.preempt_ids, t.admit_ids, t.counts)
    torch.cuda.synchronize()
    trail_trace_enable(t.h, 4096)
    for rep in range(3):
        trail_schedule_select(t.h, rec, m, budget, 0, t.run_ids, t.preempt_ids, t.admit_ids, t.counts)
        torch.cuda.synchronize()
        tr = trail_trace_read(t.h, 4096).astype(np.int64)
        b3, b0, b1, b2 = tr[B3:B0], tr[B0:B1], tr[B1:B2], tr[B2:4096]
        b3, b0, b1, b2 = [a[a[:, 0] > 0] for a in (b3, b0, b1, b2)]
        t0 = b0[:, 0].min()

        def ph(a, i, j):
            d = a[:, j] - a[:, i]
            return [int(np.median(d)), int(d.max())]
        last = b3[b3[:, 14] == 1]
        out = {"m": m, "ctas": [len(b0), len(b1), len(b2), len(b3)],
               "b0_wait_done": int(b0[:, 1].min() - t0), "b0_samples": ph(b0, 1, 2), "b0_rank": ph(b0, 2, 3),
               "b0_end": int(b0[:, 3].max() - t0),
               "b1_first": int(b1[:, 0].min() - t0), "b1_wait_done": int(b1[:, 1].min() - t0),
               "b1_work": ph(b1, 1, 2), "b1_end": int(b1[:, 2].max() - t0),
               "b2_wait_done": int(b2[:, 1].min() - t0), "b2_scan": ph(b2, 1, 2), "b2_scatter": ph(b2, 2, 3),
               "b2_end": int(b2[:, 3].max() - t0),
               "b3_wait_done": int(b3[:, 1].min() - t0), "b3_scan": ph(b3, 1, 2), "b3_stage": ph(b3, 2, 3),
               "b3_rank": ph(b3, 3, 4), "b3_atomic": ph(b3, 4, 5), "b3_rank_end": int(b3[:, 4].max() - t0),
               "tail": int(last[0, 6] - last[0, 5]) if len(last) else -1,
               "end": int(last[0, 6] - t0) if len(last) else -1}
        trail_trace_enable(t.h, 0); trail_trace_enable(t.h, 4096)
        if rep == 2:
            print(json.dumps(out), flush=True)
    trail_trace_enable(t.h, 0)
    t.close()
