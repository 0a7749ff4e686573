"""Per-CTA phase timeline of the rank-counting selection kernel (TRAIL_TRACE_SELECT=1 +
trail_trace_*), after a realistic predict step.  Diagnostic."""
import json
import os
import sys

import numpy as np
import torch

os.environ["TRAIL_TRACE_SELECT"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_01035_b200 import Trail, trail_trace_enable, trail_trace_read  # noqa: E402
from synth import workload as W  # noqa: E402


def to_dev(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).cuda()


for n in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "512,4096").split(",")]:
    eng = W.EngineScript(n, d=4096, dtype="bf16", seed=1)
    w = W.make_weights(4096, 512, 10, "bf16", seed=1)
    b0 = eng.batch(); eng.advance(); b = eng.batch()
    x0 = [to_dev(a) for a in (b0.emb, b0.row_offsets, b0.request_ids, b0.is_prefill)]
    x = [to_dev(a) for a in (b.emb, b.row_offsets, b.request_ids, b.is_prefill)]
    sc = [to_dev(a) for a in (b.sched_ids, b.arrival_seq, b.kv_blocks, b.is_running)]
    t = Trail(w, 0.8, eng.max_slots, eng.max_slots, eng.max_slots, dtype="bf16")
    t.predict(*x0)
    fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for flush in (False, True):
        res = []
        for it in range(4):
            t.predict(*x)
            torch.cuda.synchronize()
            if flush:
                fl.zero_()
            trail_trace_enable(t.h, 0)
            trail_trace_enable(t.h, 4096)
            torch.cuda.synchronize()
            t.schedule(*sc, b.kv_budget)
            tr = trail_trace_read(t.h, 4096).astype(np.int64)
            tr = tr[tr[:, 0] > 0]
            t0 = tr[:, 0].min()
            last = tr[tr[:, 14] == 1][0]
            res.append({"ctas": int(len(tr)), "start_skew": int(tr[:, 0].max() - t0),
                        "wait": int(np.median(tr[:, 1] - tr[:, 0])),
                        "keys": int(np.median(tr[:, 2] - tr[:, 1])),
                        "rank": int(np.median(tr[:, 3] - tr[:, 2])),
                        "atomics": int(np.median(tr[:, 4] - tr[:, 3])),
                        "last_start": int(last[4] - t0), "counters": int(last[5] - last[4]),
                        "preempt_list": int(last[6] - last[5]), "tail": int(last[7] - last[6]),
                        "total": int(last[7] - t0)})
        print(json.dumps({"n": n, "m": int(b.m), "flush": flush, "runs": res[1:3]}))
    t.close()
