"""Whole-step timeline (pool -> fused -> select) of one CUDA-graph replay of the bench's
steady-state step, from the kernels' globaltimer traces (trail_trace_*).  Diagnostic."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_01035_b200 import Trail, trail_trace_enable, trail_trace_read  # noqa: E402
from synth import workload as W  # noqa: E402


def to_dev(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).cuda()


n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
eng = W.EngineScript(n, n // 4, d=4096, dtype="bf16", seed=W.MASTER_SEED + 1)
w = W.make_weights(4096, 512, 10, "bf16", edges=W.paper_bin_edges(10, 512.0), seed=W.MASTER_SEED)
init = eng.batch(); eng.advance()
bs = []
for _ in range(4):
    bs.append(eng.batch()); eng.advance()
t = Trail(w, 0.8, eng.max_slots, eng.max_slots, eng.max_slots, dtype="bf16")
s = torch.cuda.Stream()


def mk(b):
    return [to_dev(a) for a in (b.emb, b.row_offsets, b.request_ids, b.is_prefill)], \
        [to_dev(a) for a in (b.sched_ids, b.arrival_seq, b.kv_blocks, b.is_running)], b.kv_budget


x0, s0, bud0 = mk(init)
with torch.cuda.stream(s):
    t.predict(*x0, stream=s); t.schedule(*s0, bud0, stream=s)
torch.cuda.synchronize()
trail_trace_enable(t.h, 8192)
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for bi, b in enumerate(bs):
    x, sc, bud = mk(b)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        t.predict(*x, stream=s); t.schedule(*sc, bud, stream=s)
    for rep in range(3):
        with torch.cuda.stream(s):
            fl.zero_()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s); g.replay(); e1.record(s)
        torch.cuda.synchronize()
        tr = trail_trace_read(t.h, 8192).astype(np.int64)
        fu, se, po = tr[:2048], tr[2048:4096], tr[4096:]
        fu = fu[fu[:, 0] > 0]; se = se[se[:, 0] > 0]; po = po[po[:, 0] > 0]
        t0 = po[:, 0].min()
        last = se[se[:, 14] == 1]
        res = {"batch": bi, "prefill_rows": int(b.row_offsets[-1] - b.n), "event_us": e0.elapsed_time(e1) * 1e3,
               "pool_start": 0, "pool_wait_done": int(po[:, 1].min() - t0),
               "pool_last_start": int(po[:, 0].max() - t0),
               "fused_first_start": int(fu[:, 0].min() - t0), "fused_last_start": int(fu[:, 0].max() - t0),
               "fused_first_stage_max": int(fu[:, 2].max() - t0),
               "fused_end": int(fu[:, 8].max() - t0),
               "select_first_start": int(se[:, 0].min() - t0), "select_wait_done": int(se[:, 1].min() - t0),
               "select_end": int(last[0, 7] - t0) if len(last) else -1}
        trail_trace_enable(t.h, 0); trail_trace_enable(t.h, 8192)
        if rep == 2:
            print(json.dumps(res))
