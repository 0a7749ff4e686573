"""Per-kernel timing of the predict+schedule step (CUDA events around each library launch,
profile mode 1), warm and L2-flushed, for a few batch sizes.  Diagnostic, not the bench."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_01035_b200 import Trail, trail_profile_enable, trail_profile_read  # noqa: E402
from synth import workload as W  # noqa: E402


def to_dev(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).cuda()


def run(n, d, k, iters, flush, l1_mode):
    eng = W.EngineScript(n, d=d, dtype="bf16", seed=1)
    w = W.make_weights(d, 512, k, "bf16", seed=1)
    t = Trail(w, 0.8, eng.max_slots, eng.max_slots, eng.max_slots, dtype="bf16", l1_mode=l1_mode)
    b0 = eng.batch(); eng.advance()
    b = eng.batch()
    x0 = [to_dev(a) for a in (b0.emb, b0.row_offsets, b0.request_ids, b0.is_prefill)]
    x = [to_dev(a) for a in (b.emb, b.row_offsets, b.request_ids, b.is_prefill)]
    s = [to_dev(a) for a in (b.sched_ids, b.arrival_seq, b.kv_blocks, b.is_running)]
    t.predict(*x0)
    fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(5):
        t.predict(*x); t.schedule(*s, b.kv_budget)
    torch.cuda.synchronize()
    trail_profile_enable(t.h, 1)
    trail_profile_read(t.h, "pool", reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tot = 0.0
    for _ in range(iters):
        if flush:
            fl.zero_()
        e0.record()
        t.predict(*x); t.schedule(*s, b.kv_budget)
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    out = {"n": n, "d": d, "flush": flush, "step_us": 1e3 * tot / iters}
    for kname in ("pool", "gemv", "umma", "head", "pack", "select"):
        ms, cnt = trail_profile_read(t.h, kname)
        if cnt:
            out[kname] = round(1e3 * ms / cnt, 2)
    # empty-kernel reference: a 1-element fill
    z = torch.zeros(1, device="cuda")
    torch.cuda.synchronize()
    e0.record()
    for _ in range(100):
        z.fill_(1.0)
    e1.record()
    torch.cuda.synchronize()
    out["tiny_kernel_us"] = round(10 * e0.elapsed_time(e1), 2)
    t.close()
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--sizes", default="1,16,64,512,4096")
    args = ap.parse_args()
    for n in [int(v) for v in args.sizes.split(",")]:
        for flush in (False, True):
            print(json.dumps(run(n, 4096, 10, args.iters, flush, 0)), flush=True)
