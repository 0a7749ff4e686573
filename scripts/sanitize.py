"""Small-shape workload that launches every kernel of libtrail.so once or twice, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck python scripts/sanitize.py

Covers: K1 pooling (register and bulk variants), K2a GEMV + K3 head, K2t 3xTF32 tcgen05 + K3,
K2c split-K tcgen05 (fused head), K2d CTA-pair tcgen05, K4 selection by rank counting and by
the bucketed sample sort (local build and given records with padding), K5 pack, K6 time update, K1c chunked prefill,
K1m multi-layer mix, release and state read.  Exits non-zero on a CUDA error; the sanitizer
reports its own findings."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_01035_b200 import Trail, trail_schedule_pack, trail_schedule_select  # noqa: E402
from paper_2410_01035_b200.trail import trail_prefill_chunk, trail_set_rows_hint  # noqa: E402
from synth import workload as W  # noqa: E402


def dv(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).cuda()


def run(n, d, dtype, l1_mode, waiting):
    w = W.make_weights(d, 512, 10, dtype, seed=3)
    eng = W.EngineScript(n, waiting, d=d, dtype=dtype, seed=3)
    t = Trail(w, 0.8, eng.max_slots, eng.max_slots, eng.max_slots, dtype=dtype, l1_mode=l1_mode)
    for step in range(2):
        b = eng.batch()
        t.predict(dv(b.emb), dv(b.row_offsets), dv(b.request_ids), dv(b.is_prefill))
        run_, pre, adm, cnt = t.schedule(dv(b.sched_ids), dv(b.arrival_seq), dv(b.kv_blocks),
                                         dv(b.is_running), b.kv_budget)
        torch.cuda.synchronize()
        eng.advance(run_[:int(cnt[0].item())].cpu().numpy())
    # bulk pooling variant: a large row hint switches K1 to the cp.async.bulk kernel
    b = eng.batch()
    trail_set_rows_hint(t.h, 1 << 20)
    t.predict(dv(b.emb), dv(b.row_offsets), dv(b.request_ids), dv(b.is_prefill), rows=1 << 20)
    trail_set_rows_hint(t.h, 0)
    t._rows_hint = 0
    # pack (padded) + select over given records
    cap = eng.max_slots
    rec = torch.empty((cap, 4), dtype=torch.int32, device="cuda")
    m = b.m - 3
    trail_schedule_pack(t.h, dv(b.sched_ids), dv(b.arrival_seq), dv(b.kv_blocks), dv(b.is_running),
                        m, cap, rec)
    trail_schedule_select(t.h, rec, cap, b.kv_budget, 0, t.run_ids, t.preempt_ids, t.admit_ids,
                          t.counts)
    # time update, chunked prefill, multi-layer mix, release, state read
    ids = dv(b.request_ids)
    t.time_update(ids, 3)
    pooled = torch.empty((b.n, d), dtype=torch.uint16 if dtype == "bf16" else torch.float32,
                         device="cuda")
    fin = np.ones(b.n, np.uint8)
    fin[::2] = 0
    trail_prefill_chunk(t.h, dv(b.emb), d, dv(b.row_offsets), ids, dv(fin), b.n, pooled, d)
    t.predict_layers([dv(b.emb), dv(b.emb)], [1.0, 3.0], dv(b.row_offsets), ids,
                     dv(b.is_prefill))
    t.release(ids[:4])
    t.read_state(ids)
    torch.cuda.synchronize()
    t.close()


def main():
    torch.cuda.init()
    run(24, 1024, "f32", 1, 8)        # GEMV + head (fp32)
    run(70, 1024, "f32", 5, 8)        # K2t 3xTF32 tcgen05 (two request blocks) + head
    run(40, 1024, "bf16", 2, 10)      # K2c split-K tcgen05
    run(300, 1024, "bf16", 4, 100)    # K2d CTA pair; rank-counting selection (<= 2048 records)
    run(600, 512, "bf16", 2, 4000)    # bucketed sample-sort selection (4600 records)
    print("sanitize workload done")


if __name__ == "__main__":
    main()
