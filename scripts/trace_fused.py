"""Per-CTA phase timeline of the fused tcgen05 predict kernel (trail_trace_*), for a few
split factors: median/max phase durations across CTAs and the launch skew.  Diagnostic."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_01035_b200 import Trail, trail_trace_enable, trail_trace_read  # noqa: E402
from synth import workload as W  # noqa: E402

PH = ["prologue", "first_stage", "mainloop", "tile_to_smem", "cluster_sync1", "exchange",
      "reduce_l2", "head_tail"]


def to_dev(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).cuda()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--splits", default="8")
    ap.add_argument("--no-flush", action="store_true")
    args = ap.parse_args()
    eng = W.EngineScript(args.n, d=args.d, dtype="bf16", seed=1)
    w = W.make_weights(args.d, 512, args.k, "bf16", seed=1)
    b0 = eng.batch(); eng.advance(); b = eng.batch()
    x0 = [to_dev(a) for a in (b0.emb, b0.row_offsets, b0.request_ids, b0.is_prefill)]
    x = [to_dev(a) for a in (b.emb, b.row_offsets, b.request_ids, b.is_prefill)]
    fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for sp in args.splits.split(","):
        if sp != "0":
            os.environ["TRAIL_FUSED_SPLITS"] = sp
        else:
            os.environ.pop("TRAIL_FUSED_SPLITS", None)
        t = Trail(w, 0.8, eng.max_slots, eng.max_slots, eng.max_slots, dtype="bf16", l1_mode=2)
        t.predict(*x0)
        for _ in range(3):
            t.predict(*x)
        torch.cuda.synchronize()
        trail_trace_enable(t.h, 4096)
        res = []
        for it in range(5):
            if not args.no_flush:
                fl.zero_()
            torch.cuda.synchronize()
            t.predict(*x)
            torch.cuda.synchronize()
            tr = trail_trace_read(t.h, 4096).astype(np.int64)
            tr = tr[tr[:, 0] > 0]
            t0 = tr[:, 0].min()
            ph = {p: np.diff(tr[:, [i, i + 1]], axis=1)[:, 0] for i, p in enumerate(PH)}
            res.append({"ctas": int(len(tr)), "span_ns": int(tr[:, 8].max() - t0),
                        "start_skew_ns": int(tr[:, 0].max() - t0),
                        "sms": int(len(np.unique(tr[:, 15]))),
                        **{p: [int(np.median(v)), int(v.max())] for p, v in ph.items()},
                        "head_ctas": [[int(x) for x in (r[9] - r[7], r[11] - r[9], r[8] - r[11],
                                                        r[8] - t0)]
                                      for r in tr[tr[:, 14] == 1][:4]]})
            trail_trace_enable(t.h, 0); trail_trace_enable(t.h, 4096)
        print(json.dumps({"n": args.n, "d": args.d, "splits": int(sp),
                          "dbg": os.environ.get("TRAIL_FUSED_DBG", "0"), "flush": not args.no_flush, "runs": res[2:4]}))
        t.close()


if __name__ == "__main__":
    main()
