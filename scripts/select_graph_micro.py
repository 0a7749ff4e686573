"""K4 selection alone inside a CUDA graph (20 back-to-back calls per replay, PDL chained):
per-call time for several record counts and key structures — excludes the host launch
overhead that an eager event pair measures.  Diagnostic."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_01035_b200 import Trail, trail_schedule_select  # noqa: E402
from synth import workload as W  # noqa: E402
from select_micro import recs  # noqa: E402


def main():
    ms = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "640,2048,4096,20480,81920").split(",")]
    w = W.make_weights(256, 128, 10, "bf16", seed=1)
    rs = np.random.default_rng(0)
    s = torch.cuda.Stream()
    for m in ms:
        t = Trail(w, 0.8, 4, 4, m, dtype="bf16")
        for unseen in (False, True):
            rec, budget = recs(m, unseen, rs)
            reps = 20
            with torch.cuda.stream(s):
                trail_schedule_select(t.h, rec, m, budget, 0, t.run_ids, t.preempt_ids, t.admit_ids,
                                      t.counts, stream=s)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(reps):
                    trail_schedule_select(t.h, rec, m, budget, 0, t.run_ids, t.preempt_ids,
                                          t.admit_ids, t.counts, stream=s)
            times = []
            for i in range(8):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(s):
                    a.record(s); g.replay(); b.record(s)
                torch.cuda.synchronize()
                if i >= 2:
                    times.append(a.elapsed_time(b) * 1e3 / reps)
            print(f"m={m} unseen={unseen}: {np.median(times):.2f} us per call (graph of {reps})",
                  flush=True)
        t.close()


if __name__ == "__main__":
    main()
