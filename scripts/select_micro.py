"""Microbenchmark of the K4 selection kernel alone (given records, CUDA events, eager
launches): median us per call for several record counts and key structures."""
import sys
import os
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_01035_b200 import Trail, trail_schedule_select  # noqa: E402
from synth import workload as W  # noqa: E402


def recs(m, unseen, rs):
    key = rs.uniform(25.6, 486.4, m).astype(np.float32)
    if unseen:
        key[m // 5:] = 256.0
    forced = rs.random(m) < 0.2
    running = forced | (rs.random(m) < 0.6)
    kb = key.view(np.uint32) & 0x7FFFFFFF
    kb = kb | np.where(forced, 0, 0x80000000).astype(np.uint32)
    r = np.zeros((m, 4), np.uint32)
    r[:, 0] = kb
    r[:, 1] = rs.permutation(m).astype(np.uint32) + 1000
    r[:, 2] = rs.integers(1, 40, m)
    r[:, 3] = np.arange(m, dtype=np.uint32) | (running.astype(np.uint32) << 31)
    return torch.from_numpy(r.view(np.int32)).cuda(), int(r[:, 2].sum() * 0.5)


def main():
    ms = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "80,640,2048,4096,20480,81920").split(",")]
    w = W.make_weights(256, 128, 10, "bf16", seed=1)
    rs = np.random.default_rng(0)
    for m in ms:
        t = Trail(w, 0.8, 4, 4, m, dtype="bf16")
        for unseen in (False, True):
            rec, budget = recs(m, unseen, rs)
            times = []
            for i in range(30):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                trail_schedule_select(t.h, rec, m, budget, 0, t.run_ids, t.preempt_ids,
                                      t.admit_ids, t.counts)
                b.record()
                torch.cuda.synchronize()
                if i >= 5:
                    times.append(a.elapsed_time(b) * 1e3)
            print(f"m={m} unseen={unseen}: median {np.median(times):.1f} us  min {np.min(times):.1f}",
                  flush=True)
        t.close()


if __name__ == "__main__":
    main()
