"""Diagnostic: layer-1 kernel crossover — K2c (split-K, mode 2) vs K2d (CTA pair, mode 4) on
decode batches of n requests (L2 flushed before each run; per-kernel CUDA events)."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_01035_b200 import Trail  # noqa: E402
from paper_2410_01035_b200.trail import (trail_profile_enable, trail_profile_read,  # noqa: E402
                                         trail_set_l1_mode)
from synth import workload as W  # noqa: E402

dv = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int32) if a.dtype == np.uint32 else np.ascontiguousarray(a)).cuda()  # noqa: E731
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for d, k in ((4096, 10), (8192, 20)):
    w = W.make_weights(d, 512, k, "bf16", seed=1)
    for n in (512, 1024, 2048, 3072, 4096, 6144, 8192, 16384):
        emb, off, pref = W.make_step_inputs(n, d, "bf16", prefill_frac=0.0, seed=3)
        x = [dv(emb), dv(off), dv(np.arange(n, dtype=np.uint32)), dv(pref)]
        t = Trail(w, 0.8, n, n, n, dtype="bf16")
        res = {}
        for mode in (2, 4):
            trail_set_l1_mode(t.h, mode)
            trail_profile_enable(t.h, 2)
            ts = []
            for it in range(6):
                flush.zero_()
                t.predict(*x)
                torch.cuda.synchronize()
                if it >= 1:
                    ts.append(trail_profile_read(t.h, "umma")[0] * 1e3)
            trail_profile_enable(t.h, 0)
            res[mode] = statistics.median(ts)
        t.close()
        fl = 2.0 * n * d * 512
        print(f"d={d} n={n:6d}  K2c {res[2]:8.2f} us  K2d {res[4]:8.2f} us  "
              f"({fl / res[4] / 1e6:7.1f} TFLOP/s)  -> {'K2d' if res[4] < res[2] else 'K2c'}", flush=True)
        del x
