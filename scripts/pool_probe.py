"""Run the predict step on a burst-prefill batch and on a decode batch (for ncu captures of
the pool kernel).  Diagnostic."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_01035_b200 import Trail  # noqa: E402
from synth import workload as W  # noqa: E402


def to_dev(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).cuda()


n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
eng = W.EngineScript(n, d=4096, dtype="bf16", seed=1)
w = W.make_weights(4096, 512, 10, "bf16", seed=1)
b0 = eng.batch(); eng.advance(); b = eng.batch()
x0 = [to_dev(a) for a in (b0.emb, b0.row_offsets, b0.request_ids, b0.is_prefill)]
x = [to_dev(a) for a in (b.emb, b.row_offsets, b.request_ids, b.is_prefill)]
t = Trail(w, 0.8, eng.max_slots, eng.max_slots, eng.max_slots, dtype="bf16")
for _ in range(2):
    t.predict(*x0)
    t.predict(*x)
torch.cuda.synchronize()
print("rows burst", int(b0.row_offsets[-1]), "decode", int(b.row_offsets[-1]))
