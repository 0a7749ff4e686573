"""the predict step beside the LLM: the paper overlaps its predictor with the
model by running it on the CPU (running it on the GPU "introduces a slowdown in the
decoding phase"); here it runs on a GPU side stream, concurrently with the LLM's layers
l+1 ... L of the same iteration, reading the layer-l hidden states in place (the tap: the API
takes a pointer + leading dimension, so the residual-stream tensor of the batch is passed
without a copy).

Stand-in LLM: Llama-3-8B-shaped decoder layers (d = 4096, MLP 14336, GQA 32/8 heads x 128)
as bf16 GEMMs on one decode batch of n tokens (attention's KV reads are not modelled; the
GEMMs are the per-token work).  Layer l = 11 (P:199 layer-11 embeddings), L = 32.  Measured
with CUDA events, CUDA graphs, L2 flushed before each iteration:
  layers      layers l+1..L alone
  serial      layers, then predict + schedule on the same stream
  overlap     predict + schedule on a side stream forked after layer l, joined at the end
Reports the iteration times and the fraction of the predict step hidden by the overlap.

  python scripts/overlap.py [--n 512] [--iters 50]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_01035_b200 import Trail  # noqa: E402
from synth import workload as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--layer", type=int, default=11)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    n, d, dff = args.n, 4096, 14336
    g = torch.Generator(device=dev).manual_seed(0)
    mk = lambda *s: (torch.randn(*s, device=dev, generator=g, dtype=torch.float32) * 0.02).to(torch.bfloat16)  # noqa: E731
    # one shared set of layer weights (the per-layer work is what matters, not distinct values)
    wqkv, wo = mk(d, d + 2 * 1024), mk(d, d)
    wgu, wd = mk(d, 2 * dff), mk(dff, d)
    h = torch.randn(n, d, device=dev, generator=g).to(torch.bfloat16)

    def layer(x):
        qkv = x @ wqkv
        x = x + qkv[:, :d] @ wo
        gu = x @ wgu
        a = torch.nn.functional.silu(gu[:, :dff]) * gu[:, dff:]
        return x + a @ wd

    eng = W.EngineScript(n, n // 4, d=d, dtype="bf16", seed=5)
    w = W.make_weights(d, 512, 10, "bf16", seed=5)
    t = Trail(w, 0.8, eng.max_slots, eng.max_slots, eng.max_slots, dtype="bf16")
    b = eng.batch()
    to = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int32) if a.dtype == np.uint32 else np.ascontiguousarray(a)).to(dev)  # noqa: E731
    off, ids, pref = to(b.row_offsets), to(b.request_ids), to(b.is_prefill)
    sids, arr, kv, run = to(b.sched_ids), to(b.arrival_seq), to(b.kv_blocks), to(b.is_running)
    # the first iteration observes every request (prefill rows); later ones are decode rows
    emb0 = to(b.emb)
    t.predict(emb0, off, ids, pref)
    eng.advance()
    b = eng.batch()
    off, ids, pref = to(b.row_offsets), to(b.request_ids), to(b.is_prefill)
    decode_only = bool((b.row_offsets[1:] - b.row_offsets[:-1] == 1).all())
    s_main, s_side = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev_tap, ev_done = torch.cuda.Event(), torch.cuda.Event()
    hl = torch.empty(n, d, device=dev, dtype=torch.bfloat16)   # the layer-l residual stream

    def prefix():
        x = h
        for _ in range(args.layer):
            x = layer(x)
        hl.copy_(x)                          # stands for the layer-l output buffer
        return hl

    def predict_on(stream, emb):
        t.predict(emb, off, ids, pref, stream=stream, rows=int(b.row_offsets[-1]))
        t.schedule(sids, arr, kv, run, b.kv_budget, stream=stream)

    def it_layers():
        x = prefix()
        for _ in range(args.layers - args.layer):
            x = layer(x)

    def it_serial():
        x = prefix()
        for _ in range(args.layers - args.layer):
            x = layer(x)
        predict_on(torch.cuda.current_stream(), hl if decode_only else emb_b)

    def it_overlap():
        x = prefix()
        ev_tap.record()
        with torch.cuda.stream(s_side):
            s_side.wait_event(ev_tap)
            predict_on(s_side, hl if decode_only else emb_b)
            ev_done.record()
        for _ in range(args.layers - args.layer):
            x = layer(x)
        torch.cuda.current_stream().wait_event(ev_done)

    emb_b = to(b.emb)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    res = {}
    for name, fn in (("layers", it_layers), ("serial", it_serial), ("overlap", it_overlap)):
        with torch.cuda.stream(s_main):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s_main):
                fn()
            ts = []
            for _ in range(args.iters):
                flush.zero_()
                a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s_main)
                gr.replay()
                z.record(s_main)
                s_main.synchronize()
                ts.append(a.elapsed_time(z) * 1e3)
        res[name] = statistics.mean(ts)
        res[name + "_se"] = statistics.stdev(ts) / len(ts) ** 0.5
    # the predict + schedule step alone on the same batch (graph, L2 flushed) for scale
    with torch.cuda.stream(s_main):
        gp = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gp, stream=s_main):
            predict_on(s_main, hl if decode_only else emb_b)
        ts = []
        for _ in range(args.iters):
            flush.zero_()
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s_main)
            gp.replay()
            z.record(s_main)
            s_main.synchronize()
            ts.append(a.elapsed_time(z) * 1e3)
    res["predict_alone"] = statistics.mean(ts)
    pred = res["serial"] - res["layers"]
    out = {"n": n, "layer_l": args.layer, "L": args.layers, "us_layers": res["layers"],
           "us_serial": res["serial"], "us_overlap": res["overlap"],
           "se_us": {k: res[k + "_se"] for k in ("layers", "serial", "overlap")},
           "us_predict_step_alone": res["predict_alone"],
           "predict_share_of_iteration": res["predict_alone"] / res["layers"],
           "us_serial_minus_layers": pred,
           "us_overlap_minus_layers": res["overlap"] - res["layers"],
           "tap": "layer-l residual-stream tensor passed in place (pointer + ld), no copy"
                  if decode_only else "prefill rows present: the step's own embedding buffer"}
    print(json.dumps(out))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)
    t.close()


if __name__ == "__main__":
    main()
