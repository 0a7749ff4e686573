"""Iteration-level batch simulator driven by the real GPU path (SPEC run_batch,
S:384-392).  Each iteration: every live job (running + waiting) is ranked and the batch is
filled under a KV budget by trail_schedule_step (limited-preemption SPRPT);
every job in the batch emits one token; the jobs that ran are observed by trail_predict_step
(prefill observation the first time, decode afterwards); finished jobs release their slots.

Observations follow SPEC's synthetic model: p = softmax(-conc * |m_i - remaining| / w),
peak shifted one bin with probability `mislabel`.  It is realised THROUGH the real classifier:
the embedding carries the score vector s in its first k coordinates and the probe weights are
W1 = [I; -I; 0], b1 = 0, W2 = [I, -I, 0], b2 = 0, so z = ReLU(s) - ReLU(-s) = s and the GPU's
softmax is the model's p (up to bf16 rounding of s).

Reports mean latency, mean TTFT (iterations) and preemptions per policy c.  Diagnostic /
demonstration tool — the product path is only the library calls it makes.

  python scripts/simulate.py [--jobs 2000] [--rate 6] [--budget-frac 0.35] [--c 0,0.5,0.8,inf]
"""
from __future__ import annotations

import argparse
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_01035_b200 import Trail  # noqa: E402
from synth import workload as W  # noqa: E402


def probe_weights(d: int, H: int, k: int, edges: np.ndarray) -> dict:
    W1 = np.zeros((H, d), np.float32)
    W2 = np.zeros((k, H), np.float32)
    for i in range(k):
        W1[i, i] = 1.0
        W1[k + i, i] = -1.0
        W2[i, i] = 1.0
        W2[i, k + i] = -1.0
    return {"W1": W.encode(W1, "bf16"), "b1": np.zeros(H, np.float32), "W2": W2,
            "b2": np.zeros(k, np.float32), "edges": edges}


def run(c: float, args, seed: int) -> dict:
    rs = np.random.default_rng(seed)
    k, d, H = 10, 256, 128
    edges = W.paper_bin_edges(k)
    m = (edges[:-1] + edges[1:]) / 2
    w = edges[1] - edges[0]
    n_jobs = args.jobs
    # workload: Poisson arrivals per iteration, Alpaca-like output lengths
    arr = np.cumsum(rs.exponential(1.0 / args.rate, n_jobs)).astype(np.int64)
    size = np.clip(np.round(rs.lognormal(math.log(150), 0.9, n_jobs)), 1, 512).astype(np.int64)
    plen = np.clip(np.round(rs.lognormal(math.log(32), 0.7, n_jobs)), 4, 512).astype(np.int64)
    slots = args.slots
    budget = int(args.budget_frac * slots * 24)   # blocks of 16 tokens
    t = Trail(probe_weights(d, H, k, edges), c, slots, slots, slots, dtype="bf16")
    free = list(range(slots))[::-1]
    live: dict = {}                     # job -> slot
    gen = np.zeros(n_jobs, np.int64)
    first = np.full(n_jobs, -1, np.int64)
    done = np.full(n_jobs, -1, np.int64)
    running = set()
    observed = set()
    recompute = np.zeros(n_jobs, np.int64)   # iterations of context recompute still owed
    nxt, it, preempt = 0, 0, 0
    dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    while (nxt < n_jobs or live) and it < args.max_iters:
        while nxt < n_jobs and arr[nxt] <= it and free:
            live[nxt] = free.pop()
            nxt += 1
        if not live:
            it = int(arr[nxt]) if nxt < n_jobs else it + 1
            continue
        jobs = np.array(sorted(live), np.int64)
        ids = np.array([live[j] for j in jobs], np.int32)
        kv = ((plen[jobs] + gen[jobs] + 1 + 15) // 16).astype(np.int32)
        run_flag = np.array([j in running for j in jobs], np.uint8)
        r, p_ids, a_ids, cnt = t.schedule(dv(ids), dv(jobs.astype(np.int32)), dv(kv), dv(run_flag),
                                          budget)
        cc = cnt.cpu().numpy()
        run_slots = set(r[:cc[0]].cpu().numpy().tolist())
        preempt += int(cc[1])
        slot2job = {live[j]: j for j in jobs}
        batch = [slot2job[s] for s in sorted(run_slots)]
        if not batch:                    # forced set over budget with nothing runnable
            it += 1
            continue
        # discard mode: a preempted job lost its KV; when it runs again it first
        # rebuilds its context at recompute_rate tokens per iteration, emitting nothing
        if args.recompute_rate > 0:
            for j in running - set(batch):
                if gen[j] < size[j]:
                    recompute[j] = -1                 # owed once re-admitted
            for j in batch:
                if recompute[j] == -1:
                    recompute[j] = int(math.ceil((plen[j] + gen[j]) / args.recompute_rate))
        emit = []
        for j in batch:
            if recompute[j] > 0:
                recompute[j] -= 1
                continue
            emit.append(j)
        running = set(batch)
        batch = emit
        if not batch:
            it += 1
            continue
        # one token each, then observe the jobs that emitted
        for j in batch:
            if first[j] < 0:
                first[j] = it
            gen[j] += 1
        rem = np.maximum(size[batch] - gen[batch], 0).astype(np.float64)
        score = -args.conc * np.abs(m[None, :] - rem[:, None]) / w
        shift = rs.random(len(batch)) < args.mislabel
        score[shift] = np.roll(score[shift], rs.choice([-1, 1]), axis=1)
        emb = np.zeros((len(batch), d), np.float32)
        emb[:, :k] = score
        pref = np.array([j not in observed for j in batch], np.uint8)
        t.predict(dv(W.encode(emb, "bf16").view(np.int16)), dv(np.arange(len(batch) + 1, dtype=np.int32)),
                  dv(np.array([live[j] for j in batch], np.int32)), dv(pref))
        observed.update(batch)
        fin = [j for j in batch if gen[j] >= size[j]]
        if fin:
            t.release(dv(np.array([live[j] for j in fin], np.int32)))
            for j in fin:
                done[j] = it + 1
                free.append(live.pop(j))
                running.discard(j)
                observed.discard(j)
        it += 1
    torch.cuda.synchronize()
    t.close()
    ok = done >= 0
    lat = (done - arr)[ok]
    ttft = (first - arr)[ok] + 1
    warm = int(0.2 * ok.sum())
    return {"c": c, "completed": int(ok.sum()), "iters": it, "mean_latency": float(lat[warm:].mean()),
            "mean_ttft": float(ttft[warm:].mean()), "preemptions": preempt}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=2000)
    ap.add_argument("--rate", type=float, default=3.0, help="arrivals per iteration")
    ap.add_argument("--slots", type=int, default=1024)
    ap.add_argument("--budget-frac", type=float, default=0.35)
    ap.add_argument("--conc", type=float, default=2.0)
    ap.add_argument("--mislabel", type=float, default=0.1)
    ap.add_argument("--c", default="0,0.5,0.8,inf")
    ap.add_argument("--recompute-rate", type=float, default=0.0,
                    help="discard mode: tokens of context rebuilt per iteration (0 = hold mode)")
    ap.add_argument("--seeds", type=int, default=2)
    ap.add_argument("--max-iters", type=int, default=200000)
    args = ap.parse_args()
    for cs in args.c.split(","):
        c = math.inf if cs == "inf" else float(cs)
        rows = [run(c, args, 1000 + s) for s in range(args.seeds)]
        print({"c": c, "mean_latency": float(np.mean([r["mean_latency"] for r in rows])),
               "mean_ttft": float(np.mean([r["mean_ttft"] for r in rows])),
               "preemptions": float(np.mean([r["preemptions"] for r in rows])),
               "completed": rows[0]["completed"], "iters": rows[0]["iters"]}, flush=True)


if __name__ == "__main__":
    main()
