"""N > 1 host logic on CPU with world_size-2 gloo process groups (no GPU needed).

Each rank owns a shard of requests (arrival_seq = rank + world * i: globally unique; ids
returned as rank * max_slots + slot).  The test encodes each rank's 16-byte records from
the fp64 oracle's keys with an encoder written here from the record layout in
include/trail.h, exchanges them with paper_2410_01035_b200.dist (padding + all-gather,
the same code the GPU path uses with NCCL), decodes, and checks that (a) every rank holds
byte-identical records, (b) every rank's selection is identical, and (c) it equals the
single-process selection over the union of the shards (global KV budget)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import trail_ref as R
from synth import workload as W

WORLD = 2
N_PER_RANK = 24


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def encode_records(key, forced, arrival, kv, running, gids, cap):
    rec = np.full((cap, 4), 0xFFFFFFFF, dtype=np.uint32)
    m = len(key)
    kb = np.asarray(key, np.float32).view(np.uint32) & np.uint32(0x7FFFFFFF)
    rec[:m, 0] = kb | np.where(forced, 0, 0x80000000).astype(np.uint32)
    rec[:m, 1] = arrival
    rec[:m, 2] = kv
    rec[:m, 3] = (np.asarray(gids, np.uint32) & 0x7FFFFFFF) | (np.asarray(running, np.uint32) << 31)
    return rec


def decode_records(rec):
    rec = rec[rec[:, 0] != 0xFFFFFFFF]
    key = (rec[:, 0] & 0x7FFFFFFF).view(np.float32).astype(np.float64)
    forced = (rec[:, 0] >> 31) == 0
    return key, forced, rec[:, 1], rec[:, 2], (rec[:, 3] >> 31) == 1, (rec[:, 3] & 0x7FFFFFFF)


def shard_state(rank, steps=6):
    """Run the oracle on this rank's shard for a few iterations; return its last batch,
    oracle, and engine."""
    eng = W.EngineScript(N_PER_RANK, 6, d=64, dtype="f32", seed=50 + rank, temporal="iid",
                         arrival_base=rank, arrival_stride=WORLD)
    w = W.make_weights(64, 128, 10, "f32", seed=9)   # replicated weights
    o = R.TrailOracle(w["W1"], w["b1"], w["W2"], w["b2"], w["edges"], 0.8, eng.max_slots,
                      x_dtype="f32")
    for _ in range(steps):
        b = eng.batch()
        o.predict_step(W.decode(b.emb, "f32"), b.row_offsets, b.request_ids, b.is_prefill)
        eng.advance()
    b = eng.batch()
    o.predict_step(W.decode(b.emb, "f32"), b.row_offsets, b.request_ids, b.is_prefill)
    return b, o, eng


def _worker(rank, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from paper_2410_01035_b200 import dist as tdist
    b, o, eng = shard_state(rank)
    key, forced = o.keys_and_forced(b.sched_ids, b.is_running)
    gids = b.sched_ids.astype(np.int64) + rank * eng.max_slots
    cap = eng.max_slots
    local = torch.from_numpy(encode_records(key, forced, b.arrival_seq, b.kv_blocks, b.is_running,
                                            gids, cap).view(np.int32))
    tdist.pad_records(local, b.m)
    allrec = tdist.gather_records(local).numpy().view(np.uint32)
    # the global budget is the sum of the shards' budgets (each rank knows its own)
    budget = torch.tensor([b.kv_budget], dtype=torch.int64)
    dist.all_reduce(budget)
    k2, f2, a2, kv2, r2, g2 = decode_records(allrec)
    run, pre, adm, st = R.select(k2, f2, a2, kv2, r2, g2.astype(np.int64), int(budget.item()))
    results[rank] = dict(rec=allrec.tobytes(), run=run.tolist(), pre=pre.tolist(),
                         adm=adm.tolist(), st=st, budget=int(budget.item()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gather_and_identical_global_selection():
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(_free_port(), results), nprocs=WORLD, join=True)
    r0, r1 = results[0], results[1]
    assert r0["rec"] == r1["rec"]                                  # byte-identical records
    assert (r0["run"], r0["pre"], r0["adm"], r0["st"]) == (r1["run"], r1["pre"], r1["adm"], r1["st"])
    # single-process reference over the union of the shards
    keys, forced, arr, kv, running, gids = [], [], [], [], [], []
    for rank in range(WORLD):
        b, o, eng = shard_state(rank)
        k, f = o.keys_and_forced(b.sched_ids, b.is_running)
        keys.append(k); forced.append(f); arr.append(b.arrival_seq); kv.append(b.kv_blocks)
        running.append(b.is_running); gids.append(b.sched_ids.astype(np.int64) + rank * eng.max_slots)
    run, pre, adm, st = R.select(np.concatenate(keys).astype(np.float32).astype(np.float64),
                                 np.concatenate(forced), np.concatenate(arr), np.concatenate(kv),
                                 np.concatenate(running), np.concatenate(gids), r0["budget"])
    assert r0["run"] == run.tolist() and r0["pre"] == pre.tolist() and r0["adm"] == adm.tolist()
    # arrivals are globally unique across ranks
    assert len(set(np.concatenate(arr).tolist())) == sum(len(a) for a in arr)


def test_pad_records_marks_tail():
    from paper_2410_01035_b200 import dist as tdist
    t = torch.zeros((5, 4), dtype=torch.int32)
    tdist.pad_records(t, 2)
    assert (t[:2] == 0).all() and (t[2:] == -1).all()
