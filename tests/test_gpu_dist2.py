"""World-size-2 parity of the multi-rank scheduling path on the ONE GPU a test box has
(SURVEY §8(a)5-6, §8(e)): two processes share cuda:0, each owns a shard of requests
(unequal sizes; arrival_seq = rank + 2*i; global ids = id_base + slot with
id_base = rank * max_slots) and predicts it with replicated weights.  Every step each rank
packs its records with the library (`trail_schedule_pack`, padded to max_sched by the
kernel), the blocks are all-gathered over a gloo group (CPU tensors: NCCL refuses two
ranks on one device), and each rank runs `trail_schedule_select` over the 2*max_sched
records with the global KV budget.  Checks, every step:
  * both ranks hold byte-identical records and return identical run/preempt/admit lists;
  * those lists equal `oracle.select` over the union of the shards run on the GPU's own
    keys (bit-exact), and the oracle's own fp64 keys only differ at near-ties;
  * predictions on each shard are within the BASELINE tolerance of the rank's oracle.
The run list drives which requests advance on each rank (closed loop across ranks); the
last step has an empty shard on rank 1 (all-padding block)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

WORLD = 2
SHARDS = [(96, 24), (40, 10)]       # (running, waiting) per rank: unequal shard sizes
D = 1024


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, steps, results):
    import torch.distributed as dist
    from oracle import trail_ref as R
    from paper_2410_01035_b200.trail import trail_schedule_pack, trail_schedule_select
    from synth import workload as W
    from gpu_util import assert_predict_close, dev, gpu_keys_forced, gpu_predict, make_pair

    import datetime
    import traceback
    logdir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                          "gpurun_out")
    os.makedirs(logdir, exist_ok=True)
    logf = open(os.path.join(logdir, f"dist2_rank{rank}.log"), "w")

    def log(*a):
        print(*a, file=logf, flush=True)

    log("start")
    try:
        _run(rank, port, steps, results, log, dist, R, trail_schedule_pack, trail_schedule_select,
             W, assert_predict_close, dev, gpu_keys_forced, gpu_predict, make_pair, datetime)
    except BaseException:
        log(traceback.format_exc())
        raise
    log("done")


def _run(rank, port, steps, results, log, dist, R, trail_schedule_pack, trail_schedule_select, W,
         assert_predict_close, dev, gpu_keys_forced, gpu_predict, make_pair, datetime):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD,
                            timeout=datetime.timedelta(seconds=180))
    log("process group up")
    torch.cuda.set_device(0)
    ms = max(a + b for a, b in SHARDS)        # common max_slots = max_sched = record block
    n_run, n_wait = SHARDS[rank]
    eng = W.EngineScript(n_run, n_wait, d=D, dtype="bf16", seed=60 + rank, temporal="coherent",
                         arrival_base=rank, arrival_stride=WORLD)
    w = W.make_weights(D, 512, 10, "bf16", seed=61)            # replicated weights
    t, o = make_pair(w, 0.8, ms, ms, ms, "bf16")
    t2 = type(t)(w, 0.8, ms, ms, ms, dtype="bf16", world_size=WORLD, id_base=rank * ms)
    t.close()
    t = t2
    id_base = rank * ms
    hist = []
    for step in range(steps + 1):
        log(f"step {step}")
        empty = step == steps and rank == 1
        b = eng.batch()
        qg, Lg = gpu_predict(t, b.emb, b.row_offsets, b.request_ids, b.is_prefill)
        qo, Lo = o.predict_step(W.decode(b.emb, "bf16"), b.row_offsets, b.request_ids,
                                b.is_prefill)
        assert_predict_close(qg, Lg, qo, Lo, f"rank {rank} step {step}")
        m = 0 if empty else b.m
        rec = torch.empty((ms, 4), dtype=torch.int32, device="cuda")
        trail_schedule_pack(t.h, dev(b.sched_ids), dev(b.arrival_seq), dev(b.kv_blocks),
                            dev(b.is_running), m, ms, rec)
        torch.cuda.synchronize()
        local = rec.cpu()
        allrec = torch.empty((WORLD * ms, 4), dtype=torch.int32)
        dist.all_gather_into_tensor(allrec, local)
        budget = torch.tensor([0 if empty else b.kv_budget], dtype=torch.int64)
        dist.all_reduce(budget)                                  # global KV budget
        trail_schedule_select(t.h, allrec.cuda(), WORLD * ms, int(budget.item()), 0, t.run_ids,
                              t.preempt_ids, t.admit_ids, t.counts)
        torch.cuda.synchronize()
        c = t.counts.cpu().numpy()
        lists = (t.run_ids[:c[0]].cpu().numpy().view(np.uint32).astype(np.int64),
                 t.preempt_ids[:c[1]].cpu().numpy().view(np.uint32).astype(np.int64),
                 t.admit_ids[:c[2]].cpu().numpy().view(np.uint32).astype(np.int64), int(c[3]))
        # this rank's shard as the GPU keyed it, and as the oracle keys it
        sl = slice(0, m)
        gk, gf, _ = gpu_keys_forced(t, b.sched_ids[sl], b.is_running[sl], o.prior_L)
        ok_, of_ = o.keys_and_forced(b.sched_ids[sl], b.is_running[sl])
        mine = dict(gk=gk, gf=gf, ok=ok_, of=of_, arr=b.arrival_seq[sl].astype(np.int64),
                    kv=b.kv_blocks[sl].astype(np.int64), run=b.is_running[sl].astype(np.int64),
                    gid=b.sched_ids[sl].astype(np.int64) + id_base)
        box = [None] * WORLD
        dist.all_gather_object(box, dict(shard=mine, lists=[x.tolist() if hasattr(x, "tolist")
                                                            else x for x in lists],
                                         rec=local.numpy().tobytes()))
        recs = [bx["rec"] for bx in box]
        assert np.frombuffer(b"".join(recs), np.uint32).reshape(-1, 4).tobytes() == \
            allrec.numpy().tobytes()
        assert box[0]["lists"] == box[1]["lists"], f"step {step}: ranks disagree"
        U = {k: np.concatenate([bx["shard"][k] for bx in box]) for k in mine}
        r2, p2, a2, s2 = R.select(U["gk"], U["gf"], U["arr"], U["kv"], U["run"], U["gid"],
                                  int(budget.item()))
        assert [r2.tolist(), p2.tolist(), a2.tolist(), s2] == box[0]["lists"], f"step {step}"
        r3, _, _, _ = R.select(U["ok"], U["of"], U["arr"], U["kv"], U["run"], U["gid"],
                               int(budget.item()))
        diff = set(r3.tolist()) ^ set(lists[0].tolist())
        if diff:   # near-ties only (DESIGN.md §5 outer bound 1e-3 relative; flags via argmax ties)
            pos = {int(g): i for i, g in enumerate(U["gid"])}
            free = [U["ok"][pos[int(g)]] for g in r3 if not U["of"][pos[int(g)]]]
            cut = max(free) if free else 0.0
            for g in diff:
                j = pos[int(g)]
                assert U["gf"][j] != U["of"][j] or abs(U["ok"][j] - cut) <= 1e-3 * cut, \
                    f"step {step}: gid {g} differs and is not a near-tie"
        hist.append(dict(step=step, n_run=len(lists[0]), diff=len(diff)))
        # closed loop: this rank advances the requests of ITS shard that the global run set holds
        own = [int(g) - id_base for g in lists[0] if id_base <= g < id_base + ms]
        eng.advance(np.array(own, dtype=np.int64))
    results[rank] = hist
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(420)
def test_two_process_gloo_pack_gather_select_vs_oracle():
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(_free_port(), 6, results), nprocs=WORLD, join=True)
    assert len(results[0]) == len(results[1]) == 7
    assert all(r["n_run"] > 0 for r in results[0])
