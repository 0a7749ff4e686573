"""GPU checks of the multi-rank code paths on the one GPU a test box has:
  * the library's own NCCL communicator (dlopen'd libnccl, 1 rank): pack -> padded
    ncclAllGather -> select must equal the communicator-free selection bit for bit;
  * the torch-owned collective variant (pack -> all_gather_into_tensor -> select) on a
    1-rank NCCL process group, same check."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth import workload as W  # noqa: E402

from gpu_util import dev, make_pair  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _prepared_pair(seed=3):
    n, d = 128, 1024
    eng = W.EngineScript(n, d=d, dtype="bf16", seed=seed)
    w = W.make_weights(d, 512, 10, "bf16", seed=seed)
    outs = []
    for _ in range(2):
        t, _ = make_pair(w, 0.8, eng.max_slots, eng.max_slots, eng.max_slots, "bf16")
        outs.append(t)
    script = W.EngineScript(n, d=d, dtype="bf16", seed=seed)
    for _ in range(4):
        b = script.batch()
        for t in outs:
            t.predict(dev(b.emb), dev(b.row_offsets), dev(b.request_ids), dev(b.is_prefill))
        script.advance()
    b = script.batch()
    for t in outs:
        t.predict(dev(b.emb), dev(b.row_offsets), dev(b.request_ids), dev(b.is_prefill))
    torch.cuda.synchronize()
    return outs, b


def _lists(t):
    c = t.counts.cpu().numpy()
    return (t.run_ids[:c[0]].cpu().numpy().tolist(), t.preempt_ids[:c[1]].cpu().numpy().tolist(),
            t.admit_ids[:c[2]].cpu().numpy().tolist(), int(c[3]))


def test_library_nccl_path_single_rank():
    from paper_2410_01035_b200 import TrailError, trail_comm_init, trail_nccl_unique_id
    (t_plain, t_nccl), b = _prepared_pair()
    try:
        uid = trail_nccl_unique_id()
    except TrailError:
        pytest.skip("libnccl.so.2 not loadable")
    trail_comm_init(t_nccl.h, uid, 0, 1)
    args = (dev(b.sched_ids), dev(b.arrival_seq), dev(b.kv_blocks), dev(b.is_running), b.kv_budget)
    t_plain.schedule(*args)
    t_nccl.schedule(*args)
    torch.cuda.synchronize()
    assert _lists(t_plain) == _lists(t_nccl)
    assert _lists(t_plain)[0]


def test_torch_collective_path_single_rank():
    import torch.distributed as dist
    from paper_2410_01035_b200 import dist as tdist
    (t_plain, t_torch), b = _prepared_pair(seed=4)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        args = (dev(b.sched_ids), dev(b.arrival_seq), dev(b.kv_blocks), dev(b.is_running))
        t_plain.schedule(*args, b.kv_budget)
        tdist.schedule_torch_collective(t_torch, *args, b.kv_budget, cap=t_torch.max_sched)
        torch.cuda.synchronize()
        assert _lists(t_plain) == _lists(t_torch)
    finally:
        dist.destroy_process_group()
