"""Multi-GPU plumbing for the request-sharded path.

Each rank predicts its own shard of requests with replicated weights; the scheduling step
exchanges one 16-byte record per live request and every rank runs the identical global
selection.  Two ways to run the exchange:

  * inside the library: `init_comm()` hands rank 0's NCCL unique id to every rank (via the
    caller's torch.distributed group) and `trail_comm_init` builds the library's own NCCL
    communicator; `trail_schedule_step` then packs, all-gathers over NVLink and selects on
    the caller's stream in one call;
  * with a torch-owned collective: `schedule_torch_collective()` = `trail_schedule_pack` ->
    `torch.distributed.all_gather_into_tensor` -> `trail_schedule_select`.

Records are exchanged in fixed per-rank blocks of `cap` records (padding records carry
keybits 0xFFFFFFFF and are ignored by the selection), so every rank sends the same byte
count.  Slot ids are local to a rank; the ids in the returned lists are global
(id_base = rank * max_slots), so each rank filters the ids it owns.
"""
from __future__ import annotations

from typing import Optional

from .trail import (RECORD_BYTES, trail_comm_init, trail_nccl_unique_id, trail_schedule_pack,
                    trail_schedule_select)

PAD_WORD = -1   # int32 view of 0xFFFFFFFF


def init_comm(trail, group=None) -> None:
    """Give the handle its NCCL communicator (rank 0's unique id broadcast over `group`)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    box = [trail_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group else 0,
                               group=group)
    trail_comm_init(trail.h, box[0], rank, world)


def pad_records(records, n: int):
    """Mark records [n, cap) as padding (in place) — for records built outside the library
    (the CPU tests); trail_schedule_pack pads its own output.  int32 [cap, 4] tensor."""
    if n < records.shape[0]:
        records[n:].fill_(PAD_WORD)
    return records


def gather_records(local, group=None):
    """All-gather fixed-size record blocks (rank-major); works for nccl and gloo groups."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out = torch.empty((world * local.shape[0], local.shape[1]), dtype=local.dtype,
                      device=local.device)
    dist.all_gather_into_tensor(out, local, group=group)
    return out


def schedule_torch_collective(trail, request_ids, arrival_seq, kv_blocks, is_running,
                              kv_budget: int, max_run: int = 0, cap: Optional[int] = None,
                              group=None, stream=None):
    """pack -> torch all-gather -> select; returns (run, preempt, admit, counts) tensors."""
    import torch
    n = int(request_ids.shape[0])
    cap = int(cap or trail.max_sched)
    local = torch.empty((cap, RECORD_BYTES // 4), dtype=torch.int32, device=request_ids.device)
    trail_schedule_pack(trail.h, request_ids, arrival_seq, kv_blocks, is_running, n, cap, local,
                        stream)   # records [n, cap) are written as padding by the kernel
    allrec = gather_records(local, group)
    trail_schedule_select(trail.h, allrec, allrec.shape[0], kv_budget, max_run, trail.run_ids,
                          trail.preempt_ids, trail.admit_ids, trail.counts, stream)
    return trail.run_ids, trail.preempt_ids, trail.admit_ids, trail.counts
