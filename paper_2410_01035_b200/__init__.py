"""TRAIL (arXiv 2410.01035) predict+schedule hot path for B200 (sm_100a).

The compute path is libtrail.so (C ABI in include/trail.h, CUDA kernels in csrc/).  This
package holds only the ctypes binding (`trail`), the in-tree build (`_build`) and the
multi-rank orchestration helpers (`dist`).  Importing it does not load CUDA; the first
call that needs the library loads it and raises if it is missing (no CPU fallback).
"""
from .trail import (  # noqa: F401
    LIB_PATH,
    RECORD_BYTES,
    Trail,
    TrailError,
    load_library,
    trail_abi_version,
    trail_comm_init,
    trail_create,
    trail_destroy,
    trail_device_errors,
    trail_nccl_unique_id,
    trail_plan_l1,
    trail_predict_step,
    trail_predict_step_layers,
    trail_profile_enable,
    trail_profile_read,
    trail_read_state,
    trail_release,
    trail_schedule_pack,
    trail_schedule_select,
    trail_schedule_step,
    trail_set_fill_mode,
    trail_set_l1_mode,
    trail_set_prefill_start,
    trail_set_w1_l2_persist,
    trail_trace_enable,
    trail_trace_read,
)

__all__ = [n for n in dir() if n.startswith("trail_")] + ["Trail", "TrailError", "load_library"]
