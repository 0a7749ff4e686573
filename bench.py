#!/usr/bin/env python
"""bench.py — TRAIL predict+schedule step on B200 (BASELINE.json metric: predict+schedule
requests/s and us/iteration; % HBM/TC roofline).

One STEP = one pass of the whole hot path over one iteration's
batch: trail_predict_step for the n running requests of this GPU (gather/mean-pool,
layer 1, head with Bayes refinement and expected length) + trail_schedule_step for all
live requests (record pack, NCCL all-gather of records when N > 1, global selection).

Default workload = BASELINE.json configs[1] ("c2"): 512 requests per GPU (+128 waiting),
Llama-3-8B-shaped d = 4096 bf16 layer-11 embeddings, MLP 4096->512->10 bins, Bayesian
refinement, limited-preemption SRPT c = 0.8 under a KV-block budget.  At N > 1 every
rank holds 512 requests (configs[2] at N = 8: 4096 requests over 8 B200): weak scaling.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c1|c4] [--impl ours|reference]

Inputs are synthetic (synth/, seeded) and resident in HBM before the timed region; L2 is
flushed (256 MiB memset + 256 MiB read of another buffer) between timed steps, outside the
per-step CUDA-event brackets.
Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import workload as W  # noqa: E402

CONFIGS = {
    # name: (n per GPU, waiting per GPU, d, H, k, dtype, c, bins_total, description)
    "c2": dict(n=512, waiting=128, d=4096, H=512, k=10, dtype="bf16", c=0.8, total=512.0,
               desc="512 req/GPU, bf16 Llama-3-8B-shaped layer-11 embeddings d=4096, MLP "
                    "4096->512->10, Bayes refinement + limited-preemption SRPT c=0.8 under a "
                    "KV block budget"),
    "c1": dict(n=64, waiting=16, d=4096, H=512, k=10, dtype="f32", c=0.8, total=512.0,
               desc="64 running requests, d=4096, MLP 4096->512->10, fp32"),
    "c4": dict(n=16384, waiting=4096, d=8192, H=512, k=20, dtype="bf16", c=0.8, total=1024.0,
               burst=False, distinct=4, strong=True,
               desc="16384 requests/GPU at d=8192 (70B-shaped), 20 bins, tcgen05 GEMM regime"),
}

L1_NAMES = {1: "gemv", 2: "tcgen05 split-K (K2c)", 3: "tcgen05 unfused",
            4: "tcgen05 CTA pair (K2d)", 5: "3xTF32 tcgen05 (K2t)"}


def sm_max_mhz():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            v = json.load(f).get("sm_max_mhz")
        if v:
            return float(v)
    return 1965.0   # B200 clocks.max.sm (B200_PROFILING.md)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), float(j["bf16_tflops"]), float(j.get("bf16_tflops_sustained", j["bf16_tflops"])), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML every ~2 ms from a
    thread (the timed region is tens of ms, too short for nvidia-smi's 100 ms loop), with
    nvidia-smi as the fallback when NVML is unavailable."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.nv = None
        self.samples = []          # (sm_mhz, max_mhz, reasons)
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
            bits = {"hw_slowdown": pynvml.nvmlClocksThrottleReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksThrottleReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksThrottleReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksThrottleReasonSwPowerCap}
            mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            self.nv = (pynvml, h, bits, mx)

            def loop():
                while not self._stop.is_set():
                    sm = float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                    r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                    self.samples.append((sm, mx, {nm for nm, b in bits.items() if r & b}))
                    time.sleep(0.002)
            self._t = threading.Thread(target=loop, daemon=True)
            self._t.start()
            return self
        except Exception:
            self.nv = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first_sample(self, timeout: float = 5.0):
        t0 = time.time()
        while (self.nv or self.proc) and not (self.lines or self.samples) and \
                time.time() - t0 < timeout:
            time.sleep(0.002)

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self._t.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        for s_, m_, r_ in list(self.samples):
            sm.append(s_)
            mx = max(mx, m_)
            reasons |= r_
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml" if self.samples else "nvidia-smi"}


# ----------------------------------------------------------------------------- workload
def make_batches(cfg, nb: int, rank: int, world: int, seed: int):
    """The scripted engine (open loop): an initial burst prefill (P:570 shape: every
    request pools its prompt) that initialises the slots, then nb consecutive steady-state
    iterations (decode + the Alpaca-like trickle of completions/arrivals) that are timed."""
    # configs whose burst prefill would not fit host memory (c4: 16K prompts x 8K wide) start
    # from staggered decode ages instead (slots are first observed by their decode row, D-23)
    eng = W.EngineScript(cfg["n"], cfg["waiting"], d=cfg["d"], dtype=cfg["dtype"],
                         seed=seed + 1000 * rank, arrival_base=rank, arrival_stride=world,
                         burst_start=cfg.get("burst", True))
    init = eng.batch()
    eng.advance()
    batches = []
    for _ in range(nb):
        batches.append(eng.batch())
        eng.advance()
    return eng, init, batches


def first_prefill(b):
    """Index of the first multi-row (prompt) request of a batch — the host-side layout the
    serving engine knows (decodes first, new prefills last, as vLLM schedules), handed to the
    library as trail_set_prefill_start; n when the batch has no prompt rows."""
    cnt = np.diff(b.row_offsets)
    multi = np.nonzero(cnt > 1)[0]
    return int(multi[0]) if multi.size else int(b.n)


def to_dev(a, torch, device):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).to(device)


def algorithmic_bytes_l1(cfg, n):
    eb = 2 if cfg["dtype"] == "bf16" else 4
    return cfg["H"] * cfg["d"] * eb + n * cfg["d"] * eb


def log(*a):
    """Progress on stderr (the JSON line alone goes to stdout)."""
    print(f"[bench {time.strftime('%H:%M:%S')}]", *a, file=sys.stderr, flush=True)


def per_rank(cfg, world):
    """Requests on one rank: configs[3] (c4) is strong scaling (16 384 requests in total over
    N GPUs, BASELINE.json configs[3] 'at 1/2/4/8 GPUs'); c2/c1 are weak (n per GPU, c2 at
    N = 8 is configs[2])."""
    if cfg.get("strong"):
        return dict(cfg, n=cfg["n"] // world, waiting=cfg["waiting"] // world)
    return cfg


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    out = measure(args, args.config, rank, world, local, device, main=True)
    subs = [c for c in args.sub.split(",") if c and c != args.config]
    if subs and out is not None:
        out["sub_configs"] = {}
    for c in subs:
        o = measure(args, c, rank, world, local, device, main=False)
        if out is not None:
            out["sub_configs"][c] = {k: o[k] for k in (
                "value", "unit", "ms_per_step", "us_per_iteration", "step_us", "scaling",
                "dtype", "config", "roofline", "burst_prefill", "cpu_baseline", "e2e",
                "gpu_launches") if k in o}
            out["gpu_launches_sub"] = out.get("gpu_launches_sub", 0) + o["gpu_launches"]
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return out


def measure(args, cfg_name, rank, world, local, device, main):
    import torch
    import torch.distributed as dist

    cfg = per_rank(CONFIGS[cfg_name], world)
    log(f"{cfg_name}: building {cfg['n']} requests x {cfg['d']} inputs")
    from paper_2410_01035_b200 import (Trail, load_library, trail_comm_init,
                                       trail_nccl_unique_id, trail_plan_l1,
                                       trail_profile_enable, trail_profile_read)
    load_library()
    hbm, tf_burst, tf_sust, peak_src = peaks()

    nb = max(1, min(args.distinct, cfg.get("distinct", args.distinct), args.steps + args.warmup))
    eng, init, batches = make_batches(cfg, nb, rank, world, args.seed)
    w = W.make_weights(cfg["d"], cfg["H"], cfg["k"], cfg["dtype"],
                       edges=W.paper_bin_edges(cfg["k"], cfg["total"]), seed=args.seed)
    max_slots = eng.max_slots
    t = Trail(w, cfg["c"], max_slots, max_slots, max_slots, dtype=cfg["dtype"], device=local,
              world_size=world, id_base=rank * max_slots)
    if world > 1:
        uid = [trail_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        trail_comm_init(t.h, uid[0], rank, world)

    # device-resident inputs for every distinct iteration
    def mk(b):
        return dict(pfs=first_prefill(b), emb=to_dev(b.emb, torch, device),
                    off=to_dev(b.row_offsets, torch, device),
                    ids=to_dev(b.request_ids, torch, device),
                    pref=to_dev(b.is_prefill, torch, device),
                    sids=to_dev(b.sched_ids, torch, device),
                    arr=to_dev(b.arrival_seq, torch, device),
                    kv=to_dev(b.kv_blocks, torch, device), run=to_dev(b.is_running, torch, device),
                    budget=b.kv_budget, n=b.n, m=b.m, rows=int(b.row_offsets[-1]))
    dev = [mk(b) for b in batches]
    dev_init = mk(init)
    stream = torch.cuda.Stream(device)
    flush = L2Flush(torch, device, read=not args.write_flush)

    def step_x(x):
        t.predict(x["emb"], x["off"], x["ids"], x["pref"], stream=stream)
        t.schedule(x["sids"], x["arr"], x["kv"], x["run"], x["budget"], stream=stream)

    def step(i):
        step_x(dev[i % nb])

    log(f"{cfg_name}: inputs resident; eager warm-up")
    # burst prefill (initialises every slot), then one eager pass over the cycled batches
    with torch.cuda.stream(stream):
        step_x(dev_init)
        for i in range(nb):
            step(i)
    torch.cuda.synchronize()

    # CUDA graphs per distinct batch: clean graphs for the timed region, and a second set with
    # per-kernel event-record nodes (profile mode 2) replayed after it for the kernel times
    # (event nodes between kernels serialise them and break PDL overlap, so they are kept
    # out of the timed graphs)
    use_graph = not args.no_graph
    graphs, graphs_prof = [], []
    if use_graph:
        for i in range(nb):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                step(i)
            graphs.append(g)
        trail_profile_enable(t.h, 2)
        for i in range(nb):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                step(i)
            graphs_prof.append(g)
        trail_profile_enable(t.h, 0)
        torch.cuda.synchronize()

    def run_step(i, prof=False):
        if use_graph:
            with torch.cuda.stream(stream):
                (graphs_prof if prof else graphs)[i % nb].replay()
        else:
            with torch.cuda.stream(stream):
                step(i)

    log(f"{cfg_name}: graphs captured; timing {args.steps} steps")
    kernels = ["pool", "gemv", "umma", "head", "pack", "select", "gather"]
    for i in range(args.warmup):
        run_step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        clk.wait_first_sample()
        for i in range(args.steps):
            if not args.no_flush:
                with torch.cuda.stream(stream):
                    flush()
            ev[i][0].record(stream)
            run_step(args.warmup + i)
            ev[i][1].record(stream)
        stream.synchronize()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # per-kernel device times (same batches, same L2 flush, event nodes inside the graph)
    kern_ms = {k: [] for k in kernels}
    trail_profile_enable(t.h, 2)   # mode 2 reads the event pairs recorded by the graph nodes
    for i in range(min(args.steps, 50)):
        if not args.no_flush:
            with torch.cuda.stream(stream):
                flush()
        run_step(args.warmup + i, prof=True)
        stream.synchronize()
        for kname in kernels:
            ms, cnt = trail_profile_read(t.h, kname)
            if cnt:
                kern_ms[kname].append(ms)
    trail_profile_enable(t.h, 0)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = float(sum(step_ms))
    if world > 1:
        tt = torch.tensor([total_ms], dtype=torch.float64, device=device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_per_step = total_ms / args.steps
    n_total = cfg["n"] * world
    value = n_total / (ms_per_step / 1e3)

    # ---- roofline of the dominant kernel
    avg = {k: (sum(v) / len(v)) for k, v in kern_ms.items() if v}
    dom = max(avg, key=avg.get) if avg else None
    n_avg = float(np.mean([x["n"] for x in dev]))
    # requests the dominant layer-1 kernel processes per launch: all n, or the decode part
    # [0, first prompt) when the decode/prefill split applies (CTA-pair regime, hint given)
    n_l1 = n_avg                     # (no decode/prefill split in the bench: see DESIGN §7)
    mode, splits = trail_plan_l1(t.h, int(n_avg))
    roof = None
    if dom in ("umma", "gemv"):
        n_dom = n_l1 if dom == "umma" else n_avg
        byts = algorithmic_bytes_l1(cfg, n_dom)
        flops = 2.0 * n_dom * cfg["d"] * cfg["H"]
        t_s = avg[dom] / 1e3
        ach_bw = byts / t_s / 1e9
        ach_tf = flops / t_s / 1e12
        # at n = 512 the contraction sits at the bf16 ridge (I = 254 vs 259 flop/B): report
        # the bound whose fraction is larger
        # fp32 FFMA peak of the CUDA cores (the GEMV kernel's unit): 148 SMs x 128 FP32
        # lanes x 2 flop x SM clock; its ridge is ~11 flop/B
        alu_tf = torch.cuda.get_device_properties(device).multi_processor_count * 128 * 2 * \
            sm_max_mhz() * 1e6 / 1e12
        # 3xTF32 on the tensor cores (K2t, fp32 handles): tf32 runs at half the bf16 rate
        # (nominal ratio) and every algorithmic product costs 3 MMAs
        tf32_eff = tf_sust / 2.0 / 3.0
        if dom == "gemv" and mode == 5:
            if ach_tf / tf32_eff > ach_bw / hbm:
                roof = {"bound": "tensor", "achieved": ach_tf, "peak": tf32_eff, "unit": "TFLOP/s",
                        "frac": ach_tf / tf32_eff,
                        "peak_note": "3xTF32: sustained bf16 peak x 1/2 (tf32 nominal ratio) / 3 "
                                     "MMAs per product"}
            else:
                roof = {"bound": "hbm", "achieved": ach_bw, "peak": hbm, "unit": "GB/s",
                        "frac": ach_bw / hbm}
        elif dom == "gemv" and ach_tf / alu_tf > ach_bw / hbm:
            roof = {"bound": "alu", "achieved": ach_tf, "peak": alu_tf, "unit": "TFLOP/s",
                    "frac": ach_tf / alu_tf,
                    "peak_note": "fp32 FFMA: SMs x 128 lanes x 2 flop x max SM clock"}
        elif dom == "umma" and ach_tf / tf_sust > ach_bw / hbm:
            roof = {"bound": "tensor", "achieved": ach_tf, "peak": tf_sust, "unit": "TFLOP/s",
                    "frac": ach_tf / tf_sust}
        else:
            roof = {"bound": "hbm", "achieved": ach_bw, "peak": hbm, "unit": "GB/s",
                    "frac": ach_bw / hbm}
    elif dom == "pool":
        byts = float(np.mean([(x["rows"] + x["n"]) * cfg["d"] * (2 if cfg["dtype"] == "bf16" else 4)
                              for x in dev]))
        ach = byts / (avg[dom] / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm}
    elif dom is not None:
        # latency-bound kernel (head / select): report against the HBM roof of its bytes
        byts = 16.0 * float(np.mean([x["m"] for x in dev])) * world * 3
        ach = byts / (avg[dom] / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm}
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp) and world == 1:
        with open(tp) as f:
            tj = json.load(f)
        traffic = tj.get(dom) if cfg_name == "c2" else tj.get(f"{dom}_{cfg_name}")
    if roof is not None:
        roof.update({"kernel": dom, "peak_source": peak_src, "avg_launch_us": avg[dom] * 1e3,
                     "traffic": traffic,
                     "traffic_source": "profiles/ncu_traffic.json (ncu --set full, dram bytes "
                                       "per launch)" if traffic else None,
                     "kernel_us": {k: round(v * 1e3, 3) for k, v in avg.items()},
                     "share_of_step": avg[dom] / ms_per_step})

    # ---- burst prefill (P:570 shape): every request mean-pools its prompt rows (K1 streams
    # ~(rows + n) * d * eb bytes); reported beside the steady-state step, not in `value`
    burst = None
    if not args.no_burst and cfg.get("burst", True):
        bt = []
        trail_profile_enable(t.h, 2)
        for _ in range(5):
            a, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                flush()
                a.record(stream)
                step_x(dev_init)
                b2.record(stream)
            stream.synchronize()
            pool_ms, _ = trail_profile_read(t.h, "pool")
            bt.append((a.elapsed_time(b2), pool_ms))
        trail_profile_enable(t.h, 0)
        eb = 2 if cfg["dtype"] == "bf16" else 4
        byts = (dev_init["rows"] + dev_init["n"]) * cfg["d"] * eb
        pool_ms = statistics.median(x[1] for x in bt)
        burst = {"requests": dev_init["n"], "prompt_rows": dev_init["rows"],
                 "step_us": statistics.median(x[0] for x in bt) * 1e3,
                 "pool_us": pool_ms * 1e3, "pool_bytes": byts,
                 "pool_GBps": byts / (pool_ms / 1e3) / 1e9,
                 "pool_frac_of_hbm": byts / (pool_ms / 1e3) / 1e9 / hbm}

    # ---- end to end through the C ABI with HOST buffers (pinned), copies in the timed region
    log(f"{cfg_name}: device-timed {ms_per_step * 1e3:.1f} us/step; e2e")
    e2e = run_e2e(args, cfg, t, batches, stream, flush, torch, device, world)

    # ---- gpu launches of our kernels in the timed region
    # our kernels per step: pool + fused tcgen05 (or pool + GEMV + head) + select (+ pack when
    # the records are all-gathered)
    per_step = (2 if mode == 2 else 3) + (2 if world > 1 else 1)
    gpu_launches = per_step * args.steps

    out = None
    if rank == 0:
        log(f"{cfg_name}: e2e {e2e['ms_per_step'] * 1e3:.1f} us/step; CPU oracle baseline")
        cpu = (cpu_baseline(cfg, args, args.cpu_seconds if main else args.cpu_seconds / 3,
                            prebuilt=(eng, init, batches))
               if (world == 1 and not args.no_cpu) else None)
        st = sorted(step_ms)
        out = {
            "metric": "predict+schedule requests/s",
            "value": value,
            "unit": "requests/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "us_per_iteration": ms_per_step * 1e3,
            "step_us": {"mean": ms_per_step * 1e3, "median": 1e3 * statistics.median(st),
                        "p99": 1e3 * st[min(len(st) - 1, int(math.ceil(0.99 * len(st))) - 1)],
                        "min": 1e3 * st[0], "max": 1e3 * st[-1],
                        "note": "rank-local CUDA-event step times (value uses the max over "
                                "ranks of the total)"},
            "higher_is_better": True,
            "scaling": "strong" if cfg.get("strong") else "weak",
            "vs_baseline": None,
            "dtype": cfg["dtype"],
            "data": "synthetic (seeded; random-init probe of the paper's shape)",
            "config": {
                "workload": workload_name(cfg_name, world),
                "n_total": cfg["n"] * world, "n_per_gpu": cfg["n"], "waiting_per_gpu": cfg["waiting"], "d": cfg["d"],
                "hidden": cfg["H"], "bins": cfg["k"], "c": cfg["c"],
                "l1_kernel": L1_NAMES[mode], "l1_splits": splits,
                "l2": "flushed between timed steps, outside the step events: a 256 MiB memset "
                      "(> the 126 MB L2) then a 256 MiB read of another buffer, so the step "
                      "starts with none of its data in L2 and no dirty lines to write back"
                      if not args.no_flush else "warm",
                "cuda_graph": use_graph,

                "parallelism": f"request-sharded x{world}, replicated weights" +
                               (", NCCL all-gather of 16 B records, identical global selection"
                                if world > 1 else ""),
            },
            "roofline": roof,
            "burst_prefill": burst,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": gpu_launches,
            "clocks": clk.summary(),
        }
    t.close()
    del graphs, graphs_prof, dev, dev_init, flush
    torch.cuda.empty_cache()
    if world > 1:
        dist.barrier()
    return out


# ----------------------------------------------------------------------------- sweep
def run_sweep(args):
    """configs[4] (BASELINE.json): requests n = 1 ... 65 536 x c in
    {0, 0.5, 0.8, inf}, d = 4096 bf16, k = 10, on one GPU.  Per point: the steady-state
    predict+schedule step (n running + n/4 waiting, KV budget 0.8 x need) as CUDA graphs, L2
    flushed between timed steps, median / p99 us per step and requests/s; the layer-1
    kernel's HBM and tensor fractions (the regime crossover at n ~ 525); and the fp64 oracle
    timed on a bounded sample of the same step on the host cores, all cores and one thread
    (the cpu_baseline leg).  Parity at these points is tests/test_gpu_sweep.py."""
    import torch
    from paper_2410_01035_b200 import (Trail, load_library, trail_plan_l1, trail_profile_enable,
                                       trail_profile_read)
    load_library()
    hbm, tf_burst, tf_sust, src = peaks()
    device = torch.device("cuda", 0)
    d, k = 4096, 10
    w = W.make_weights(d, 512, k, "bf16", seed=args.seed)
    cs = [math.inf if v == "inf" else float(v) for v in args.sweep_c.split(",")]
    flush = L2Flush(torch, device)
    pts = []
    for n in [int(v) for v in args.sweep_n.split(",")]:
        log(f"sweep n={n}")
        eng = W.EngineScript(n, max(1, n // 4), d=d, dtype="bf16", seed=args.seed + n,
                             burst_start=False)
        bs = []
        for _ in range(3):
            bs.append(eng.batch())
            eng.advance()
        for c in cs:
            t = Trail(w, c, eng.max_slots, eng.max_slots, eng.max_slots, dtype="bf16")
            x = [dict(p=[to_dev(a, torch, device) for a in (b.emb, b.row_offsets, b.request_ids,
                                                              b.is_prefill)],
                      s=[to_dev(a, torch, device) for a in (b.sched_ids, b.arrival_seq,
                                                            b.kv_blocks, b.is_running)],
                      budget=b.kv_budget) for b in bs]
            stream = torch.cuda.Stream(device)
            with torch.cuda.stream(stream):
                for b in x:
                    t.predict(*b["p"], stream=stream)
                    t.schedule(*b["s"], b["budget"], stream=stream)
            torch.cuda.synchronize()
            graphs, gprof = [], []
            for prof in (0, 2):
                trail_profile_enable(t.h, prof)
                for b in x[1:]:
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=stream):
                        t.predict(*b["p"], stream=stream)
                        t.schedule(*b["s"], b["budget"], stream=stream)
                    (gprof if prof else graphs).append(g)
            trail_profile_enable(t.h, 0)
            ms = []
            for i in range(args.warmup + args.steps):
                with torch.cuda.stream(stream):
                    flush()
                    a, bb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    graphs[i % len(graphs)].replay()
                    bb.record(stream)
                stream.synchronize()
                if i >= args.warmup:
                    ms.append(a.elapsed_time(bb))
            kern = {}
            trail_profile_enable(t.h, 2)
            for i in range(10):
                with torch.cuda.stream(stream):
                    flush()
                    gprof[i % len(gprof)].replay()
                stream.synchronize()
                for kn in ("pool", "gemv", "umma", "head", "select"):
                    v, cn = trail_profile_read(t.h, kn)
                    if cn:
                        kern.setdefault(kn, []).append(v)
            trail_profile_enable(t.h, 0)
            kus = {kn: 1e3 * statistics.median(v) for kn, v in kern.items()}
            mode, splits = trail_plan_l1(t.h, int(bs[1].n))
            l1 = "gemv" if mode in (1, 5) else "umma"
            l1_us = kus.get(l1)
            byts = 512 * d * 2 + bs[1].n * d * 2
            flops = 2.0 * bs[1].n * d * 512
            st_ = sorted(ms)
            rec = {"n": n, "c": "inf" if math.isinf(c) else c, "records": int(bs[1].m),
                   "us_per_step_median": 1e3 * statistics.median(ms),
                   "us_per_step_p99": 1e3 * st_[min(len(st_) - 1, int(math.ceil(0.99 * len(st_))) - 1)],
                   "requests_per_s": n / (statistics.median(ms) / 1e3),
                   "kernel_us": {kk: round(v, 3) for kk, v in kus.items()},
                   "l1_kernel": L1_NAMES[mode],
                   "l1_bytes": byts, "l1_flops": flops,
                   "l1_hbm_frac": (byts / (l1_us / 1e6) / 1e9 / hbm) if l1_us else None,
                   "l1_tensor_frac_burst": (flops / (l1_us / 1e6) / 1e12 / tf_burst) if l1_us else None}
            if c == cs[0] and not args.no_cpu:
                cfg = dict(n=n, waiting=max(1, n // 4), d=d, H=512, k=k, dtype="bf16", c=c,
                           total=512.0)
                rec["cpu_baseline"] = cpu_baseline(cfg, args, min(args.cpu_seconds, 3.0),
                                                   prebuilt=(eng, bs[0], bs[1:]))
            pts.append(rec)
            log(json.dumps(rec))
            del graphs, gprof, x
            t.close()
            torch.cuda.empty_cache()
    return {"sweep": "BASELINE.json configs[4] on 1 GPU: d=4096 bf16, k=10, H=512, n running + "
                     "n/4 waiting, KV budget 0.8 x need, steady-state decode step",
            "peaks": {"hbm_GBps": hbm, "bf16_tflops_burst": tf_burst, "source": src},
            "l2": "flushed between timed steps (L2Flush)", "points": pts}


def workload_name(cfg_name, world):
    cfg = CONFIGS[cfg_name]
    idx = {"c1": 0, "c2": 1, "c4": 3}[cfg_name]
    extra = ""
    if world > 1:
        extra = (f" at N={world} (strong: {cfg['n']} requests in total)" if cfg.get("strong")
                 else f" / configs[2] shape at N={world} ({cfg['n']} requests per GPU)")
    return f"BASELINE configs[{idx}]{extra}: {cfg['desc']}"


class L2Flush:
    """Between timed steps: write a 256 MiB buffer (more than the 126 MB L2), then read a
    second 256 MiB buffer, which evicts the written lines (their write-back happens here,
    outside the step's events).  The step then finds none of its inputs or weights in L2 and
    no dirty lines to write back — the state after the LLM's own layers, minus their
    write-back, which belongs to those layers.  `--write-flush` keeps only the write (round
    1's flush): measured 30.8 us/step at configs[2] against 35.2 with the read (r02t), so the
    write-only flush leaves part of the step's working set reachable; the stricter flush is
    the default and every round-2 number uses it."""

    def __init__(self, torch, device, read: bool = True):
        self.w = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=device)
        self.r = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=device) if read else None
        self.acc = torch.zeros((), dtype=torch.float32, device=device)
        self.torch = torch

    def __call__(self):
        self.w.zero_()
        if self.r is not None:
            self.acc = self.r.sum()


def run_e2e(args, cfg, t, batches, stream, flush, torch, device, world):
    """Same metric through the public API with pinned HOST inputs/outputs: per step the H2D
    copy of that step's inputs, predict + schedule, and the D2H read of posteriors, expected
    lengths, counts and the three lists, all inside the per-step CUDA-event bracket.  The
    step's inputs live in ONE pinned host buffer (16-byte aligned fields) and travel in one
    copy; the outputs are views of ONE device buffer read back in one copy (the API takes
    plain pointers, so the caller chooses the layout)."""
    nb = len(batches)
    names = ("emb", "off", "ids", "pref", "sids", "arr", "kv", "run")

    def al(x):
        return (x + 15) & ~15

    host = []
    for b in batches:
        arrs = {}
        for name, arr in zip(names, (b.emb, b.row_offsets, b.request_ids, b.is_prefill,
                                     b.sched_ids, b.arrival_seq, b.kv_blocks, b.is_running)):
            a = np.ascontiguousarray(arr)
            if a.dtype == np.uint32:
                a = a.view(np.int32)
            arrs[name] = a
        offs, tot = {}, 0
        for name in names:
            offs[name] = tot
            tot = al(tot + arrs[name].nbytes)
        buf = torch.empty(tot, dtype=torch.uint8).pin_memory()
        bn = buf.numpy()
        for name in names:
            bn[offs[name]:offs[name] + arrs[name].nbytes] = arrs[name].view(np.uint8).reshape(-1)
        h = {"buf": buf, "bytes": tot, "offs": offs, "pfs": first_prefill(b),
             "meta": {nm: (arrs[nm].dtype, arrs[nm].shape) for nm in names},
             "budget": b.kv_budget, "n": b.n, "m": b.m}
        host.append(h)
    dbuf = torch.empty(max(h["bytes"] for h in host), dtype=torch.uint8, device=device)
    tdt = {np.dtype(np.uint16): torch.uint16, np.dtype(np.float32): torch.float32,
           np.dtype(np.int32): torch.int32, np.dtype(np.uint8): torch.uint8}
    # outputs: one device arena, the handle's output pointers are views of it
    k, cap, R = cfg["k"], t.run_ids.numel(), t.post.shape[0]
    osz = [al(R * k * 4), al(R * 4), 16, al(cap * 4), al(cap * 4), al(cap * 4)]
    oarena = torch.zeros(sum(osz), dtype=torch.uint8, device=device)
    o = np.cumsum([0] + osz)
    t.post = oarena[o[0]:o[0] + R * k * 4].view(torch.float32).view(R, k)
    t.L = oarena[o[1]:o[1] + R * 4].view(torch.float32)
    t.counts = oarena[o[2]:o[2] + 16].view(torch.int32)
    t.run_ids = oarena[o[3]:o[3] + cap * 4].view(torch.int32)
    t.preempt_ids = oarena[o[4]:o[4] + cap * 4].view(torch.int32)
    t.admit_ids = oarena[o[5]:o[5] + cap * 4].view(torch.int32)
    out_host = torch.empty(oarena.numel(), dtype=torch.uint8).pin_memory()

    def step(i):
        h = host[i % nb]
        dv = dbuf[: h["bytes"]]
        dv.copy_(h["buf"], non_blocking=True)
        views = {}
        for nm in names:
            dt, shp = h["meta"][nm]
            nbytes = int(np.prod(shp)) * np.dtype(dt).itemsize
            views[nm] = dv[h["offs"][nm]:h["offs"][nm] + nbytes].view(tdt[np.dtype(dt)]).view(shp)
        t.predict(views["emb"], views["off"], views["ids"], views["pref"], stream=stream)
        t.schedule(views["sids"], views["arr"], views["kv"], views["run"], h["budget"],
                   stream=stream)
        out_host.copy_(oarena, non_blocking=True)
        return h["bytes"], oarena.numel()

    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            step(i)
    torch.cuda.synchronize()
    steps = max(3, min(args.steps, 50))
    tot, h2d_b, d2h_b = 0.0, 0, 0
    for i in range(steps):
        with torch.cuda.stream(stream):
            if not args.no_flush:
                flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            h2d, d2h = step(args.warmup + i)
            b.record(stream)
        stream.synchronize()
        tot += a.elapsed_time(b)
        h2d_b += h2d
        d2h_b += d2h
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([tot], dtype=torch.float64, device=device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        tot = float(tt.item())
    ms = tot / steps
    return {"value": cfg["n"] * world / (ms / 1e3), "unit": "requests/s", "ms_per_step": ms,
            "h2d_bytes_per_step": int(h2d_b / steps), "d2h_bytes_per_step": int(d2h_b / steps),
            "steps": steps}


# ----------------------------------------------------------------------------- CPU oracle
def _threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max([i.get("num_threads", 1) for i in info] + [1])
    except Exception:
        return 1


def _subbatch(b, S):
    """The first S predicted requests of a batch and the first S + S/4 scheduled records (a
    bounded sample of the same workload for the CPU oracle; SURVEY §8(d) oracle timing)."""
    if S is None or S >= b.n:
        return b.emb, b.row_offsets, b.request_ids, b.is_prefill, b.sched_ids, b.arrival_seq, \
            b.kv_blocks, b.is_running, b.kv_budget, b.n
    ms = min(b.m, S + S // 4)
    r1 = int(b.row_offsets[S])
    frac = float(np.sum(b.kv_blocks[:ms])) / max(1.0, float(np.sum(b.kv_blocks)))
    return (b.emb[:r1], b.row_offsets[:S + 1], b.request_ids[:S], b.is_prefill[:S],
            b.sched_ids[:ms], b.arrival_seq[:ms], b.kv_blocks[:ms], b.is_running[:ms],
            int(b.kv_budget * frac), S)


def oracle_steps(cfg, args, seconds: float, max_steps: int, sample=None, prebuilt=None):
    from oracle import trail_ref as R
    nb = max(1, min(args.distinct, cfg.get("distinct", args.distinct), max_steps))
    eng, init, batches = prebuilt if prebuilt is not None else make_batches(cfg, nb, 0, 1, args.seed)
    nb = len(batches)
    w = W.make_weights(cfg["d"], cfg["H"], cfg["k"], cfg["dtype"],
                       edges=W.paper_bin_edges(cfg["k"], cfg["total"]), seed=args.seed)
    o = R.TrailOracle(W.decode(w["W1"], cfg["dtype"]), w["b1"], w["W2"], w["b2"], w["edges"],
                      cfg["c"], eng.max_slots, x_dtype=cfg["dtype"])
    e0, off0, ids0, pf0 = _subbatch(init, sample)[:4]
    o.predict_step(W.decode(e0, cfg["dtype"]), off0, ids0, pf0)   # first observations, untimed
    cache = {}

    def emb64(i, rows):   # decoded lazily (c4: 1 GB of fp64 per batch)
        if i not in cache:
            if len(cache) >= 2:
                cache.pop(next(iter(cache)))
            cache[i] = W.decode(rows, cfg["dtype"])
        return cache[i]
    times, reqs = [], 0
    t_start = time.perf_counter()
    for s in range(max_steps):
        i = s % nb
        emb, off, ids, pref, sids, arr, kv, run, budget, n = _subbatch(batches[i], sample)
        x = emb64(i, emb)
        t0 = time.perf_counter()
        o.predict_step(x, off, ids, pref)
        o.schedule_step(sids, arr, kv, run, budget)
        times.append(time.perf_counter() - t0)
        reqs += n
        if time.perf_counter() - t_start > seconds:
            break
    return times, reqs


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(cfg, args, seconds, prebuilt=None):
    """The fp64 oracle as it stands, on the host cores: all cores (BLAS threads), then one
    thread on a shorter sample (SURVEY §8(d) oracle timing)."""
    times, reqs = oracle_steps(cfg, args, seconds=seconds, max_steps=10_000, prebuilt=prebuilt)
    tot = sum(times)
    out = {"value": reqs / tot, "unit": "requests/s", "cores": _threads(), "kind": "oracle",
           "ms_per_step": 1e3 * tot / len(times), "cpu_model": cpu_model(),
           "host_cpus": os.cpu_count(),
           "sample": f"{len(times)} full steps of the same workload (numpy fp64 oracle, "
                     f"{cfg['n']} predicted + {cfg['n'] + cfg['waiting']} scheduled requests "
                     f"each), {tot:.1f} s of CPU work on {_threads()} BLAS threads"}
    try:
        from threadpoolctl import threadpool_limits
        S = 1024 if cfg["n"] > 1024 else None
        with threadpool_limits(limits=1):
            t1, r1 = oracle_steps(cfg, args, seconds=seconds / 3, max_steps=10_000, sample=S,
                                  prebuilt=prebuilt)
        out["one_thread"] = {"value": r1 / sum(t1), "unit": "requests/s", "cores": 1,
                             "ms_per_step": 1e3 * sum(t1) / len(t1),
                             "sample": f"{len(t1)} steps of " + (f"the first {S} predicted + {S + S // 4} "
                                       "scheduled requests" if S else "the full workload") +
                                       f", {sum(t1):.1f} s"}
    except Exception as e:   # noqa: BLE001 (report, do not fail the bench)
        out["one_thread"] = {"unavailable": str(e)}
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if rank != 0:
        return None
    cfg = CONFIGS[args.config]
    # each reference step is a bounded sample of the workload (<= 512 predicted requests), and
    # the run stops after ~150 s of oracle work whatever K is (steps actually timed reported)
    S = 512 if cfg["n"] > 512 else None
    times, reqs = oracle_steps(cfg, args, seconds=150.0, max_steps=args.warmup + args.steps,
                               sample=S)
    per_step = min(S, cfg["n"]) if S else cfg["n"]
    times = times[args.warmup:] if len(times) > args.warmup else times
    n_steps = len(times)
    tot = sum(times)
    ms = 1e3 * tot / n_steps
    val = per_step / (ms / 1e3)
    return {
        "impl": "reference",
        "metric": "predict+schedule requests/s", "value": val, "unit": "requests/s",
        "n_gpus": world, "steps": n_steps, "warmup": args.warmup, "ms_per_step": ms,
        "us_per_iteration": ms * 1e3, "higher_is_better": True,
        "scaling": "strong" if cfg.get("strong") else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
        "config": {"workload": workload_name(args.config, world),
                   "n_total": cfg["n"] * (1 if cfg.get("strong") else world), "n_per_gpu": cfg["n"], "waiting_per_gpu": cfg["waiting"], "d": cfg["d"],
                   "hidden": cfg["H"], "bins": cfg["k"], "c": cfg["c"],
                   "note": "the fp64 CPU oracle (oracle/trail_ref.py) is the reference arm: the "
                           "paper ships no code"},
        "cpu_baseline": {"value": val, "unit": "requests/s", "cores": _threads(), "kind": "oracle",
                         "cpu_model": cpu_model(),
                         "sample": f"{n_steps} timed steps of " +
                                   (f"the first {S} predicted + {S + S // 4} scheduled requests "
                                    "of each iteration" if S else "the full workload") +
                                   ", rank 0 only"},
        "e2e": {"value": val, "unit": "requests/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS),
                    help="headline workload (default configs[3], the largest single-GPU config)")
    ap.add_argument("--sub", default="c2,c1",
                    help="comma list of further configs reported as sub-records of the line")
    ap.add_argument("--distinct", type=int, default=16, help="distinct iterations cycled")
    ap.add_argument("--seed", type=int, default=W.MASTER_SEED)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--sweep", action="store_true", help="configs[4] sweep instead of one line")
    ap.add_argument("--sweep-n", default="1,4,16,64,256,512,1024,2048,4096,16384,65536")
    ap.add_argument("--sweep-c", default="0,0.5,0.8,inf")
    ap.add_argument("--sweep-out", default=os.path.join(ROOT, "profiles", "r02_sweep.json"))
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--write-flush", action="store_true",
                    help="flush L2 with the 256 MiB memset only (dirty lines left behind)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-burst", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        relaunch(args.gpus)
        return
    if args.sweep:
        doc = run_sweep(args)
        with open(args.sweep_out, "w") as f:
            json.dump(doc, f, indent=1)
        log(f"sweep written to {args.sweep_out}")
        return
    out = run_reference(args) if args.impl == "reference" else run_ours(args)
    if out is not None:
        print(json.dumps(out), flush=True)


def relaunch(n):
    """`python bench.py --gpus N` without torchrun: re-exec under torch.distributed.run with
    N local ranks (127.0.0.1 rendezvous), so the N-GPU line is always measured with N ranks."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    raise SystemExit(subprocess.call(cmd))


if __name__ == "__main__":
    main()
