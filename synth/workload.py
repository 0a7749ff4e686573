"""Seeded synthetic workload for the TRAIL predict+schedule path ("input recipe").

Nothing here computes any step of the method.  It draws:
  * classifier weights of the paper's shape ("first layer maps the input embedding
    to a 512-dimensional space ... second layer ... k=10 equal-width bins"; "around
    2.1 million parameters"), random-init because no trained probe exists offline;
  * layer-l hidden states of Llama-3-8B shape d=4096 ("[1,44,4096]" at prefill,
    "[1,1,4096]" per decode iteration), as i.i.d. or temporally coherent Gaussians;
  * Alpaca-like prompt/output lengths (P:432 uses 10k Alpaca prompts; P:199 example
    prompt of 44 tokens; P:201 outputs in [0,512]);
  * a scripted serving trajectory (iteration-level batches) that yields, per
    step, the flat token batch + CSR row offsets the predictor consumes and the
    (ids, arrival order, KV blocks, running flag, budget) the scheduler consumes.

Storage encodings: fp32 arrays, or bf16 as uint16 bit patterns (round-to-nearest-even
from fp32).  Both are plain input encodings, not method arithmetic.
"""
from __future__ import annotations

import dataclasses
import zlib
from typing import Dict, List, Optional

import numpy as np

MASTER_SEED = 241001035  # arXiv id 2410.01035


def rng(name: str, seed: int = MASTER_SEED, *extra: int) -> np.random.Generator:
    """Named, independent PCG64 sub-stream: SeedSequence([seed, crc32(name), *extra])."""
    ss = np.random.SeedSequence([int(seed), zlib.crc32(name.encode()), *[int(e) for e in extra]])
    return np.random.Generator(np.random.PCG64(ss))


# --------------------------------------------------------------------------- encodings
def f32_to_bf16_bits(x) -> np.ndarray:
    """fp32 -> bf16 bit pattern (uint16), round-to-nearest-even; NaN -> canonical qNaN."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    r[np.isnan(x)] = 0x7FC0
    return r


def bf16_bits_to_f32(b) -> np.ndarray:
    b = np.ascontiguousarray(np.asarray(b, dtype=np.uint16))
    return (b.astype(np.uint32) << 16).view(np.float32)


def encode(x, dtype: str) -> np.ndarray:
    """dtype 'bf16' -> uint16 bits, 'f32' -> float32."""
    if dtype == "bf16":
        return f32_to_bf16_bits(x)
    if dtype == "f32":
        return np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    raise ValueError(dtype)


def decode(a: np.ndarray, dtype: str) -> np.ndarray:
    """Storage -> exact fp64 values."""
    if dtype == "bf16":
        return bf16_bits_to_f32(a).astype(np.float64)
    return np.asarray(a, dtype=np.float32).astype(np.float64)


# --------------------------------------------------------------------------- constants
def paper_bin_edges(k: int = 10, total: float = 512.0) -> np.ndarray:
    """k equal-width bins over [0, total]: b_i = total*i/k (bin i covers
    [512i/10, 512(i+1)/10), last bin closed).  k=20,total=1024 is reading D-20."""
    return np.array([total * i / k for i in range(k + 1)], dtype=np.float64)


# --------------------------------------------------------------------------- lengths
def sample_prompt_len(g: np.random.Generator, size=None):
    """P ~ round(LogNormal(ln 32, 0.7)) clipped to [4, 512] (mean ~41; P:199 example: 44)."""
    return np.clip(np.rint(g.lognormal(np.log(32.0), 0.7, size)), 4, 512).astype(np.int64)


def sample_output_len(g: np.random.Generator, size=None):
    """N ~ round(LogNormal(ln 150, 0.9)) clipped to [1, 512] (P:201 outputs in [0,512])."""
    return np.clip(np.rint(g.lognormal(np.log(150.0), 0.9, size)), 1, 512).astype(np.int64)


# --------------------------------------------------------------------------- weights
def make_weights(d: int = 4096, H: int = 512, k: int = 10, wdtype: str = "bf16",
                 w2_scale: float = 4.0, edges: Optional[np.ndarray] = None,
                 seed: int = MASTER_SEED) -> Dict[str, np.ndarray]:
    """Random-init probe of the paper's shape: W1[H][d] ~ N(0, 2/d), b1 ~ N(0, 0.01^2),
    W2[k][H] ~ N(0, 1/H)*w2_scale, b2 = log(bin marginal of the output-length law).
    W1 is stored in `wdtype` ('bf16' bits or 'f32'); b1, W2, b2 are fp32."""
    if edges is None:
        edges = paper_bin_edges(k)
    g = rng("weights", seed, d, H, k)
    W1 = g.normal(0.0, np.sqrt(2.0 / d), size=(H, d)).astype(np.float32)
    b1 = g.normal(0.0, 0.01, size=H).astype(np.float32)
    W2 = (g.normal(0.0, np.sqrt(1.0 / H), size=(k, H)) * w2_scale).astype(np.float32)
    lens = sample_output_len(rng("b2-marginal", seed), 200_000).astype(np.float64)
    hist = np.histogram(np.clip(lens, edges[0], edges[-1]), bins=edges)[0].astype(np.float64)
    marg = (hist + 1e-3 * hist.sum() / k)
    marg /= marg.sum()
    b2 = np.log(marg).astype(np.float32)
    return {
        "W1": encode(W1, wdtype), "b1": b1, "W2": W2, "b2": b2,
        "edges": np.asarray(edges, dtype=np.float64), "wdtype": wdtype,
    }


# --------------------------------------------------------------------------- one-off inputs
def make_step_inputs(n: int, d: int, dtype: str = "bf16", prefill_frac: float = 0.0,
                     mean_prompt: Optional[int] = None, seed: int = MASTER_SEED,
                     step: int = 0, outliers: bool = False, max_rows_per_req: int = 512):
    """A single predict batch of n requests: decode requests have 1 row, prefill requests
    P_j rows (Alpaca-like, or fixed `mean_prompt`).  Rows are i.i.d. N(0,1) (the
    adversarial 'iid' temporal variant).  Returns (emb_storage, row_offsets, is_prefill)."""
    g = rng("step-inputs", seed, n, d, step)
    is_prefill = (g.random(n) < prefill_frac).astype(np.uint8)
    if mean_prompt is None:
        plen = sample_prompt_len(g, n)
    else:
        plen = np.full(n, int(mean_prompt), dtype=np.int64)
    plen = np.minimum(plen, max_rows_per_req)
    rows = np.where(is_prefill == 1, plen, 1).astype(np.int64)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(rows, out=off[1:])
    R = int(off[-1])
    x = g.standard_normal((R, d), dtype=np.float32)
    if outliers:
        ch = rng("outlier-channels", seed).choice(d, 4, replace=False)
        first = off[:-1][is_prefill == 1]
        x[np.ix_(first, ch)] = 64.0
    return encode(x, dtype), off.astype(np.int32), is_prefill


# --------------------------------------------------------------------------- trajectory
@dataclasses.dataclass
class StepBatch:
    """One iteration's inputs to trail_predict_step + trail_schedule_step."""
    emb: np.ndarray               # [R, d] storage (uint16 bf16 bits or float32)
    row_offsets: np.ndarray       # [n+1] int32 CSR
    request_ids: np.ndarray       # [n] uint32 slot ids of the requests that just ran
    is_prefill: np.ndarray        # [n] uint8
    sched_ids: np.ndarray         # [m] uint32 all live requests (running + waiting)
    arrival_seq: np.ndarray       # [m] uint32
    kv_blocks: np.ndarray         # [m] int32
    is_running: np.ndarray        # [m] uint8  (1 = was in this iteration's batch)
    kv_budget: int
    max_run: int = 0

    @property
    def n(self) -> int:
        return int(self.request_ids.shape[0])

    @property
    def m(self) -> int:
        return int(self.sched_ids.shape[0])


@dataclasses.dataclass
class _Req:
    slot: int
    arrival: int
    P: int
    N: int
    a: int = 0          # generated tokens so far
    seen: bool = False  # prefill has been observed by the predictor


class EngineScript:
    """Scripted iteration-level serving loop (burst shape P:570).

    n_running requests are in the batch, n_waiting wait.  Every step each batched request
    produces one embedding observation (its prompt rows at its first step = prefill, one
    row afterwards = decode).  After the step every batched request has generated one more
    token; finished requests (a >= N) leave and are replaced by fresh arrivals.  By
    default the batch for the next step is chosen by the script itself (open loop,
    FCFS refill plus a small scripted preemption rate so that seen requests also wait);
    `set_batch()` lets a caller drive it from a scheduler's run list (closed loop).

    KV blocks per request = ceil((P + a + 1)/16) (16-token blocks, assumption);
    budget = floor(budget_frac * sum of KV over all live requests).
    Temporal structure of the rows: 'coherent' = bf16(0.8*base_j + 0.6*noise),
    'iid' = fresh N(0,1) every step.
    """

    def __init__(self, n_running: int, n_waiting: Optional[int] = None, d: int = 4096,
                 dtype: str = "bf16", seed: int = MASTER_SEED, temporal: str = "coherent",
                 budget_frac: float = 0.8, preempt_rate: float = 0.01,
                 outliers: bool = False, burst_start: bool = True, block: int = 16,
                 max_prompt: int = 512, slot_base: int = 0, arrival_base: int = 0,
                 arrival_stride: int = 1):
        self.n_running = int(n_running)
        self.n_waiting = int(n_running // 4 if n_waiting is None else n_waiting)
        self.d, self.dtype, self.seed = int(d), dtype, int(seed)
        self.temporal, self.budget_frac = temporal, float(budget_frac)
        self.preempt_rate, self.outliers, self.block = float(preempt_rate), outliers, int(block)
        self.max_prompt = int(max_prompt)
        self.slot_base = int(slot_base)
        self.arrival_base, self.arrival_stride = int(arrival_base), int(arrival_stride)
        self.max_slots = self.n_running + self.n_waiting
        self._free: List[int] = list(range(self.max_slots - 1, -1, -1))
        self._g = rng("engine", seed, n_running, d)
        self._arrivals = 0
        self._base: Dict[int, np.ndarray] = {}
        self._out_ch = rng("outlier-channels", seed).choice(d, 4, replace=False)
        self.step_idx = 0
        self.running: List[_Req] = [self._new_req() for _ in range(self.n_running)]
        self.waiting: List[_Req] = [self._new_req() for _ in range(self.n_waiting)]
        if not burst_start:  # stagger ages so that completions are spread out
            for r in self.running:
                r.seen, r.a = True, int(self._g.integers(0, max(1, r.N)))
        self.finished = 0

    # ------------------------------------------------------------------ helpers
    def _new_req(self) -> _Req:
        slot = self._free.pop()
        arr = self.arrival_base + self._arrivals * self.arrival_stride
        self._arrivals += 1
        P = int(min(sample_prompt_len(self._g), self.max_prompt))
        N = int(sample_output_len(self._g))
        return _Req(slot=slot, arrival=arr, P=P, N=N)

    def _rows_for(self, r: _Req, nrows: int, g: np.random.Generator) -> np.ndarray:
        if self.temporal == "iid":
            return g.standard_normal((nrows, self.d), dtype=np.float32)
        base = self._base.get(r.arrival)
        if base is None:
            base = rng("base", self.seed, r.arrival).standard_normal(self.d, dtype=np.float32)
            self._base[r.arrival] = base
        noise = g.standard_normal((nrows, self.d), dtype=np.float32)
        return (0.8 * base[None, :] + 0.6 * noise).astype(np.float32)

    def kv_of(self, r: _Req) -> int:
        return -(-(r.P + r.a + 1) // self.block)

    # ------------------------------------------------------------------ the step
    def batch(self) -> StepBatch:
        """Inputs for the current iteration (does not advance the script)."""
        g = rng("engine-rows", self.seed, self.step_idx)
        rows, counts, pref = [], [], []
        for r in self.running:
            if not r.seen:
                x = self._rows_for(r, r.P, g)
                if self.outliers:
                    x[0, self._out_ch] = 64.0
                pref.append(1)
            else:
                x = self._rows_for(r, 1, g)
                pref.append(0)
            rows.append(x)
            counts.append(x.shape[0])
        X = np.concatenate(rows, axis=0) if rows else np.zeros((0, self.d), np.float32)
        off = np.zeros(len(counts) + 1, dtype=np.int64)
        np.cumsum(counts, out=off[1:])
        live = self.running + self.waiting
        kv = np.array([self.kv_of(r) for r in live], dtype=np.int64)
        return StepBatch(
            emb=encode(X, self.dtype),
            row_offsets=off.astype(np.int32),
            request_ids=np.array([self.slot_base + r.slot for r in self.running], dtype=np.uint32),
            is_prefill=np.array(pref, dtype=np.uint8),
            sched_ids=np.array([self.slot_base + r.slot for r in live], dtype=np.uint32),
            arrival_seq=np.array([r.arrival for r in live], dtype=np.uint32),
            kv_blocks=kv.astype(np.int32),
            is_running=np.array([1] * len(self.running) + [0] * len(self.waiting), dtype=np.uint8),
            kv_budget=int(np.floor(self.budget_frac * kv.sum())),
        )

    def advance(self, run_ids: Optional[np.ndarray] = None) -> None:
        """Every batched request generated one token; retire finished ones, admit new
        arrivals, and form the next batch (from `run_ids` if given, else scripted)."""
        for r in self.running:
            if r.seen:
                r.a += 1
            r.seen = True
        done = [r for r in self.running if r.a >= r.N]
        self.running = [r for r in self.running if r.a < r.N]
        for r in done:
            self._base.pop(r.arrival, None)
            self._free.append(r.slot)
            self.finished += 1
        for _ in done:
            self.waiting.append(self._new_req())
        if run_ids is not None:
            self.set_batch(run_ids)
        else:
            # scripted preemption of a few seen requests, FCFS refill from waiting
            keep = []
            for r in self.running:
                if self._g.random() < self.preempt_rate:
                    self.waiting.append(r)
                else:
                    keep.append(r)
            self.running = keep
            self.waiting.sort(key=lambda r: r.arrival)
            while len(self.running) < self.n_running and self.waiting:
                self.running.append(self.waiting.pop(0))
        self.step_idx += 1

    def set_batch(self, run_ids) -> None:
        """Closed loop: the next batch is exactly the scheduler's run list (slot ids)."""
        want = set(int(i) - self.slot_base for i in np.asarray(run_ids).ravel())
        live = self.running + self.waiting
        self.running = [r for r in live if r.slot in want]
        self.waiting = [r for r in live if r.slot not in want]
        self.waiting.sort(key=lambda r: r.arrival)
