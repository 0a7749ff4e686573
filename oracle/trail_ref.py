"""TEST INFRASTRUCTURE ONLY — fp64 reference of TRAIL's predict+schedule step.

Plain definitions in the paper's order and notation; numpy fp64; one library matmul per
linear layer; no blocking, fusion or reordering.  Citations: P:<line> = PAPER.md line,
D-<n> = reading listed in DESIGN.md §2.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / reference legs may use this module.
"""
from __future__ import annotations

import math
from typing import Optional, Tuple

import numpy as np

UINT32_MAX = 0xFFFFFFFF

# status codes mirrored from include/trail.h (values are part of the ABI contract)
STATUS_OK = 0
STATUS_WARN_OVER_BUDGET = 1


# ----------------------------------------------------------------------------- bins
def bin_widths(edges: np.ndarray) -> np.ndarray:
    """w_i = b_{i+1} - b_i, the 'bin size' of P:216 (reading D-3: real width, 51.2)."""
    e = np.asarray(edges, dtype=np.float64)
    return e[1:] - e[:-1]


def bin_midpoints(edges: np.ndarray) -> np.ndarray:
    """m_i = (b_i + b_{i+1}) / 2 (= 128(2i+1)/5 for the paper's bins, 0-based, D-7)."""
    e = np.asarray(edges, dtype=np.float64)
    return (e[:-1] + e[1:]) / 2.0


def transition_matrix(edges: np.ndarray) -> np.ndarray:
    """T in [0,1]^{k x k}: T[i,i] = 1 - 1/w_i, T[i,i+1] = 1/w_{i+1} (App. A
    P:744-752).  Orientation per reading D-1: mass moves from bin B_{i+1} (longer
    remaining length) into B_i each iteration; mass leaving B_0 leaks (D-4)."""
    w = bin_widths(edges)
    k = w.shape[0]
    T = np.zeros((k, k), dtype=np.float64)
    for i in range(k):
        T[i, i] = 1.0 - 1.0 / w[i]
        if i + 1 < k:
            T[i, i + 1] = 1.0 / w[i + 1]
    return T


def prior_mean_length(edges: np.ndarray, prior: Optional[np.ndarray]) -> float:
    """E_pi[L] = sum_i pi_i m_i: the key of a request never observed (reading a4/D-9);
    256.0 for a uniform prior on the paper's bins."""
    m = bin_midpoints(edges)
    pi = np.full(m.shape[0], 1.0 / m.shape[0]) if prior is None else np.asarray(prior, np.float64)
    return float(np.sum(pi * m))


# ----------------------------------------------------------------------------- bf16
def bf16_round(v: np.ndarray) -> np.ndarray:
    """Nearest bf16 value (ties to even) of fp64 values, as fp64.  bf16 keeps 8
    significant bits; written with frexp/rint, independent of any bit-twiddling helper."""
    v = np.asarray(v, dtype=np.float64)
    out = np.zeros_like(v)
    nz = v != 0
    mant, ex = np.frexp(v[nz])                       # v = mant * 2**ex, |mant| in [0.5, 1)
    step_exp = np.maximum(ex - 8, -133)              # spacing of bf16 numbers near v
    q = np.rint(np.ldexp(v[nz], -step_exp))          # round half to even
    r = np.ldexp(q, step_exp)
    r[np.abs(r) >= 2.0 ** 128] = np.inf * np.sign(r[np.abs(r) >= 2.0 ** 128])
    out[nz] = r
    return out


# ----------------------------------------------------------------------------- predict
def pool_embedding(rows: np.ndarray, x_dtype: str) -> np.ndarray:
    """u^(0) = mean of the prompt rows at layer l (P:190 'averaging the embeddings of all
    the input tokens'); a decode observation is its single row.  The mean
    is taken in fp64 and, for bf16 inputs, rounded to bf16 before layer 1 (reading D-12)."""
    rows = np.asarray(rows, dtype=np.float64)
    u = rows.mean(axis=0)
    return bf16_round(u) if x_dtype == "bf16" else u


def classifier_logits(X: np.ndarray, W1: np.ndarray, b1: np.ndarray,
                      W2: np.ndarray, b2: np.ndarray) -> np.ndarray:
    """Two linear layers with a ReLU: h = max(0, W1 x + b1), z = W2 h + b2.
    X is [n, d]; W1 [H, d]; W2 [k, H]; all fp64."""
    H = np.maximum(0.0, X @ W1.T + b1[None, :])
    return H @ W2.T + b2[None, :]


def softmax(z: np.ndarray) -> np.ndarray:
    """p = exp(z - max z) / sum (reading D-6: CrossEntropyLoss training)."""
    z = np.asarray(z, dtype=np.float64)
    e = np.exp(z - z.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def init_posterior(p: np.ndarray, prior: np.ndarray) -> np.ndarray:
    """q^(0) = normalise(pi * p^(0)); with a uniform pi this is P:219 'Initialize
    q^(0) = p^(0)'.  A per-request pi (e.g. a BERT prompt prior) is reading D-9.  A prior
    with no mass where p has any (normaliser < 1e-300) falls back to p, as the update does
    (reading D-5)."""
    num = prior * p
    Z = num.sum(axis=-1, keepdims=True)
    safe = Z >= 1e-300
    return np.where(safe, num / np.where(safe, Z, 1.0), p)


def bayes_update(q_prev: np.ndarray, p: np.ndarray, T: np.ndarray) -> np.ndarray:
    """One refinement step, P:220-222 with reading D-2 (the prior is T applied to the
    previous *posterior*):  q_prior = T q_prev;  q(i) = q_prior(i) p(i) / sum_j ...
    Linear domain fp64; if the normaliser is < 1e-300 the update falls back to p (D-5)."""
    q_prior = q_prev @ T.T                       # row-wise T . q
    num = q_prior * p
    Z = num.sum(axis=-1, keepdims=True)
    safe = Z >= 1e-300
    return np.where(safe, num / np.where(safe, Z, 1.0), p)


def bayes_update_log(lq_prev: np.ndarray, logp: np.ndarray, T: np.ndarray) -> np.ndarray:
    """The same recursion in the log domain (used only to pin bayes_update, reading
    D-22): log q_prior(i) = log sum_j T[i,j] exp(lq(j)); lq = lnum - logsumexp(lnum)."""
    with np.errstate(divide="ignore"):
        logT = np.log(T)
    a = logT[None, :, :] + lq_prev[:, None, :]          # [n, i, j]
    mx = a.max(axis=-1, keepdims=True)
    mx = np.where(np.isfinite(mx), mx, 0.0)
    lprior = (mx + np.log(np.exp(a - mx).sum(axis=-1, keepdims=True)))[..., 0]
    lnum = lprior + logp
    m2 = lnum.max(axis=-1, keepdims=True)
    return lnum - (m2 + np.log(np.exp(lnum - m2).sum(axis=-1, keepdims=True)))


def time_update(q_prev: np.ndarray, T: np.ndarray, steps: int) -> np.ndarray:
    """Predict-every-K variant ("making predictions ... every K iterations"; SURVEY
    §8(f)3): between two observations only the transition acts, q <- normalise(T q), once
    per iteration (readings D-1/D-4; no likelihood term, reading D-25)."""
    q = np.asarray(q_prev, dtype=np.float64)
    for _ in range(int(steps)):
        q = q @ T.T
        q = q / q.sum(axis=-1, keepdims=True)
    return q


def expected_length(q: np.ndarray, m: np.ndarray) -> np.ndarray:
    """L_t = sum_i q^(t)(i) m_i."""
    return q @ m


def initial_prediction(q0: np.ndarray, m: np.ndarray) -> np.ndarray:
    """r = the middle of the predicted bin, predicted bin = argmax q^(0), lowest
    index on ties (reading D-9)."""
    return m[np.argmax(q0, axis=-1)]


def preempt_threshold(c: float, r: np.ndarray) -> np.ndarray:
    """Preemption allowed only for the first floor(C*r) iterations (D-10).
    c = inf means unlimited preemption (D-14) -> threshold UINT32_MAX."""
    r = np.asarray(r, dtype=np.float64)
    if math.isinf(c):
        return np.full(r.shape, UINT32_MAX, dtype=np.int64)
    return np.floor(c * r).astype(np.int64)


class OracleState:
    """Per-slot state the path carries between iterations (q, age a, threshold, L)."""

    def __init__(self, max_slots: int, k: int):
        self.q = np.zeros((max_slots, k), dtype=np.float64)
        self.age = np.zeros(max_slots, dtype=np.int64)
        self.thr = np.zeros(max_slots, dtype=np.int64)
        self.L = np.zeros(max_slots, dtype=np.float64)
        self.seen = np.zeros(max_slots, dtype=bool)

    def release(self, ids) -> None:
        ids = np.asarray(ids, dtype=np.int64)
        self.seen[ids] = False
        self.q[ids] = 0.0
        self.age[ids] = 0
        self.thr[ids] = 0
        self.L[ids] = 0.0


class TrailOracle:
    """fp64 oracle with the same create/predict/schedule/release roles as the C-ABI."""

    def __init__(self, W1, b1, W2, b2, edges, c: float, max_slots: int,
                 prior: Optional[np.ndarray] = None, x_dtype: str = "bf16"):
        self.W1 = np.asarray(W1, dtype=np.float64)
        self.b1 = np.asarray(b1, dtype=np.float64)
        self.W2 = np.asarray(W2, dtype=np.float64)
        self.b2 = np.asarray(b2, dtype=np.float64)
        self.edges = np.asarray(edges, dtype=np.float64)
        self.k = self.edges.shape[0] - 1
        self.m = bin_midpoints(self.edges)
        self.T = transition_matrix(self.edges)
        self.c = float(c)
        self.prior = (np.full(self.k, 1.0 / self.k) if prior is None
                      else np.asarray(prior, dtype=np.float64))
        self.prior_L = prior_mean_length(self.edges, self.prior)
        self.x_dtype = x_dtype
        self.threshold = "static"      # or "dynamic" (reading D-26)
        self.state = OracleState(max_slots, self.k)

    # ------------------------------------------------------------------ predict
    def pooled_inputs(self, emb: np.ndarray, row_offsets: np.ndarray) -> np.ndarray:
        """X[j] = pool of request j's rows [o_j, o_{j+1}) (a1)."""
        n = row_offsets.shape[0] - 1
        X = np.empty((n, emb.shape[1]), dtype=np.float64)
        for j in range(n):
            X[j] = pool_embedding(emb[row_offsets[j]:row_offsets[j + 1]], self.x_dtype)
        return X

    def prefill_chunk(self, emb: np.ndarray, row_offsets: np.ndarray, request_ids: np.ndarray,
                      is_final: np.ndarray) -> np.ndarray:
        """Chunked prefill (P:432 vLLM chunked prefill, reading D-27): the
        rows of a prompt arrive over several iterations; the pooled input is still the mean
        of ALL prompt rows.  Accumulates each chunk's rows per slot; for requests
        whose chunk is the last returns the pooled row (pool_embedding of every row seen),
        NaN rows otherwise."""
        if not hasattr(self, "_chunks"):
            self._chunks = {}
        ids = np.asarray(request_ids, dtype=np.int64)
        off = np.asarray(row_offsets, dtype=np.int64)
        out = np.full((ids.shape[0], emb.shape[1]), np.nan)
        for j, sid in enumerate(ids):
            rows = np.asarray(emb[off[j]:off[j + 1]], dtype=np.float64)
            self._chunks.setdefault(int(sid), []).append(rows)
            if is_final[j]:
                out[j] = pool_embedding(np.concatenate(self._chunks.pop(int(sid))), self.x_dtype)
        return out

    def probs(self, X: np.ndarray) -> np.ndarray:
        """p^(t) = softmax(MLP(u^(t))) (a2 + first half of a3)."""
        return softmax(classifier_logits(X, self.W1, self.b1, self.W2, self.b2))

    def mixed_inputs(self, embs, row_offsets: np.ndarray, layer_weights) -> np.ndarray:
        """Multi-layer weighted embeddings (P:194 'estimate the prediction using ... a
        weighted average of their outputs'; P:717 'leveraging multiple-layer embeddings
        through weighted averaging', reading D-28): the probe input of
        request j is u_j = sum_l a_l u_{l,j} with a = w / sum(w), where u_{l,j} is layer l's
        embedding of request j (its prompt mean at prefill; its row at decode).  Each
        layer is pooled in fp64, the weighted sum is fp64, and bf16 inputs are rounded to
        bf16 once, at the end (D-12)."""
        w = np.asarray(layer_weights, dtype=np.float64)
        a = w / w.sum()
        off = np.asarray(row_offsets, np.int64)
        n = off.shape[0] - 1
        X = np.zeros((n, np.asarray(embs[0]).shape[1]), dtype=np.float64)
        for j in range(n):
            for al, e in zip(a, embs):
                X[j] += al * np.asarray(e[off[j]:off[j + 1]], dtype=np.float64).mean(axis=0)
        return bf16_round(X) if self.x_dtype == "bf16" else X

    def predict_step_layers(self, embs, row_offsets: np.ndarray, request_ids: np.ndarray,
                            is_prefill: np.ndarray, layer_weights,
                            prior_override: Optional[np.ndarray] = None
                            ) -> Tuple[np.ndarray, np.ndarray]:
        """predict_step on the weighted average of several layers' embeddings (D-28)."""
        return self.predict_from_inputs(self.mixed_inputs(embs, row_offsets, layer_weights),
                                        request_ids, is_prefill, prior_override)

    def predict_step(self, emb: np.ndarray, row_offsets: np.ndarray, request_ids: np.ndarray,
                     is_prefill: np.ndarray, prior_override: Optional[np.ndarray] = None
                     ) -> Tuple[np.ndarray, np.ndarray]:
        """One iteration for the n requests that just ran.  emb: fp64 values [R, d]."""
        return self.predict_from_inputs(self.pooled_inputs(emb, np.asarray(row_offsets, np.int64)),
                                        request_ids, is_prefill, prior_override)

    def predict_from_inputs(self, X: np.ndarray, request_ids: np.ndarray, is_prefill: np.ndarray,
                            prior_override: Optional[np.ndarray] = None
                            ) -> Tuple[np.ndarray, np.ndarray]:
        """The classifier, softmax, Bayes step and L for given probe inputs X [n, d]."""
        ids = np.asarray(request_ids, dtype=np.int64)
        p = self.probs(X)
        st = self.state
        first = (np.asarray(is_prefill) != 0) | ~st.seen[ids]
        q = np.empty_like(p)
        if first.any():
            pri = (np.broadcast_to(self.prior, p.shape) if prior_override is None
                   else np.asarray(prior_override, dtype=np.float64))
            q0 = init_posterior(p[first], pri[first])
            q[first] = q0
            fi = ids[first]
            st.thr[fi] = preempt_threshold(self.c, initial_prediction(q0, self.m))
            st.age[fi] = 0
            st.seen[fi] = True
        dec = ~first
        if dec.any():
            di = ids[dec]
            q[dec] = bayes_update(st.q[di], p[dec], self.T)
            st.age[di] += 1                                  # reading D-11
        L = expected_length(q, self.m)
        st.q[ids] = q
        st.L[ids] = L
        return q, L

    def time_update(self, request_ids: np.ndarray, steps: int) -> Tuple[np.ndarray, np.ndarray]:
        """Iterations without an observation: observed slots get `steps`
        transitions, age a += steps (D-11), L refreshed; unobserved slots are untouched and
        report the prior pi and E_pi[L] (D-24)."""
        ids = np.asarray(request_ids, dtype=np.int64)
        st = self.state
        q = np.broadcast_to(self.prior, (ids.shape[0], self.k)).copy()
        L = np.full(ids.shape[0], self.prior_L)
        seen = st.seen[ids]
        if seen.any() and steps > 0:
            si = ids[seen]
            st.q[si] = time_update(st.q[si], self.T, steps)
            st.age[si] += int(steps)
            st.L[si] = expected_length(st.q[si], self.m)
        q[seen] = st.q[ids[seen]]
        L[seen] = st.L[ids[seen]]
        return q, L

    # ------------------------------------------------------------------ schedule
    def keys_and_forced(self, ids, is_running) -> Tuple[np.ndarray, np.ndarray]:
        """key = L_t of the slot (E_pi[L] if never observed); forced (rank -inf, P:394,
        P:830-831) iff running, observed, and age >= floor(c r) — or, with
        threshold='dynamic' (reading D-26), age >= c (age + L_t)."""
        ids = np.asarray(ids, dtype=np.int64)
        st = self.state
        key = np.where(st.seen[ids], st.L[ids], self.prior_L)
        if self.threshold == "dynamic":
            a = st.age[ids].astype(np.float64)
            frozen = a >= self.c * (a + st.L[ids]) if not math.isinf(self.c) else np.zeros(ids.shape, bool)
        else:
            frozen = st.age[ids] >= st.thr[ids]
        forced = (np.asarray(is_running) != 0) & st.seen[ids] & frozen
        return key, forced

    def schedule_step(self, ids, arrival_seq, kv_blocks, is_running, kv_budget: int,
                      max_run: int = 0, id_base: int = 0, fill: str = "prefix"):
        key, forced = self.keys_and_forced(ids, is_running)
        return select(key, forced, arrival_seq, kv_blocks, is_running,
                      np.asarray(ids, dtype=np.int64) + id_base, kv_budget, max_run, fill)

    def release(self, ids) -> None:
        """A finished (or aborted) request frees its slot: the slot is unseen again and any
        partial chunked-prefill rows it had accumulated (D-27) are dropped."""
        self.state.release(ids)
        for sid in np.asarray(ids, dtype=np.int64).ravel():
            getattr(self, "_chunks", {}).pop(int(sid), None)


def select(key, forced, arrival_seq, kv_blocks, is_running, ids, kv_budget: int,
           max_run: int = 0, fill: str = "prefix"):
    """Limited-preemption SPRPT over running + waiting requests.

    Order: forced (rank -inf) first, then ascending predicted remaining length, ties by
    arrival (FCFS; D-18), then input position (stable).  Run set = every forced
    request plus the longest prefix of the rest whose cumulative KV blocks, added to the
    forced total, stays within the budget (and whose size stays within max_run if > 0);
    stop at the first request that does not fit (D-15).  fill='first_fit' (SURVEY §8(f)3,
    the D-15 alternative): walk the whole order and take every request that still fits,
    skipping the ones that do not.  If the forced set alone violates a limit the run set is
    the forced set and the status is WARN_OVER_BUDGET (D-16).
    Returns (run_ids, preempt_ids, admit_ids, status), lists in sorted order."""
    key = np.asarray(key, dtype=np.float64)
    forced = np.asarray(forced, dtype=bool)
    arrival_seq = np.asarray(arrival_seq, dtype=np.int64)
    kv = np.asarray(kv_blocks, dtype=np.int64)
    running = np.asarray(is_running) != 0
    ids = np.asarray(ids, dtype=np.int64)
    m = key.shape[0]
    order = sorted(range(m), key=lambda j: (0 if forced[j] else 1, key[j], arrival_seq[j]))
    n_forced = int(forced.sum())
    S_f = int(kv[forced].sum())
    status = STATUS_OK
    cap = max_run if max_run > 0 else m
    if S_f > kv_budget or n_forced > cap:
        n_run = n_forced
        status = STATUS_WARN_OVER_BUDGET
    else:
        used, n_run = S_f, n_forced
        for pos in range(n_forced, m):
            j = order[pos]
            if used + kv[j] > kv_budget or n_run + 1 > cap:
                break
            used += kv[j]
            n_run += 1
    in_run = np.zeros(m, dtype=bool)
    in_run[order[:n_run]] = True
    if fill == "first_fit" and status == STATUS_OK:
        for pos in range(n_run, m):
            j = order[pos]
            if n_run + 1 > cap:
                break
            if used + kv[j] <= kv_budget:
                used += kv[j]
                n_run += 1
                in_run[j] = True
    elif fill not in ("prefix", "first_fit"):
        raise ValueError(fill)
    run = [ids[j] for j in order if in_run[j]]
    preempt = [ids[j] for j in order if running[j] and not in_run[j]]
    admit = [ids[j] for j in order if (not running[j]) and in_run[j]]
    return (np.array(run, dtype=np.int64), np.array(preempt, dtype=np.int64),
            np.array(admit, dtype=np.int64), status)
