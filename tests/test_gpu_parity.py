"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on identical
seeded inputs.  Contract: posteriors within 2e-3 absolute, expected
remaining length within 1e-3 relative, integer state (age, threshold) exact except at
argmax near-ties, selection bit-exact on the GPU's own keys."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import trail_ref as R  # noqa: E402
from synth import workload as W  # noqa: E402

from gpu_util import (assert_predict_close, dev, gpu_keys_forced, gpu_predict, gpu_schedule,  # noqa: E402
                      gpu_state, make_pair, oracle_predict, report_exemptions, top2_gap)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2410_01035_b200 import load_library
    load_library()


# ----------------------------------------------------------------------------- one step
CASES = [
    # dtype, n, d, H, k, l1_mode, prefill_frac
    ("bf16", 1, 4096, 512, 10, 1, 0.0),
    ("bf16", 7, 4096, 512, 10, 1, 0.5),
    ("bf16", 16, 4096, 512, 10, 0, 0.2),
    ("bf16", 17, 4096, 512, 10, 0, 0.2),     # AUTO -> tcgen05 GEMM, one ragged M tile
    ("bf16", 200, 4096, 512, 10, 2, 0.1),    # two M tiles, ragged tail
    ("bf16", 512, 4096, 512, 10, 0, 0.05),   # config 2 shape, full size
    ("bf16", 513, 4096, 512, 10, 2, 0.0),
    ("bf16", 300, 4096, 512, 10, 1, 0.0),    # GEMV forced at large n (request tiles loop)
    ("bf16", 1300, 1024, 512, 10, 2, 0.0),   # BN = 256 tiles
    ("bf16", 96, 8192, 512, 20, 2, 0.3),     # config 4 shape (d=8192, 20 bins)
    ("bf16", 64, 512, 256, 10, 2, 0.0),      # H = 256
    ("bf16", 40, 256, 128, 5, 2, 0.0),       # H = 128, k = 5
    ("bf16", 33, 4096, 384, 32, 2, 0.0),     # H = 384, k = 32 (every lane a bin)
    ("bf16", 512, 4096, 512, 10, 3, 0.05),   # unfused tcgen05 GEMM + separate head
    ("bf16", 200, 1024, 256, 20, 3, 0.1),
    ("bf16", 2000, 512, 512, 10, 2, 0.0),    # fused kernel, no split (S = 1), 16 M tiles
    ("bf16", 129, 8192, 512, 20, 2, 0.5),    # fused kernel, 16-CTA clusters
    ("bf16", 300, 4096, 512, 10, 4, 0.2),    # wide CTA-pair kernel: 2 pairs, ragged tail
    ("bf16", 129, 8192, 512, 20, 4, 0.5),    # wide, config 4 width, peer CTA 1 row
    ("bf16", 1000, 1024, 512, 32, 4, 0.1),   # wide, k = 32
    ("bf16", 64, 512, 512, 16, 4, 0.0),      # wide, 8 K blocks (< 2 laps of the ring), empty peer
    ("f32", 64, 4096, 512, 10, 0, 0.0),      # config 1 shape (AUTO -> fp32 GEMV K2a)
    ("f32", 64, 4096, 512, 10, 5, 0.0),      # config 1 shape on the 3xTF32 tcgen05 kernel K2t
    ("f32", 64, 4096, 512, 10, 5, 0.3),      # K2t with prompt means from xs
    ("f32", 130, 1024, 256, 20, 5, 0.1),     # K2t: 3 request blocks (ragged), 2 M tiles
    ("f32", 9, 4000, 384, 3, 5, 1.0),        # K2t: last K split past d (TMA zero fill), H = 384
    ("f32", 9, 1024, 256, 3, 1, 1.0),
]


@pytest.mark.parametrize("n,d,k,pf", [(300, 4096, 10, 0.2), (520, 8192, 20, 0.05), (260, 1024, 32, 0.5)])
def test_wide_tensor_core_layer2_matches_fused(n, d, k, pf):
    """K2d computes layer 2 on the tensor cores (3xTF32 pair MMA over an exact hi/lo split of
    h and W2); K2c computes it in fp32 FFMA.  Same bf16 inputs, same layer-1 arithmetic up to
    summation order (K2c splits K over a cluster): posteriors within 2e-5 — a plain 1xTF32
    or bf16 layer 2 misses this by two orders of magnitude — and expected lengths within
    1e-4 relative (|dL| <= sum_i |dq_i| m_i with bin middles up to ~1000: the q bound
    carried over, still 10x inside the BASELINE 1e-3)."""
    edges = W.paper_bin_edges(k) if k != 20 else W.paper_bin_edges(20, 1024.0)
    w = W.make_weights(d, 512, k, "bf16", edges=edges, seed=21 + n)
    ids = (np.arange(n) * 2 + 1).astype(np.uint32)
    outs = []
    for l1 in (4, 2):
        t, _ = make_pair(w, 0.8, max_slots=2 * n + 3, max_requests=n, max_sched=n, dtype="bf16",
                         l1_mode=l1)
        res = []
        for step in range(2):
            emb, off, pref = W.make_step_inputs(n, d, "bf16", prefill_frac=pf if step else 1.0,
                                                seed=13, step=step)
            res.append(gpu_predict(t, emb, off, ids, pref))
        outs.append(res)
        t.close()
    for (qa, La), (qb, Lb) in zip(*outs):
        assert float(np.abs(qa - qb).max()) <= 2e-5
        assert float((np.abs(La - Lb) / Lb).max()) <= 1e-4


@pytest.mark.parametrize("n,d,H,pf", [(64, 4096, 512, 0.2), (130, 1024, 256, 0.5)])
def test_tf32_split_matches_fp32_ffma(n, d, H, pf):
    """K2t's 3xTF32 product (hi*hi + hi*lo + lo*hi, exact hi/lo split) against the fp32 FFMA
    GEMV K2a on the same fp32 inputs: posteriors within 2e-5 and expected lengths within 1e-5
    relative — a plain 1xTF32 contraction (10-bit mantissas) misses this by ~100x."""
    k = 10
    w = W.make_weights(d, H, k, "f32", seed=3 + n)
    ids = (np.arange(n) * 2 + 1).astype(np.uint32)
    outs = []
    for l1 in (5, 1):
        t, _ = make_pair(w, 0.8, max_slots=2 * n + 3, max_requests=n, max_sched=n, dtype="f32",
                         l1_mode=l1)
        res = []
        for step in range(2):
            emb, off, pref = W.make_step_inputs(n, d, "f32", prefill_frac=pf if step else 1.0,
                                                seed=9, step=step)
            res.append(gpu_predict(t, emb, off, ids, pref))
        outs.append(res)
        t.close()
    for (qa, La), (qb, Lb) in zip(*outs):
        assert float(np.abs(qa - qb).max()) <= 2e-5
        assert float((np.abs(La - Lb) / Lb).max()) <= 1e-5


@pytest.mark.parametrize("dtype,n,d,H,k,l1,pf", CASES)
def test_predict_two_steps(dtype, n, d, H, k, l1, pf):
    edges = W.paper_bin_edges(k) if k != 20 else W.paper_bin_edges(20, 1024.0)
    w = W.make_weights(d, H, k, dtype, edges=edges, seed=11 + n)
    t, o = make_pair(w, 0.8, max_slots=2 * n + 3, max_requests=n, max_sched=n, dtype=dtype,
                     l1_mode=l1)
    ids = (np.arange(n) * 2 + 1).astype(np.uint32)
    for step in range(3):
        emb, off, pref = W.make_step_inputs(n, d, dtype, prefill_frac=pf if step else 1.0,
                                            seed=5, step=step)
        qg, Lg = gpu_predict(t, emb, off, ids, pref)
        qo, Lo = oracle_predict(o, emb, off, ids, pref, dtype)
        assert_predict_close(qg, Lg, qo, Lo, f"step {step}")
        st = gpu_state(t, ids)
        np.testing.assert_array_equal(st["age"], o.state.age[ids])
        near = top2_gap(o.state.q[ids]) < 2e-3
        ok = (st["thr"] == o.state.thr[ids]) | near
        assert ok.all()


def test_adversarial_iid_200_steps_log_domain():
    """D-22: confident (W2 x4), contradictory iid observations for 200 steps — the case
    that breaks a linear-domain fp32 filter — stays within tolerance of fp64."""
    n, d, k = 64, 1024, 10
    w = W.make_weights(d, 512, k, "bf16", seed=3)
    t, o = make_pair(w, 0.8, n, n, n, "bf16", l1_mode=2)
    ids = np.arange(n, dtype=np.uint32)
    worst = 0.0
    for step in range(200):
        emb, off, pref = W.make_step_inputs(n, d, "bf16", prefill_frac=1.0 if step == 0 else 0.0,
                                            seed=17, step=step)
        qg, Lg = gpu_predict(t, emb, off, ids, pref)
        qo, Lo = oracle_predict(o, emb, off, ids, pref, "bf16")
        dq, _ = assert_predict_close(qg, Lg, qo, Lo, f"step {step}")
        worst = max(worst, dq)
    assert np.all(gpu_state(t, ids)["age"] == 199)


def test_prefill_pooling_long_prompts_and_outliers():
    """Burst-prefill shape: every request pools ~44 rows; plus 512-row prompts and
    massive-activation outlier channels (fp32 accumulation, D-12)."""
    n, d = 48, 4096
    w = W.make_weights(d, 512, 10, "bf16", seed=8)
    t, o = make_pair(w, 0.5, n, n, n, "bf16")
    ids = np.arange(n, dtype=np.uint32)
    emb, off, pref = W.make_step_inputs(n, d, "bf16", prefill_frac=1.0, seed=9, outliers=True)
    qg, Lg = gpu_predict(t, emb, off, ids, pref)
    qo, Lo = oracle_predict(o, emb, off, ids, pref, "bf16")
    assert_predict_close(qg, Lg, qo, Lo)
    emb, off, pref = W.make_step_inputs(4, d, "bf16", prefill_frac=1.0, mean_prompt=512, seed=10)
    qg, Lg = gpu_predict(t, emb, off, ids[:4], pref)
    qo, Lo = oracle_predict(o, emb, off, ids[:4], pref, "bf16")
    assert_predict_close(qg, Lg, qo, Lo)


@pytest.mark.parametrize("dtype,n,d,pad,pf", [
    ("bf16", 512, 4096, 0, 1.0),      # burst prefill (P:570 shape), config 2 width
    ("bf16", 300, 4096, 64, 0.7),     # row stride > d, decode rows mixed in
    ("bf16", 160, 8192, 0, 1.0),      # config 4 width: 2 rows per 32 KB stage
    ("f32", 128, 4096, 32, 1.0),      # config 1 dtype
    ("bf16", 4000, 1024, 0, 0.05),    # decode-heavy: prompts in a few chunks of the flat batch
])
def test_bulk_pool_bit_identical_to_register_pool(dtype, n, d, pad, pf):
    """K1 bulk-copy variant (selected by the host row-count hint) against the register
    variant (hint 0) and the oracle.  All-prompt batches: both chunk the same rows in the
    same order, so bit-identical; mixed batches: the bulk kernel chunks only the rows that
    need pooling, so prompts crossing a chunk boundary may differ in the last bit."""
    from paper_2410_01035_b200.trail import trail_predict_step, trail_set_rows_hint
    H, k = 512, 20 if d == 8192 else 10
    w = W.make_weights(d, H, k, dtype, seed=21)
    emb, off, pref = W.make_step_inputs(n, d, dtype, prefill_frac=pf, seed=22)
    rows = int(off[-1])
    assert rows >= 8 * torch.cuda.get_device_properties(0).multi_processor_count
    st = np.zeros((rows, d + pad), dtype=emb.dtype)
    st[:, :d] = emb
    e, o_, i_, p_ = dev(st), dev(off), dev(np.arange(n, dtype=np.uint32)), dev(pref)
    outs = []
    for hint in (0, rows):
        t, o = make_pair(w, 0.8, n, n, n, dtype)
        trail_set_rows_hint(t.h, hint)
        trail_predict_step(t.h, e, d + pad, o_, i_, p_, None, n, t.post, t.L)
        torch.cuda.synchronize()
        outs.append((t.post[:n].cpu().numpy().copy(), t.L[:n].cpu().numpy().copy()))
        t.close()
    if pf == 1.0:
        assert outs[0][0].tobytes() == outs[1][0].tobytes()
        assert outs[0][1].tobytes() == outs[1][1].tobytes()
    else:
        assert np.abs(outs[0][0] - outs[1][0]).max() <= 1e-5
    qo, Lo = oracle_predict(o, emb, off, np.arange(n, dtype=np.uint32), pref, dtype)
    assert_predict_close(outs[1][0].astype(np.float64), outs[1][1].astype(np.float64), qo, Lo)


def test_prior_override_and_uniform_reduces_to_softmax():
    n, d, k = 32, 512, 10
    w = W.make_weights(d, 128, k, "bf16", seed=4)
    t, o = make_pair(w, 0.8, n, n, n, "bf16")
    ids = np.arange(n, dtype=np.uint32)
    rs = np.random.default_rng(0)
    pri = rs.dirichlet(np.ones(k), size=n).astype(np.float32)
    emb, off, pref = W.make_step_inputs(n, d, "bf16", prefill_frac=1.0, seed=1)
    qg, Lg = gpu_predict(t, emb, off, ids, pref, prior_override=pri)
    qo, Lo = oracle_predict(o, emb, off, ids, pref, "bf16", prior_override=pri.astype(np.float64))
    assert_predict_close(qg, Lg, qo, Lo)
    # uniform prior: q^(0) = softmax(z)
    qg2, _ = gpu_predict(t, emb, off, ids, pref)
    p = o.probs(o.pooled_inputs(W.decode(emb, "bf16"), off))
    assert np.abs(qg2 - p).max() <= 2e-3


@pytest.mark.parametrize("l1", [1, 2, 4])
def test_prior_override_zero_support_falls_back_to_p(l1):
    """Per-request priors with zeros, including rows with no mass anywhere: q^(0) falls back
    to p (reading D-5) and the threshold comes from argmax p on every head (K3 on the GEMV
    path, the K2c / K2d epilogue head) exactly as in the oracle."""
    n, d, k = 48, 1024, 10
    w = W.make_weights(d, 512, k, "bf16", seed=5)
    t, o = make_pair(w, 0.8, n, n, n, "bf16", l1_mode=l1)
    ids = np.arange(n, dtype=np.uint32)
    rs = np.random.default_rng(6)
    pri = rs.dirichlet(np.ones(k), size=n)
    pri[rs.random((n, k)) < 0.5] = 0.0
    pri[::3] = 0.0                                   # no support at all
    pri[1::3, 0] = 1.0
    pri = (pri / np.maximum(pri.sum(axis=1, keepdims=True), 1e-30)).astype(np.float32)
    emb, off, pref = W.make_step_inputs(n, d, "bf16", prefill_frac=1.0, seed=7)
    qg, Lg = gpu_predict(t, emb, off, ids, pref, prior_override=pri)
    qo, Lo = oracle_predict(o, emb, off, ids, pref, "bf16", prior_override=pri.astype(np.float64))
    assert_predict_close(qg, Lg, qo, Lo)
    gap = np.array([top2_gap(q) for q in qo])
    thr = gpu_state(t, ids)["thr"]
    ok = gap >= 2e-3
    np.testing.assert_array_equal(thr[ok], o.state.thr[ids[ok].astype(np.int64)])
    t.close()


def test_decode_on_unseen_slot_is_first_observation_and_release():
    n, d = 8, 256
    w = W.make_weights(d, 128, 10, "bf16", seed=2)
    t, o = make_pair(w, 0.8, 16, n, n, "bf16")
    ids = np.arange(n, dtype=np.uint32)
    emb, off, pref = W.make_step_inputs(n, d, "bf16", prefill_frac=0.0, seed=1)
    qg, Lg = gpu_predict(t, emb, off, ids, pref)        # all unseen -> treated as prefill (D-23)
    qo, Lo = oracle_predict(o, emb, off, ids, pref, "bf16")
    assert_predict_close(qg, Lg, qo, Lo)
    assert np.all(gpu_state(t, ids)["age"] == 0)
    t.release(torch.from_numpy(ids[:3].view(np.int32)).cuda())
    st = gpu_state(t, ids)
    assert list(st["seen"]) == [0, 0, 0] + [1] * (n - 3)


def test_bad_ids_flagged_not_fatal():
    from paper_2410_01035_b200 import trail_device_errors
    n, d = 4, 256
    w = W.make_weights(d, 128, 10, "bf16", seed=2)
    t, o = make_pair(w, 0.8, 4, n, n, "bf16")
    emb, off, pref = W.make_step_inputs(n, d, "bf16", seed=1)
    qg, Lg = gpu_predict(t, emb, off, np.array([0, 1, 2, 99], np.uint32), pref)
    assert np.isnan(Lg[3]) and np.all(np.isfinite(Lg[:3]))
    assert trail_device_errors(t.h, clear=True) & 1


def test_invalid_arguments_rejected_on_host():
    from paper_2410_01035_b200 import TrailError, trail_predict_step
    n, d = 4, 256
    w = W.make_weights(d, 128, 10, "bf16", seed=2)
    t, _ = make_pair(w, 0.8, 4, n, n, "bf16")
    x = torch.zeros((n, d), dtype=torch.bfloat16, device="cuda")
    off = torch.arange(n + 1, dtype=torch.int32, device="cuda")
    ids = torch.arange(n, dtype=torch.int32, device="cuda")
    pf = torch.zeros(n, dtype=torch.uint8, device="cuda")
    with pytest.raises(TrailError):          # n > max_requests
        trail_predict_step(t.h, x, d, off, ids, pf, None, n + 1, None, None)
    with pytest.raises(TrailError):          # emb_ld < d
        trail_predict_step(t.h, x, d - 8, off, ids, pf, None, n, None, None)
    assert trail_predict_step(t.h, x, d, off, ids, pf, None, 0, None, None) == 0   # empty


def test_deterministic_bitwise():
    n, d = 300, 4096
    w = W.make_weights(d, 512, 10, "bf16", seed=6)
    outs = []
    for _ in range(2):
        t, _ = make_pair(w, 0.8, n, n, n, "bf16")
        ids = np.arange(n, dtype=np.uint32)
        r = []
        for step in range(3):
            emb, off, pref = W.make_step_inputs(n, d, "bf16", prefill_frac=0.1, seed=2, step=step)
            r.append(gpu_predict(t, emb, off, ids, pref))
        outs.append(r)
        t.close()
    for (q1, L1), (q2, L2) in zip(*outs):
        assert q1.tobytes() == q2.tobytes() and L1.tobytes() == L2.tobytes()


def test_gemv_and_umma_agree():
    n, d = 16, 4096
    w = W.make_weights(d, 512, 10, "bf16", seed=12)
    res = []
    for mode in (1, 2, 3):
        t, _ = make_pair(w, 0.8, n, n, n, "bf16", l1_mode=mode)
        emb, off, pref = W.make_step_inputs(n, d, "bf16", prefill_frac=0.0, seed=3)
        res.append(gpu_predict(t, emb, off, np.arange(n, dtype=np.uint32), pref))
    assert np.abs(res[0][0] - res[1][0]).max() < 1e-4
    assert np.abs(res[0][0] - res[2][0]).max() < 1e-4


# ----------------------------------------------------------------------------- selection
def _records(key, forced, arrival, kv, running, ids):
    kb = np.asarray(key, np.float32).view(np.uint32).astype(np.uint64) & 0x7FFFFFFF
    kb |= np.where(forced, 0, 0x80000000).astype(np.uint64)
    rec = np.zeros((len(key), 4), np.uint32)
    rec[:, 0] = kb.astype(np.uint32)
    rec[:, 1] = arrival
    rec[:, 2] = kv
    rec[:, 3] = (np.asarray(ids, np.uint32) & 0x7FFFFFFF) | (np.asarray(running, np.uint32) << 31)
    return rec


@pytest.mark.parametrize("m", [0, 1, 2, 5, 64, 640, 1000, 2049, 4097, 16384, 20480, 65536,
                               81920])
@pytest.mark.parametrize("variant", ["ties", "distinct", "unseen", "dup"])
def test_select_bit_exact(m, variant):
    """K4 on given records vs oracle.select, bit-exact lists and counts: keys with ties
    (bin middles), distinct keys, an all-unseen burst (every non-forced key = E_pi[L] = 256,
    so FCFS decides: the round-1 tie cliff), and duplicated (key, arrival) pairs (the
    stable order falls back to input position, D-18)."""
    from paper_2410_01035_b200 import trail_schedule_select
    rs = np.random.default_rng(m + {"ties": 7, "distinct": 0, "unseen": 11, "dup": 13}[variant])
    if variant == "ties":
        key = rs.choice(W.paper_bin_edges(10)[:-1] + 25.6, size=m).astype(np.float32)
    elif variant == "unseen":
        key = np.full(m, 256.0, np.float32)
    else:
        key = rs.uniform(25.6, 486.4, size=m).astype(np.float32)
    forced = rs.random(m) < (0.02 if variant == "unseen" else 0.2)
    running = forced | (rs.random(m) < 0.6)
    arrival = rs.permutation(m).astype(np.uint32) * 3 + 5
    if variant == "dup":
        key = np.round(key / 64).astype(np.float32) * 64 + 32
        arrival = (arrival // 9).astype(np.uint32)
    kv = rs.integers(0, 40, size=m).astype(np.uint32)
    ids = rs.permutation(m).astype(np.uint32)
    budget = int(kv.sum() * 0.6)
    max_run = 0 if m % 2 else int(m * 0.7)
    w = W.make_weights(256, 128, 10, "bf16", seed=1)
    t, _ = make_pair(w, 0.8, 4, 4, max(m, 1), "bf16")
    rec = torch.from_numpy(_records(key, forced, arrival, kv, running, ids).view(np.int32)).cuda()
    trail_schedule_select(t.h, rec, m, budget, max_run, t.run_ids, t.preempt_ids, t.admit_ids,
                          t.counts)
    torch.cuda.synchronize()
    c = t.counts.cpu().numpy()
    run, pre, adm, st = R.select(key.astype(np.float64), forced, arrival, kv, running,
                                 ids.astype(np.int64), budget, max_run)
    assert c[3] == st and c[0] == len(run) and c[1] == len(pre) and c[2] == len(adm)
    np.testing.assert_array_equal(t.run_ids[:c[0]].cpu().numpy(), run)
    np.testing.assert_array_equal(t.preempt_ids[:c[1]].cpu().numpy(), pre)
    np.testing.assert_array_equal(t.admit_ids[:c[2]].cpu().numpy(), adm)


@pytest.mark.parametrize("world,m_local", [(2, 300), (8, 2560), (4, 16384)])
def test_select_padded_rank_blocks(world, m_local):
    """Records as the all-gather delivers them: `world` rank-major blocks of max_sched
    records, each with a different number of valid records followed by padding
    (trail_schedule_pack's tail).  The selection ignores the padding and equals
    oracle.select over the valid records in rank-major order."""
    from paper_2410_01035_b200 import trail_schedule_select
    rs = np.random.default_rng(world * 1000 + m_local)
    blocks, valid = [], []
    for rk in range(world):
        nv = int(rs.integers(0, m_local + 1)) if rk else m_local
        key = rs.uniform(25.6, 486.4, size=nv).astype(np.float32)
        key[rs.random(nv) < 0.2] = 256.0
        forced = rs.random(nv) < 0.15
        running = forced | (rs.random(nv) < 0.6)
        arrival = (np.arange(nv) * world + rk).astype(np.uint32)
        kv = rs.integers(0, 40, size=nv).astype(np.uint32)
        gid = (rk * m_local + np.arange(nv)).astype(np.uint32)
        rec = np.full((m_local, 4), 0xFFFFFFFF, np.uint32)
        rec[:, 2] = 0
        rec[:nv] = _records(key, forced, arrival, kv, running, gid)
        blocks.append(rec)
        valid.append((key, forced, arrival, kv, running, gid))
    allrec = np.concatenate(blocks)
    cat = [np.concatenate([v[i] for v in valid]) for i in range(6)]
    budget = int(cat[3].sum() * 0.5)
    w = W.make_weights(256, 128, 10, "bf16", seed=1)
    t = make_pair(w, 0.8, 4, 4, m_local, "bf16")[0]
    from paper_2410_01035_b200 import Trail
    t.close()
    t = Trail(w, 0.8, 4, 4, m_local, dtype="bf16", world_size=world)
    rec = torch.from_numpy(allrec.view(np.int32)).cuda()
    trail_schedule_select(t.h, rec, world * m_local, budget, 0, t.run_ids, t.preempt_ids,
                          t.admit_ids, t.counts)
    torch.cuda.synchronize()
    c = t.counts.cpu().numpy()
    run, pre, adm, st = R.select(cat[0].astype(np.float64), cat[1], cat[2], cat[3], cat[4],
                                 cat[5].astype(np.int64), budget)
    assert c[3] == st and c[0] == len(run) and c[1] == len(pre) and c[2] == len(adm)
    np.testing.assert_array_equal(t.run_ids[:c[0]].cpu().numpy(), run)
    np.testing.assert_array_equal(t.preempt_ids[:c[1]].cpu().numpy(), pre)
    np.testing.assert_array_equal(t.admit_ids[:c[2]].cpu().numpy(), adm)
    t.close()


def test_select_unseen_burst_65536_time():
    """configs[4]'s top point as a burst of never-observed arrivals: 65 536 waiting requests
    whose keys all tie at E_pi[L] (plus 16 384 running), selected in one launch within
    100 us (median of 20 CUDA-event timed launches) — the round-1 bucketed kernel's O(b^2)
    tie cluster is gone."""
    from paper_2410_01035_b200 import trail_schedule_select
    m = 81920
    rs = np.random.default_rng(5)
    key = np.full(m, 256.0, np.float32)
    key[:16384] = rs.uniform(25.6, 486.4, 16384)
    running = np.zeros(m, bool)
    running[:16384] = True
    forced = running & (rs.random(m) < 0.3)
    arrival = rs.permutation(m).astype(np.uint32) + 1000
    kv = rs.integers(1, 40, size=m).astype(np.uint32)
    ids = np.arange(m, dtype=np.uint32)
    budget = int(kv.sum() * 0.3)
    w = W.make_weights(256, 128, 10, "bf16", seed=1)
    t = make_pair(w, 0.8, 4, 4, m, "bf16")[0]
    rec = torch.from_numpy(_records(key, forced, arrival, kv, running, ids).view(np.int32)).cuda()
    times = []
    for i in range(25):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        trail_schedule_select(t.h, rec, m, budget, 0, t.run_ids, t.preempt_ids, t.admit_ids,
                              t.counts)
        b.record()
        torch.cuda.synchronize()
        if i >= 5:
            times.append(a.elapsed_time(b) * 1e3)
    c = t.counts.cpu().numpy()
    run, pre, adm, st = R.select(key.astype(np.float64), forced, arrival, kv, running,
                                 ids.astype(np.int64), budget)
    assert c[0] == len(run) and c[1] == len(pre) and c[2] == len(adm)
    np.testing.assert_array_equal(t.run_ids[:c[0]].cpu().numpy(), run)
    med = float(np.median(times))
    print(f"81920-record unseen burst selection: median {med:.1f} us")
    assert med <= 100.0, med
    t.close()


def test_select_edge_budgets():
    from paper_2410_01035_b200 import trail_schedule_select
    key = np.array([10.0, 20.0, 30.0, 40.0], np.float32)
    cases = [  # forced, kv, running, budget, max_run
        ([0, 0, 0, 0], [5, 8, 2, 1], [0, 0, 0, 0], 9, 0),     # D-15: strict prefix {A}
        ([0, 0, 0, 0], [5, 4, 2, 1], [1, 1, 1, 1], 9, 0),     # exactly at budget
        ([1, 1, 0, 0], [5, 8, 2, 1], [1, 1, 0, 1], 9, 0),     # forced over budget -> WARN
        ([1, 0, 0, 0], [1, 1, 1, 1], [1, 1, 1, 1], 100, 2),   # run cap
        ([1, 1, 1, 0], [1, 1, 1, 1], [1, 1, 1, 1], 100, 2),   # forced over cap -> WARN
        ([0, 0, 0, 0], [0, 0, 0, 0], [0, 1, 0, 1], 0, 0),     # zero kv, zero budget
        ([0, 0, 0, 0], [3, 3, 3, 3], [1, 1, 1, 1], -1, 0),    # negative budget
    ]
    w = W.make_weights(256, 128, 10, "bf16", seed=1)
    t, _ = make_pair(w, 0.8, 4, 4, 8, "bf16")
    for forced, kv, running, budget, max_run in cases:
        forced = np.array(forced, bool)
        running = np.array(running, bool)
        kv = np.array(kv, np.uint32)
        arrival = np.arange(4, dtype=np.uint32)
        ids = np.arange(4, dtype=np.uint32)
        rec = torch.from_numpy(_records(key, forced, arrival, kv, running, ids).view(np.int32)).cuda()
        trail_schedule_select(t.h, rec, 4, budget, max_run, t.run_ids, t.preempt_ids,
                              t.admit_ids, t.counts)
        torch.cuda.synchronize()
        c = t.counts.cpu().numpy()
        run, pre, adm, st = R.select(key.astype(np.float64), forced, arrival, kv, running,
                                     ids.astype(np.int64), budget, max_run)
        assert (c[0], c[1], c[2], c[3]) == (len(run), len(pre), len(adm), st)
        np.testing.assert_array_equal(t.run_ids[:c[0]].cpu().numpy(), run)


# ----------------------------------------------------------------------------- closed loop
@pytest.mark.parametrize("cfg", [
    dict(n=64, dtype="f32", c=0.8, steps=200, temporal="coherent"),   # config 1 (200 iterations)
    dict(n=512, dtype="bf16", c=0.8, steps=12, temporal="coherent"),  # config 2 shape
    dict(n=96, dtype="bf16", c=0.0, steps=40, temporal="iid"),
    dict(n=96, dtype="bf16", c=math.inf, steps=40, temporal="iid"),
    dict(n=96, dtype="bf16", c=0.5, steps=60, temporal="coherent"),
])
def test_closed_loop_trajectory(cfg):
    """GPU run list drives who advances (SURVEY §8c trajectory parity); the oracle keeps
    its own fp64 state.  Each step: predictions within tolerance; the oracle's selection on
    the GPU's own keys is bit-exact; against the oracle's keys, disagreements only at
    near-ties."""
    n, dtype, c = cfg["n"], cfg["dtype"], cfg["c"]
    d = 4096
    eng = W.EngineScript(n, d=d, dtype=dtype, seed=21, temporal=cfg["temporal"])
    w = W.make_weights(d, 512, 10, dtype, seed=21)
    t, o = make_pair(w, c, eng.max_slots, eng.max_slots, eng.max_slots, dtype)
    key_exempt = 0
    exemptions = []
    max_rl = 0.0
    q0gap = {}
    for step in range(cfg["steps"]):
        b = eng.batch()
        first = (b.is_prefill != 0) | ~o.state.seen[b.request_ids.astype(np.int64)]
        qg, Lg = gpu_predict(t, b.emb, b.row_offsets, b.request_ids, b.is_prefill)
        qo, Lo = oracle_predict(o, b.emb, b.row_offsets, b.request_ids, b.is_prefill, dtype)
        _, rl = assert_predict_close(qg, Lg, qo, Lo, f"step {step}")
        max_rl = max(max_rl, rl)
        # tie band: 4 x the observed max |dL|/L, floored 1e-6, capped 1e-3
        eps = min(1e-3, max(1e-6, 4.0 * max_rl))
        for j in np.nonzero(first)[0]:
            q0gap[int(b.request_ids[j])] = float(top2_gap(qo[j]))
        run, pre, adm, st = gpu_schedule(t, b)
        if c == 0.0:
            assert len(pre) == 0
        # bit-exact on the GPU's own keys
        gk, gf, gst = gpu_keys_forced(t, b.sched_ids, b.is_running, o.prior_L)
        r2, p2, a2, s2 = R.select(gk, gf, b.arrival_seq, b.kv_blocks, b.is_running,
                                  b.sched_ids.astype(np.int64), b.kv_budget)
        np.testing.assert_array_equal(run, r2)
        np.testing.assert_array_equal(pre, p2)
        np.testing.assert_array_equal(adm, a2)
        assert st == s2
        # against the oracle's own keys: only near-tie differences
        ok_, of_ = o.keys_and_forced(b.sched_ids, b.is_running)
        r3, _, _, _ = R.select(ok_, of_, b.arrival_seq, b.kv_blocks, b.is_running,
                               b.sched_ids.astype(np.int64), b.kv_budget)
        # forced flags may differ only through an argmax near-tie of q^(0) (contract iii)
        for j in np.nonzero(gf != of_)[0]:
            gap = q0gap.get(int(b.sched_ids[j]), 0.0)
            assert gap < 2e-3, f"step {step}: forced flag"
            exemptions.append(dict(step=step, kind="forced", id=int(b.sched_ids[j]), q0_top2_gap=gap))
        if set(r3) != set(run):
            diff = set(r3) ^ set(run)
            pos = {int(s): i for i, s in enumerate(b.sched_ids)}
            free = [ok_[pos[int(s)]] for s in r3 if not of_[pos[int(s)]]]
            cut = max(free) if free else 0.0
            key_only = False
            for s in diff:
                j = pos[int(s)]
                near_forced = gf[j] != of_[j] or any(gf[pos[int(x)]] != of_[pos[int(x)]]
                                                     for x in diff)
                near_key = abs(ok_[j] - cut) <= eps * max(cut, 1.0)
                assert near_key or near_forced, f"step {step}: id {s} not a near-tie"
                key_only |= not near_forced
                exemptions.append(dict(step=step, kind="forced" if near_forced else "key",
                                       id=int(s), rel_gap_to_cut=float(abs(ok_[j] - cut) / max(cut, 1.0)),
                                       band=eps))
            key_exempt += int(key_only)
        eng.advance(run)
    # every exemption is reported, every exempted gap is inside the tie band
    # (asserted above), and their number is bounded (at most half the steps —
    # collapsed posteriors put several requests at the same bin middle to within 1e-7, where
    # the fp32 and fp64 orders are arbitrary; measured 60 of 200 steps at configs[0])
    report_exemptions(f"closed_loop_{cfg['n']}_{cfg['dtype']}_c{cfg['c']}_{cfg['temporal']}",
                      dict(cfg={k: (str(v) if isinstance(v, float) and math.isinf(v) else v)
                                for k, v in cfg.items()},
                           key_exempt_steps=key_exempt, max_rel_dL=max_rl,
                           tie_band=min(1e-3, max(1e-6, 4 * max_rl)), exemptions=exemptions))
    assert key_exempt <= max(2, cfg["steps"] // 2), (key_exempt, exemptions)


def test_cuda_graph_capture_matches_eager():
    n, d = 256, 4096
    w = W.make_weights(d, 512, 10, "bf16", seed=31)
    eng = W.EngineScript(n, d=d, dtype="bf16", seed=31)
    b = eng.batch()
    res = []
    for use_graph in (False, True):
        t, _ = make_pair(w, 0.8, eng.max_slots, eng.max_slots, eng.max_slots, "bf16")
        from gpu_util import dev
        args = dict(emb=dev(b.emb), off=dev(b.row_offsets), ids=dev(b.request_ids),
                    pref=dev(b.is_prefill))
        sargs = [dev(b.sched_ids), dev(b.arrival_seq), dev(b.kv_blocks), dev(b.is_running)]

        def step():
            t.predict(args["emb"], args["off"], args["ids"], args["pref"])
            t.schedule(*sargs, b.kv_budget)
        if use_graph:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                step()                     # warm-up (prefill) outside the graph
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step()
            g.replay()
        else:
            step()
            step()
        torch.cuda.synchronize()
        c0 = int(t.counts[0].item())
        res.append((t.L[:n].cpu().numpy().copy(), t.run_ids[:c0].cpu().numpy().copy(),
                    t.counts.cpu().numpy().copy()))
    for a, bb in zip(res[0], res[1]):
        np.testing.assert_array_equal(a, bb)


# ----------------------------------------------------------------------------- time update
@pytest.mark.parametrize("dtype,n,d,k", [("bf16", 200, 4096, 10), ("f32", 48, 1024, 20),
                                         ("bf16", 37, 512, 32)])
def test_time_update_predict_every_k(dtype, n, d, k):
    """Predict every K iterations: observed requests get a predict step, the rest
    only the transition (trail_time_update, K6).  Posteriors, L, age and the schedule keys
    match the oracle after a mixed sequence of gaps; unobserved slots report the prior."""
    from paper_2410_01035_b200.trail import trail_time_update
    edges = W.paper_bin_edges(k) if k != 20 else W.paper_bin_edges(20, 1024.0)
    w = W.make_weights(d, 512 if d >= 1024 else 128, k, dtype, edges=edges, seed=31)
    t, o = make_pair(w, 0.8, n + 8, n, n + 8, dtype)
    ids = np.arange(n, dtype=np.uint32)
    emb, off, pref = W.make_step_inputs(n, d, dtype, prefill_frac=1.0, seed=32)
    gpu_predict(t, emb, off, ids, pref)
    oracle_predict(o, emb, off, ids, pref, dtype)
    rs = np.random.default_rng(33)
    for it in range(6):
        obs = rs.random(n) < 0.4
        steps = int(rs.integers(1, 5))
        lag = ids[~obs]
        if lag.size:
            post = torch.empty((lag.size, k), dtype=torch.float32, device="cuda")
            Lg = torch.empty(lag.size, dtype=torch.float32, device="cuda")
            trail_time_update(t.h, dev(lag), lag.size, steps, post, Lg)
            torch.cuda.synchronize()
            qo, Lo = o.time_update(lag, steps)
            assert_predict_close(post.cpu().numpy().astype(np.float64),
                                 Lg.cpu().numpy().astype(np.float64), qo, Lo, f"time update {it}")
        ob = ids[obs]
        if ob.size:
            emb, off, pref = W.make_step_inputs(ob.size, d, dtype, prefill_frac=0.0, seed=40 + it)
            qg, Lg2 = gpu_predict(t, emb, off, ob, pref)
            qo, Lo = oracle_predict(o, emb, off, ob, pref, dtype)
            assert_predict_close(qg, Lg2, qo, Lo, f"observation {it}")
        st = gpu_state(t, ids)
        np.testing.assert_array_equal(st["age"], o.state.age[ids])
    # unobserved slots: prior and E_pi[L]; no state change
    extra = np.arange(n, n + 4, dtype=np.uint32)
    post = torch.empty((4, k), dtype=torch.float32, device="cuda")
    Lg = torch.empty(4, dtype=torch.float32, device="cuda")
    trail_time_update(t.h, dev(extra), 4, 3, post, Lg)
    torch.cuda.synchronize()
    qo, Lo = o.time_update(extra, 3)
    assert np.abs(post.cpu().numpy() - qo).max() <= 1e-6
    assert np.abs(Lg.cpu().numpy() - Lo).max() <= 1e-3 * Lo.max()
    assert not gpu_state(t, extra)["seen"].any()
    t.close()


@pytest.mark.parametrize("c,l1", [(0.5, 0), (0.25, 4), (0.3, 1)])
def test_dynamic_threshold_mode(c, l1):
    """Dynamic-threshold variant (trail_set_threshold_mode 1, reading D-26): forced iff
    a >= c (a + L_t), re-evaluated by every kernel that refreshes L_t (head, fused, wide,
    time update).  Forced flags match the oracle except within the fp32 band of the
    boundary; the selection is bit-exact on the GPU's own keys and flags."""
    from paper_2410_01035_b200.trail import trail_set_threshold_mode
    n, d, k = 300, 1024, 10
    w = W.make_weights(d, 512, k, "bf16", seed=51)
    t, o = make_pair(w, c, n, n, n, "bf16", l1_mode=l1)
    trail_set_threshold_mode(t.h, 1)
    o.threshold = "dynamic"
    ids = np.arange(n, dtype=np.uint32)
    emb, off, pref = W.make_step_inputs(n, d, "bf16", prefill_frac=1.0, seed=52)
    gpu_predict(t, emb, off, ids, pref)
    oracle_predict(o, emb, off, ids, pref, "bf16")
    rs = np.random.default_rng(53)
    running = (rs.random(n) < 0.85).astype(np.uint8)
    arrival = rs.permutation(n).astype(np.uint32)
    kv = rs.integers(1, 40, n).astype(np.int32)
    n_forced = 0
    for it in range(40):
        if it % 3 == 2:
            t.time_update(dev(ids), 5)
            torch.cuda.synchronize()
            o.time_update(ids, 5)
        else:
            emb, off, pref = W.make_step_inputs(n, d, "bf16", prefill_frac=0.0, seed=60 + it)
            gpu_predict(t, emb, off, ids, pref)
            oracle_predict(o, emb, off, ids, pref, "bf16")
        key, forced, st = gpu_keys_forced(t, ids, running, o.prior_L)
        _, fo = o.keys_and_forced(ids, running)
        a, L = o.state.age[ids].astype(np.float64), o.state.L[ids]
        near = np.abs(a * (1 - c) - c * L) <= 4e-3 * c * L + 1e-6
        assert np.all((forced == fo) | near), it
        n_forced += int(forced.sum())
        run, pre, adm, cnt = t.schedule(dev(ids), dev(arrival), dev(kv), dev(running),
                                        int(0.6 * kv.sum()))
        torch.cuda.synchronize()
        cc = cnt.cpu().numpy()
        r_o, p_o, a_o, s_o = R.select(key, forced, arrival, kv, running, ids.astype(np.int64),
                                      int(0.6 * kv.sum()), 0)
        np.testing.assert_array_equal(run[:cc[0]].cpu().numpy(), r_o)
        np.testing.assert_array_equal(pre[:cc[1]].cpu().numpy(), p_o)
        assert cc[3] == s_o
    assert n_forced > 0
    t.close()


@pytest.mark.parametrize("l1", [1, 2, 4])
def test_log_spaced_bins(l1):
    """Log-spaced bins: unequal widths w_i give a non-uniform T
    (T_ii = 1 - 1/w_i, T_i,i+1 = 1/w_{i+1}); every layer-1 kernel + head path follows the
    oracle over a prefill and 30 decode steps with time updates in between."""
    edges = np.array([0.0, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048])
    k, n, d = edges.size - 1, 96, 1024
    w = W.make_weights(d, 512, k, "bf16", edges=edges, seed=71)
    t, o = make_pair(w, 0.5, n, n, n, "bf16", l1_mode=l1)
    ids = np.arange(n, dtype=np.uint32)
    for step in range(31):
        emb, off, pref = W.make_step_inputs(n, d, "bf16", prefill_frac=1.0 if step == 0 else 0.0,
                                            seed=72, step=step)
        qg, Lg = gpu_predict(t, emb, off, ids, pref)
        qo, Lo = oracle_predict(o, emb, off, ids, pref, "bf16")
        assert_predict_close(qg, Lg, qo, Lo, f"step {step}")
        if step % 10 == 9:
            post, L = t.time_update(dev(ids), 3)
            torch.cuda.synchronize()
            qo, Lo = o.time_update(ids, 3)
            assert_predict_close(post.cpu().numpy().astype(np.float64),
                                 L.cpu().numpy().astype(np.float64), qo, Lo, f"time update {step}")
    np.testing.assert_array_equal(gpu_state(t, ids)["age"], o.state.age[ids])
    t.close()


@pytest.mark.parametrize("dtype,d,l1", [("bf16", 4096, 0), ("f32", 1024, 0), ("bf16", 1024, 4)])
def test_chunked_prefill(dtype, d, l1):
    """Chunked prefill (trail_prefill_chunk, reading D-27): prompts split into 1-4 chunks over
    successive calls, interleaved across requests; the finalised pooled rows equal the mean
    of all prompt rows (within one bf16 ulp / fp32 rounding of the oracle's fp64 mean) and
    the prediction made from them matches the oracle."""
    from paper_2410_01035_b200.trail import trail_prefill_chunk
    n, k = 60, 10
    w = W.make_weights(d, 512, k, dtype, seed=81)
    t, o = make_pair(w, 0.8, n, n, n, dtype, l1_mode=l1)
    rs = np.random.default_rng(82)
    plen = rs.integers(1, 200, n)
    nchunks = rs.integers(1, 5, n)
    full = [W.make_step_inputs(1, d, dtype, prefill_frac=1.0, mean_prompt=int(plen[j]),
                               seed=83 + j)[0] for j in range(n)]
    cuts = [np.unique(np.concatenate([[0, plen[j]], rs.integers(1, max(2, plen[j]), nchunks[j] - 1)]))
            for j in range(n)]
    pooled_all = np.zeros((n, d), dtype=full[0].dtype)
    ref_all = np.zeros((n, d))
    rnd = 0
    pending = set(range(n))
    while pending:
        js = sorted(j for j in pending if rnd < len(cuts[j]) - 1)
        if not js:
            break
        rows, off, fin = [], [0], []
        for j in js:
            a, b = cuts[j][rnd], cuts[j][rnd + 1]
            rows.append(full[j][a:b])
            off.append(off[-1] + (b - a))
            fin.append(1 if rnd + 2 == len(cuts[j]) else 0)
        emb = np.concatenate(rows)
        off, fin = np.array(off, np.int32), np.array(fin, np.uint8)
        ids = np.array(js, np.uint32)
        pooled = torch.empty((len(js), d), dtype=torch.uint16 if dtype == "bf16" else torch.float32,
                             device="cuda")
        trail_prefill_chunk(t.h, dev(emb), d, dev(off), dev(ids), dev(fin), len(js), pooled, d)
        torch.cuda.synchronize()
        ref = o.prefill_chunk(W.decode(emb, dtype), off, ids, fin)
        pg = pooled.cpu().numpy()
        for q, j in enumerate(js):
            if fin[q]:
                pooled_all[j] = pg[q].view(pooled_all.dtype) if dtype == "bf16" else pg[q]
                ref_all[j] = ref[q]
                pending.discard(j)
        rnd += 1
    assert not pending
    got = W.decode(pooled_all, dtype)
    tol = np.abs(ref_all) * (2.0 ** -7 if dtype == "bf16" else 1e-5) + 1e-6
    assert np.all(np.abs(got - ref_all) <= tol)
    # predict from the pooled rows (one-row prefill observations) vs the oracle on its own
    ids = np.arange(n, dtype=np.uint32)
    off1 = np.arange(n + 1, dtype=np.int32)
    pref = np.ones(n, np.uint8)
    qg, Lg = gpu_predict(t, pooled_all, off1, ids, pref)
    ref_store = W.encode(ref_all.astype(np.float32), dtype) if dtype == "bf16" else ref_all.astype(np.float32)
    qo, Lo = oracle_predict(o, ref_store, off1, ids, pref, dtype)
    assert_predict_close(qg, Lg, qo, Lo, "chunked prefill")
    t.close()


@pytest.mark.parametrize("dtype,d", [("bf16", 1024), ("f32", 512)])
def test_release_mid_prefill_drops_partial_chunks(dtype, d):
    """A request aborted between two prefill chunks and released: the slot's next prompt
    is pooled over its own rows only (trail_release clears the K1c running sum + count;
    the oracle's release drops its chunk list).  Compared bit-for-bit with the same slot
    pooled on a fresh handle, and with the oracle."""
    from paper_2410_01035_b200.trail import trail_prefill_chunk
    w = W.make_weights(d, 512, 10, dtype, seed=91)
    rs = np.random.default_rng(92)
    a = W.make_step_inputs(1, d, dtype, prefill_frac=1.0, mean_prompt=37, seed=93)[0]
    b = W.make_step_inputs(1, d, dtype, prefill_frac=1.0, mean_prompt=11, seed=94)[0]
    outs = []
    for aborted in (True, False):
        t, o = make_pair(w, 0.8, 4, 4, 4, dtype)
        ids = np.array([2], np.uint32)
        pooled = torch.empty((1, d), dtype=torch.uint16 if dtype == "bf16" else torch.float32,
                             device="cuda")
        if aborted:   # first chunk of prompt a, then the request is aborted and released
            off = np.array([0, a.shape[0]], np.int32)
            trail_prefill_chunk(t.h, dev(a), d, dev(off), dev(ids), dev(np.zeros(1, np.uint8)), 1,
                                pooled, d)
            o.prefill_chunk(W.decode(a, dtype), off, ids, np.zeros(1, np.uint8))
            t.release(dev(ids))
            o.release(ids)
        off = np.array([0, b.shape[0]], np.int32)
        trail_prefill_chunk(t.h, dev(b), d, dev(off), dev(ids), dev(np.ones(1, np.uint8)), 1,
                            pooled, d)
        torch.cuda.synchronize()
        ref = o.prefill_chunk(W.decode(b, dtype), off, ids, np.ones(1, np.uint8))
        got = pooled.cpu().numpy()
        outs.append(got.copy())
        g = W.decode(got.view(np.uint16) if dtype == "bf16" else got, dtype)
        tol = np.abs(ref) * (2.0 ** -7 if dtype == "bf16" else 1e-5) + 1e-6
        assert np.all(np.abs(g - ref) <= tol)
        np.testing.assert_allclose(ref[0], W.decode(b, dtype).mean(axis=0) if dtype == "f32"
                                   else ref[0])
        t.close()
    np.testing.assert_array_equal(outs[0], outs[1])


@pytest.mark.parametrize("dtype,d,l1,L", [("bf16", 4096, 0, 3), ("bf16", 1024, 4, 2),
                                          ("bf16", 1024, 1, 4), ("f32", 1024, 0, 2)])
def test_multi_layer_weighted_embeddings(dtype, d, l1, L):
    """trail_predict_step_layers (reading D-28): the probe input is the
    weighted average of L layers' embeddings (prompt means at prefill, rows at decode);
    posteriors and L within the BASELINE tolerance of the oracle over a prefill and two
    decode steps, on the GEMV, split-K and CTA-pair paths."""
    n, k = 72, 10
    w = W.make_weights(d, 512, k, dtype, seed=95)
    t, o = make_pair(w, 0.8, n, n, n, dtype, l1_mode=l1)
    ids = np.arange(n, dtype=np.uint32)
    lw = [1.0 + 0.5 * i for i in range(L)]
    for step in range(3):
        embs, offs, prefs = [], None, None
        for layer in range(L):
            e, off, pref = W.make_step_inputs(n, d, dtype, prefill_frac=1.0 if step == 0 else 0.05,
                                              seed=96 + step, step=step)
            if layer == 0:
                offs, prefs = off, pref
                base = W.decode(e, dtype)
            # layers differ: a layer-dependent mix of the shared rows and fresh noise
            g = np.random.default_rng(1000 * step + layer)
            x = 0.7 * base + 0.7 * g.standard_normal(base.shape)
            embs.append(W.encode(x.astype(np.float32), dtype) if dtype == "bf16" else x.astype(np.float32))
        if step > 0:
            prefs = np.zeros(n, np.uint8)
        dembs = [dev(e) for e in embs]
        qg, Lg = t.predict_layers(dembs, lw, dev(offs), dev(ids), dev(prefs))
        torch.cuda.synchronize()
        qo, Lo = o.predict_step_layers([W.decode(e, dtype) for e in embs], offs, ids, prefs, lw)
        assert_predict_close(qg.cpu().numpy().astype(np.float64),
                             Lg.cpu().numpy().astype(np.float64), qo, Lo, f"step {step}")
    t.close()


@pytest.mark.parametrize("m", [5, 640, 4097, 20480])
def test_select_first_fit(m):
    """trail_set_fill_mode(1) (the D-15 alternative): lists bit-exact against
    oracle.select(fill='first_fit'), on a single-CTA and on a cluster selection, with a run
    cap on half the cases; the D-15 example gives {A, C}."""
    from paper_2410_01035_b200 import trail_schedule_select, trail_set_fill_mode
    w = W.make_weights(256, 128, 10, "bf16", seed=1)
    t, _ = make_pair(w, 0.8, 4, 4, max(m, 4), "bf16")
    trail_set_fill_mode(t.h, 1)
    if m == 5:   # D-15 example (+ two padding-free extra records behind it)
        key = np.array([10.0, 20.0, 30.0, 40.0, 50.0], np.float32)
        kv = np.array([5, 8, 2, 9, 1], np.uint32)
        forced = np.zeros(5, bool)
        running = np.array([0, 1, 0, 1, 0], bool)
        budget, max_run = 9, 0
    else:
        rs = np.random.default_rng(m)
        key = rs.uniform(25.6, 486.4, size=m).astype(np.float32)
        key[rs.random(m) < 0.2] = 256.0
        forced = rs.random(m) < 0.1
        running = forced | (rs.random(m) < 0.6)
        kv = rs.integers(1, 40, size=m).astype(np.uint32)
        budget = int(kv.sum() * 0.5)
        max_run = 0 if m % 2 else int(m * 0.6)
    arrival = np.arange(m, dtype=np.uint32) * 7 + 3
    ids = np.arange(m, dtype=np.uint32)
    rec = torch.from_numpy(_records(key, forced, arrival, kv, running, ids).view(np.int32)).cuda()
    trail_schedule_select(t.h, rec, m, budget, max_run, t.run_ids, t.preempt_ids, t.admit_ids,
                          t.counts)
    torch.cuda.synchronize()
    c = t.counts.cpu().numpy()
    run, pre, adm, st = R.select(key.astype(np.float64), forced, arrival, kv, running,
                                 ids.astype(np.int64), budget, max_run, fill="first_fit")
    assert c[3] == st and c[0] == len(run) and c[1] == len(pre) and c[2] == len(adm)
    np.testing.assert_array_equal(t.run_ids[:c[0]].cpu().numpy(), run)
    np.testing.assert_array_equal(t.preempt_ids[:c[1]].cpu().numpy(), pre)
    np.testing.assert_array_equal(t.admit_ids[:c[2]].cpu().numpy(), adm)
    if m == 5:
        assert run.tolist() == [0, 2, 4]
    t.close()


def test_prefill_start_hint_split_path():
    """trail_set_prefill_start (decodes first, prompts last, as vLLM orders a batch): the CTA-
    pair kernel takes the decode tiles while the side stream pools the prompt tail and runs it
    through the split-K kernel; the joined result equals the oracle's, and equals the unsplit
    path's.  A hint that puts a prompt inside the decode part raises TRAIL_DEV_BAD_HINT."""
    from paper_2410_01035_b200.trail import trail_device_errors
    n, d = 1024, 1024
    w = W.make_weights(d, 512, 10, "bf16", seed=97)
    rs = np.random.default_rng(98)
    plen = np.ones(n, np.int64)
    plen[-40:] = rs.integers(2, 60, 40)                       # prompts at the end
    pref = (plen > 1).astype(np.uint8)
    off = np.concatenate([[0], np.cumsum(plen)]).astype(np.int32)
    emb = W.encode(rs.standard_normal((int(off[-1]), d)).astype(np.float32), "bf16")
    ids = np.arange(n, dtype=np.uint32)
    first = int(np.nonzero(plen > 1)[0][0])
    outs = []
    for hint in (first, -1):
        t, o = make_pair(w, 0.8, n, n, n, "bf16", l1_mode=4)
        q, L = t.predict(dev(emb), dev(off), dev(ids), dev(pref), prefill_start=hint)
        torch.cuda.synchronize()
        qg, Lg = q.cpu().numpy().astype(np.float64), L.cpu().numpy().astype(np.float64)
        qo, Lo = oracle_predict(o, emb, off, ids, pref, "bf16")
        assert_predict_close(qg, Lg, qo, Lo, f"hint {hint}")
        outs.append((qg, Lg))
        t.close()
    assert np.abs(outs[0][0] - outs[1][0]).max() <= 1e-5
    # a broken promise: a prompt request inside the hinted decode part is flagged
    t, o = make_pair(w, 0.8, n, n, n, "bf16", l1_mode=4)
    plen2 = plen.copy()
    plen2[5] = 7
    off2 = np.concatenate([[0], np.cumsum(plen2)]).astype(np.int32)
    emb2 = W.encode(rs.standard_normal((int(off2[-1]), d)).astype(np.float32), "bf16")
    t.predict(dev(emb2), dev(off2), dev(ids), dev((plen2 > 1).astype(np.uint8)), prefill_start=first)
    torch.cuda.synchronize()
    assert trail_device_errors(t.h, True) & 0x10
    t.close()
