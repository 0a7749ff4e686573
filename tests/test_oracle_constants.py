"""Pins of the fp64 oracle (oracle/trail_ref.py) against what the paper and mathematics
fix: printed constants, worked examples, closed forms, invariants and textbook
routines.  CPU only."""
import json
import math
import os

import numpy as np
import pytest
import scipy.special
import torch

from oracle import trail_ref as R
from synth import workload as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


# ----------------------------------------------------------------------------- shape
def test_mlp_parameter_count_matches_paper():
    """P:362 'around 2.1 million parameters': d=4096 -> 512 -> k=10."""
    w = W.make_weights(4096, 512, 10)
    n = w["W1"].size + w["b1"].size + w["W2"].size + w["b2"].size
    assert n == 4096 * 512 + 512 + 512 * 10 + 10 == 2_102_794
    assert abs(n / 1e6 - 2.1) < 0.01


# ----------------------------------------------------------------------------- bins
def test_bins_and_midpoints_paper_values():
    g = _golden("paper_bins.json")
    e = W.paper_bin_edges(10)
    np.testing.assert_allclose(e, g["edges"], rtol=0, atol=1e-12)
    m = R.bin_midpoints(e)
    # P:226 closed form m_i = 128 (2i+1) / 5 (0-based)
    np.testing.assert_allclose(m, [128 * (2 * i + 1) / 5 for i in range(10)], atol=1e-12)
    np.testing.assert_allclose(m, g["midpoints"], atol=1e-12)
    assert m[0] == pytest.approx(25.6) and m[9] == pytest.approx(486.4)


def test_transition_matrix_entries():
    """1 - 1/51.2 = 0.98046875 and 1/51.2 = 0.01953125; binsize 2 -> 0.5/0.5;
    k = 1 -> [1 - 1/w].  Only diagonal + the (i, i+1) entry are non-zero."""
    T = R.transition_matrix(W.paper_bin_edges(10))
    assert np.allclose(np.diag(T), 0.98046875, atol=1e-15)
    assert np.allclose(np.diag(T, 1), 0.01953125, atol=1e-15)
    mask = np.eye(10, dtype=bool) | np.eye(10, k=1, dtype=bool)
    assert np.all(T[~mask] == 0.0)
    T2 = R.transition_matrix(np.array([0.0, 2.0, 4.0, 6.0]))
    assert np.allclose(np.diag(T2), 0.5) and np.allclose(np.diag(T2, 1), 0.5)
    T1 = R.transition_matrix(np.array([0.0, 4.0]))
    assert T1.shape == (1, 1) and T1[0, 0] == 0.75
    # column sums: 1 except the lowest bin, which leaks 1/w_0 (D-4)
    cs = T.sum(axis=0)
    assert cs[0] == pytest.approx(1 - 1 / 51.2) and np.allclose(cs[1:], 1.0)


def test_threshold_tables_paper_bins():
    """floor(c * m_j) (D-10); c=inf never freezes (D-14)."""
    g = _golden("paper_bins.json")
    m = R.bin_midpoints(W.paper_bin_edges(10))
    assert list(R.preempt_threshold(0.8, m)) == g["thr_c0.8"]
    assert list(R.preempt_threshold(0.5, m)) == g["thr_c0.5"]
    assert list(R.preempt_threshold(0.0, m)) == [0] * 10
    assert np.all(R.preempt_threshold(math.inf, m) == R.UINT32_MAX)
    # r = 8, C = 0.5 -> a0 = 4: age 3 preemptible, age 4 not
    thr = int(R.preempt_threshold(0.5, np.array([8.0]))[0])
    assert 3 < thr and not (4 < thr)
    # r = 7.5, C = 0.8 -> preemptible for ages 0..5
    thr = int(R.preempt_threshold(0.8, np.array([7.5]))[0])
    assert [a for a in range(10) if a < thr] == [0, 1, 2, 3, 4, 5]


def test_initial_prediction_argmax_midpoint():
    """one-hot at (0-based) bin 2 -> 128.0; ties go to the lower bin."""
    m = R.bin_midpoints(W.paper_bin_edges(10))
    q = np.zeros((2, 10))
    q[0, 2] = 1.0
    q[1, :2] = 0.5
    np.testing.assert_allclose(R.initial_prediction(q, m), [128.0, 25.6])


# ----------------------------------------------------------------------------- Bayes
def test_spec_three_bin_example():
    """k=3, binsize 2, q_prev=[0,0,1], p=[0.2,0.5,0.3] -> [0, 0.625, 0.375];
    with edges [0,2,4,6] (m = [1,3,5]) L = 3.75."""
    g = _golden("spec_three_bin.json")
    e = np.array(g["edges"])
    T = R.transition_matrix(e)
    q = R.bayes_update(np.array([g["q_prev"]]), np.array([g["p"]]), T)
    np.testing.assert_allclose(q[0], g["posterior"], atol=1e-12)
    assert R.expected_length(q, R.bin_midpoints(e))[0] == pytest.approx(g["L"], abs=1e-12)


def test_expected_length_examples():
    """uniform over the paper bins -> 256.0; [0.5, 0.5, 0, ...] -> 51.2."""
    m = R.bin_midpoints(W.paper_bin_edges(10))
    assert R.expected_length(np.full(10, 0.1), m) == pytest.approx(256.0, abs=1e-12)
    q = np.zeros(10)
    q[:2] = 0.5
    assert R.expected_length(q, m) == pytest.approx(51.2, abs=1e-12)
    assert R.prior_mean_length(W.paper_bin_edges(10), None) == pytest.approx(256.0, abs=1e-12)


def test_uniform_prior_reduces_to_softmax():
    """P:219 'Initialize q^(0) = p^(0)' = the general init with a uniform prior; and with
    T = I a uniform previous posterior returns p."""
    rs = np.random.default_rng(1)
    z = rs.normal(size=(64, 10)) * 3
    p = R.softmax(z)
    np.testing.assert_allclose(p, scipy.special.softmax(z, axis=-1), rtol=1e-13, atol=1e-16)
    q0 = R.init_posterior(p, np.full((64, 10), 0.1))
    np.testing.assert_allclose(q0, p, rtol=1e-13)
    q = R.bayes_update(np.full((64, 10), 0.1), p, np.eye(10))
    np.testing.assert_allclose(q, p, rtol=1e-13)


def test_init_posterior_weights_by_prior():
    """q^(0) = normalise(pi * p^(0)) with a non-uniform pi (D-9; P:219 is the uniform case).
    Hand-computed goldens (tests/golden/prior_weighting.json): an oracle that ignored pi
    or divided by it fails every case."""
    g = _golden("prior_weighting.json")
    for case in g["init_posterior"]:
        pi, p = np.array([case["prior"]]), np.array([case["p"]])
        np.testing.assert_allclose(R.init_posterior(p, pi)[0], case["q0"], rtol=0, atol=1e-15)


def test_prior_moves_the_initial_prediction_and_threshold():
    """r = m[argmax q^(0)] with q^(0) prior-weighted: pi = [0.75, 0.25] turns
    p = [0.4, 0.6] into q^(0) = [2/3, 1/3], so r = m_0 and floor(0.8 r) = 0; a uniform
    prior keeps r = m_1 (golden).  Checked through TrailOracle's prefill bookkeeping."""
    case = _golden("prior_weighting.json")["init_posterior"][2]
    e, p = np.array(case["edges"]), np.array([case["p"]])
    m = R.bin_midpoints(e)
    q0 = R.init_posterior(p, np.array([case["prior"]]))
    assert R.initial_prediction(q0, m)[0] == case["r"]
    assert R.preempt_threshold(0.8, R.initial_prediction(q0, m))[0] == case["thr_c08"]
    qu = R.init_posterior(p, np.full((1, 2), 0.5))
    assert R.initial_prediction(qu, m)[0] == case["r_uniform"]
    assert R.preempt_threshold(0.8, R.initial_prediction(qu, m))[0] == case["thr_c08_uniform"]
    # the same through the stateful oracle: a 1-d probe whose logits are log p exactly
    o = R.TrailOracle(np.zeros((1, 1)), np.zeros(1), np.zeros((2, 1)), np.log(p[0]), e, 0.8, 2,
                      prior=np.array(case["prior"]), x_dtype="f32")
    q, L = o.predict_step(np.zeros((1, 1)), np.array([0, 1]), np.array([0]), np.array([1]))
    np.testing.assert_allclose(q[0], case["q0"], atol=1e-15)
    assert o.state.thr[0] == case["thr_c08"]


def test_prior_mean_length_non_uniform():
    """E_pi[L] = sum_i pi_i m_i (D-24) for non-uniform pi, hand-computed (golden): 76.8 on
    the paper bins for pi = [0.4, 0.3, 0.2, 0.1, 0, ...]; 1.5 on edges [0, 2, 4].  Also the
    key of an unseen request in an oracle created with that prior."""
    g = _golden("prior_weighting.json")["prior_mean_length"]
    e0 = W.paper_bin_edges(10)
    assert R.prior_mean_length(e0, np.array(g[0]["prior"])) == pytest.approx(g[0]["E_L"], abs=1e-12)
    assert R.prior_mean_length(np.array(g[1]["edges"]), np.array(g[1]["prior"])) == \
        pytest.approx(g[1]["E_L"], abs=1e-15)
    w = W.make_weights(16, 8, 10, "f32")
    o = R.TrailOracle(w["W1"], w["b1"], w["W2"], w["b2"], e0, 0.8, 4,
                      prior=np.array(g[0]["prior"]), x_dtype="f32")
    key, forced = o.keys_and_forced(np.array([2]), np.array([0]))
    assert key[0] == pytest.approx(g[0]["E_L"], abs=1e-12) and not forced[0]


def test_two_step_refinement_is_posterior_fed():
    """Reading D-2 pinned by a hand-computed two-step example (golden two_step): the prior
    of step t is T applied to the previous POSTERIOR, giving q^(2) = [9/13, 4/13]
    and L = 21/13; the literal prior-fed recursion of P:220 would give [3/7, 4/7]."""
    g = _golden("prior_weighting.json")["two_step"]
    e = np.array(g["edges"])
    T, m = R.transition_matrix(e), R.bin_midpoints(e)
    p = np.array(g["p"])
    q = R.init_posterior(p[:1], np.full((1, 2), 0.5))
    q = R.bayes_update(q, p[1:2], T)
    np.testing.assert_allclose(q[0], g["q1"], atol=1e-15)
    q = R.bayes_update(q, p[2:3], T)
    np.testing.assert_allclose(q[0], g["q2"], atol=1e-15)
    assert R.expected_length(q, m)[0] == pytest.approx(g["L2"], abs=1e-15)
    assert abs(q[0, 0] - g["q2_prior_fed"][0]) > 0.2
    # and through the stateful oracle (three observations of one slot)
    o = R.TrailOracle(np.zeros((1, 1)), np.zeros(1), np.zeros((2, 1)), np.zeros(2), e, 0.8, 1,
                      x_dtype="f32")
    for t in range(3):
        o.b2 = np.log(p[t])
        q, L = o.predict_step(np.zeros((1, 1)), np.array([0, 1]), np.array([0]),
                              np.array([1 if t == 0 else 0]))
    np.testing.assert_allclose(q[0], g["q2"], atol=1e-15)


def test_L_minus_one_identity_pins_orientation():
    """Closed form (derived in DESIGN.md §4): equal widths w, m_0 = w/2, uninformative p:
    L' = (L - 1 + q_0/2) / (1 - q_0/w); so L' = L - 1 exactly when q_0 = 0.  The other T
    orientation would give L + 1 (reading D-1).  With a uniform p the prior-fed and
    posterior-fed recursions coincide up to normalisation, so this pins D-1 only; D-2 is
    pinned by test_two_step_refinement_is_posterior_fed."""
    e = W.paper_bin_edges(10)
    m, T, w = R.bin_midpoints(e), R.transition_matrix(e), 51.2
    rs = np.random.default_rng(7)
    q = rs.dirichlet(np.ones(10), size=16)
    q[:8, 0] = 0.0
    q /= q.sum(axis=1, keepdims=True)
    uni = np.full_like(q, 0.1)
    for _ in range(40):
        L, q0 = R.expected_length(q, m), q[:, 0].copy()
        qn = R.bayes_update(q, uni, T)
        np.testing.assert_allclose(R.expected_length(qn, m), (L - 1 + q0 / 2) / (1 - q0 / w),
                                   rtol=1e-12)
        q = qn
    # wrong orientation (transpose) moves L up by one for mass away from the top bin
    q = np.zeros((1, 10))
    q[0, 4] = 1.0
    up = R.bayes_update(q, np.full((1, 10), 0.1), T.T)
    assert R.expected_length(up, m)[0] == pytest.approx(R.expected_length(q, m)[0] + 1, abs=1e-9)


def test_posterior_on_simplex_and_L_in_range():
    e = W.paper_bin_edges(10)
    m, T = R.bin_midpoints(e), R.transition_matrix(e)
    rs = np.random.default_rng(3)
    q = R.softmax(rs.normal(size=(128, 10)) * 4)
    for _ in range(300):
        q = R.bayes_update(q, R.softmax(rs.normal(size=(128, 10)) * 4), T)
        assert np.all(q >= 0) and np.allclose(q.sum(axis=1), 1.0, atol=1e-12)
        L = R.expected_length(q, m)
        assert np.all(L >= m[0] - 1e-9) and np.all(L <= m[-1] + 1e-9)


def test_linear_and_log_domain_agree():
    """D-22: the linear fp64 recursion equals its log-domain form to <= 1e-12 over 200
    confident, contradictory (adversarial iid) observations."""
    e = W.paper_bin_edges(10)
    T = R.transition_matrix(e)
    rs = np.random.default_rng(11)
    z = rs.normal(size=(64, 10)) * 4
    q = R.softmax(z)
    lq = np.log(q)
    worst = 0.0
    for _ in range(200):
        z = rs.normal(size=(64, 10)) * 4
        p = R.softmax(z)
        logp = z - scipy.special.logsumexp(z, axis=1, keepdims=True)
        q = R.bayes_update(q, p, T)
        lq = R.bayes_update_log(lq, logp, T)
        worst = max(worst, float(np.abs(q - np.exp(lq)).max()))
    assert worst <= 1e-12


def test_refinement_beats_raw_on_noisy_observations():
    """Property stand-in for Fig. 3: with noisy per-iteration
    observations around the true remaining length, the refined estimate's mean absolute
    error is below the raw per-iteration estimate's; with noiseless observations the two
    coincide in the lowest bin's quantisation error only."""
    e = W.paper_bin_edges(10)
    m, T = R.bin_midpoints(e), R.transition_matrix(e)
    rs = np.random.default_rng(5)
    raw_err, ref_err = [], []
    for _ in range(300):
        N = int(rs.integers(20, 500))
        q = None
        for t in range(N):
            rem = N - t
            score = -2.0 * np.abs(m - rem) / 51.2 + rs.normal(0, 1.5, 10)
            p = R.softmax(score[None, :])
            q = p if q is None else R.bayes_update(q, p, T)
            raw_err.append(abs(R.expected_length(p, m)[0] - rem))
            ref_err.append(abs(R.expected_length(q, m)[0] - rem))
    assert np.mean(ref_err) < 0.8 * np.mean(raw_err)


# ----------------------------------------------------------------------------- MLP, pool
def test_classifier_against_torch_fp64():
    """h = ReLU(W1 x + b1), z = W2 h + b2 against torch.nn in fp64."""
    rs = np.random.default_rng(2)
    d, H, k, n = 64, 32, 10, 9
    W1, b1 = rs.normal(size=(H, d)), rs.normal(size=H)
    W2, b2 = rs.normal(size=(k, H)), rs.normal(size=k)
    X = rs.normal(size=(n, d))
    net = torch.nn.Sequential(torch.nn.Linear(d, H), torch.nn.ReLU(), torch.nn.Linear(H, k)).double()
    with torch.no_grad():
        net[0].weight.copy_(torch.from_numpy(W1)); net[0].bias.copy_(torch.from_numpy(b1))
        net[2].weight.copy_(torch.from_numpy(W2)); net[2].bias.copy_(torch.from_numpy(b2))
        ref = net(torch.from_numpy(X)).numpy()
    np.testing.assert_allclose(R.classifier_logits(X, W1, b1, W2, b2), ref, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(R.softmax(ref), torch.softmax(torch.from_numpy(ref), -1).numpy(),
                               rtol=1e-12)


def test_bf16_round_matches_torch_and_synth():
    rs = np.random.default_rng(4)
    x = np.concatenate([rs.normal(size=20000).astype(np.float32),
                        (rs.normal(size=2000) * 1e-30).astype(np.float32),
                        np.array([1.0, 1.00390625, 1.005859375, 3.0e38, -2.5], np.float32)])
    ours = R.bf16_round(x.astype(np.float64))
    tor = torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()
    np.testing.assert_array_equal(ours, tor)
    np.testing.assert_array_equal(ours, W.bf16_bits_to_f32(W.f32_to_bf16_bits(x)).astype(np.float64))


def test_pool_mean_and_decode_row():
    rs = np.random.default_rng(6)
    rows = W.bf16_bits_to_f32(W.f32_to_bf16_bits(rs.normal(size=(44, 128)))).astype(np.float64)
    np.testing.assert_array_equal(R.pool_embedding(rows[:1], "bf16"), rows[0])   # decode row exact
    u = R.pool_embedding(rows, "bf16")
    assert np.all(np.abs(u - rows.mean(axis=0)) <= np.abs(rows.mean(axis=0)) * 2 ** -8 + 1e-30)
    np.testing.assert_array_equal(R.pool_embedding(rows, "f32"), rows.mean(axis=0))


# ----------------------------------------------------------------------------- the step
def test_oracle_step_semantics():
    """Prefill initialises q, r, thr, a=0; each decode applies one update and a += 1;
    the key of an unseen request is E_pi[L]; forced iff running & seen & a >= thr."""
    d, k = 64, 10
    w = W.make_weights(d, 32, k, "f32")
    o = R.TrailOracle(w["W1"], w["b1"], w["W2"], w["b2"], w["edges"], 0.8, 8, x_dtype="f32")
    rs = np.random.default_rng(0)
    emb = rs.normal(size=(5, d))
    q, L = o.predict_step(emb, np.array([0, 4, 5]), np.array([1, 3]), np.array([1, 1]))
    assert np.all(o.state.age[[1, 3]] == 0) and o.state.seen[[1, 3]].all()
    thr0 = o.state.thr[[1, 3]].copy()
    q2, L2 = o.predict_step(emb[:2], np.array([0, 1, 2]), np.array([1, 3]), np.array([0, 0]))
    assert np.all(o.state.age[[1, 3]] == 1) and np.all(o.state.thr[[1, 3]] == thr0)
    p = o.probs(emb[:2])
    np.testing.assert_allclose(q2, R.bayes_update(q, p, o.T), rtol=1e-14)
    key, forced = o.keys_and_forced(np.array([1, 3, 5]), np.array([1, 1, 0]))
    assert key[2] == pytest.approx(256.0) and not forced[2]
    assert list(forced[:2]) == [bool(1 >= t) for t in thr0]


# ----------------------------------------------------------------------------- time update
def test_time_update_closed_form_matrix_power_and_state():
    """Predict-every-K (reading D-25): between observations only T acts.  Pinned by
    (1) the L - 1 closed form per iteration (equal widths: L' = (L - 1 + q_0/2)/(1 - q_0/w),
    derived in DESIGN.md §4 — with no likelihood term it applies directly), (2) K
    normalised steps = one normalised application of the matrix power T^K (normalisation
    commutes with the linear map up to scale), (3) the oracle's state bookkeeping: age
    advances by K, unobserved slots keep the prior and E_pi[L] (D-24)."""
    e = W.paper_bin_edges(10)
    m, T, w = R.bin_midpoints(e), R.transition_matrix(e), 51.2
    rs = np.random.default_rng(11)
    q = rs.dirichlet(np.ones(10), size=32)
    q[:16, 0] = 0.0
    q /= q.sum(axis=1, keepdims=True)
    L, q0 = R.expected_length(q, m), q[:, 0]
    np.testing.assert_allclose(R.expected_length(R.time_update(q, T, 1), m),
                               (L - 1 + q0 / 2) / (1 - q0 / w), rtol=1e-12)
    for K in (1, 2, 5, 17):
        direct = q @ np.linalg.matrix_power(T, K).T
        direct /= direct.sum(axis=1, keepdims=True)
        np.testing.assert_allclose(R.time_update(q, T, K), direct, rtol=1e-10, atol=1e-15)
    # mass concentrated away from the lowest bin: exactly one length unit per iteration
    qq = np.zeros((1, 10))
    qq[0, 5] = 1.0
    assert R.expected_length(R.time_update(qq, T, 3), m)[0] == pytest.approx(
        R.expected_length(qq, m)[0] - 3, abs=1e-9)
    # oracle state
    w_ = W.make_weights(64, 128, 10, "f32", seed=3)
    o = R.TrailOracle(w_["W1"], w_["b1"], w_["W2"], w_["b2"], w_["edges"], 0.8, 8, x_dtype="f32")
    emb, off, pref = W.make_step_inputs(4, 64, "f32", prefill_frac=1.0, seed=4)
    qa, La = o.predict_step(W.decode(emb, "f32"), off, np.arange(4), pref)
    qt, Lt = o.time_update(np.array([0, 1, 2, 3, 6]), 3)
    np.testing.assert_allclose(qt[:4], R.time_update(qa, o.T, 3), rtol=1e-12)
    assert np.all(o.state.age[:4] == 3) and o.state.age[6] == 0 and not o.state.seen[6]
    np.testing.assert_allclose(qt[4], np.full(10, 0.1))
    assert Lt[4] == pytest.approx(256.0)


def test_dynamic_threshold_special_cases():
    """Dynamic-threshold variant (reading D-26): forced iff a >= c (a + L).
    c = 0 freezes every observed running request (the static rule's c = 0 case, D-13);
    c >= 1 never freezes (full SPRPT, like c = inf, D-14); for 0 < c < 1 the boundary is
    a = c L / (1 - c), and with L falling one unit per iteration (T only) a frozen request
    stays frozen."""
    w_ = W.make_weights(64, 128, 10, "f32", seed=5)
    emb, off, pref = W.make_step_inputs(16, 64, "f32", prefill_frac=1.0, seed=6)
    run = np.ones(16, np.uint8)
    out = {}
    for c in (0.0, 0.5, 1.0, 3.0):
        o = R.TrailOracle(w_["W1"], w_["b1"], w_["W2"], w_["b2"], w_["edges"], c, 16, x_dtype="f32")
        o.threshold = "dynamic"
        o.predict_step(W.decode(emb, "f32"), off, np.arange(16), pref)
        hist = []
        for _ in range(400):
            o.time_update(np.arange(16), 1)
            _, f = o.keys_and_forced(np.arange(16), run)
            a, L = o.state.age[:16].astype(float), o.state.L[:16]
            if 0 < c < 1:
                np.testing.assert_array_equal(f, a >= c * L / (1 - c) - 1e-9 * L)
            hist.append(f)
        hist = np.array(hist)
        assert np.all(hist[1:] >= hist[:-1])          # once frozen, stays frozen
        out[c] = hist
    assert out[0.0].all()
    assert not out[1.0].any() and not out[3.0].any()
    assert out[0.5][0].sum() == 0 and out[0.5][-1].sum() == 16


def test_prefill_chunk_oracle_is_the_mean_of_all_rows():
    """Chunked prefill (D-27): however the prompt is split, the pooled row is the mean of all
    its rows — pinned against numpy's mean of the unsplit prompt, and a one-chunk
    prompt against the plain pool."""
    w_ = W.make_weights(64, 128, 10, "f32", seed=8)
    o = R.TrailOracle(w_["W1"], w_["b1"], w_["W2"], w_["b2"], w_["edges"], 0.8, 8, x_dtype="f32")
    rs = np.random.default_rng(9)
    full = rs.standard_normal((37, 64))
    cuts = [0, 5, 6, 20, 37]
    for a, b in zip(cuts[:-1], cuts[1:]):
        out = o.prefill_chunk(full[a:b], np.array([0, b - a]), np.array([3]), np.array([b == 37]))
    np.testing.assert_allclose(out[0], full.mean(axis=0), rtol=1e-12, atol=1e-15)
    one = o.prefill_chunk(full, np.array([0, 37]), np.array([4]), np.array([1]))
    np.testing.assert_allclose(one[0], R.pool_embedding(full, "f32"), rtol=0, atol=0)
    ob = R.TrailOracle(w_["W1"], w_["b1"], w_["W2"], w_["b2"], w_["edges"], 0.8, 8, x_dtype="bf16")
    xb = W.decode(W.encode(full.astype(np.float32), "bf16"), "bf16")
    ob.prefill_chunk(xb[:10], np.array([0, 10]), np.array([1]), np.array([0]))
    out = ob.prefill_chunk(xb[10:], np.array([0, 27]), np.array([1]), np.array([1]))
    np.testing.assert_array_equal(out[0], R.bf16_round(xb.mean(axis=0)))
    # a request aborted between chunks and released: the slot's next prompt pools only its
    # own rows (numpy mean of that prompt), not the aborted one's partial rows
    o.prefill_chunk(full[:20], np.array([0, 20]), np.array([5]), np.array([0]))
    o.release(np.array([5]))
    nxt = o.prefill_chunk(full[20:], np.array([0, 17]), np.array([5]), np.array([1]))
    np.testing.assert_allclose(nxt[0], full[20:].mean(axis=0), rtol=1e-12, atol=1e-15)


# ----------------------------------------------------------------------------- multi-layer
def test_multi_layer_weighted_average_oracle():
    """Multi-layer weighted embeddings (reading D-28): u = sum_l a_l u_l with
    a = w / sum(w).  Pins: one layer (or identical layers, any weights) is the plain
    predict_step; weights [3, 1] on a hand-computed 2-d example give 0.75 u_1 + 0.25 u_2 of
    the per-layer prompt means; a zero weight drops its layer."""
    w_ = W.make_weights(64, 128, 10, "f32", seed=8)
    mk = lambda: R.TrailOracle(w_["W1"], w_["b1"], w_["W2"], w_["b2"], w_["edges"], 0.8, 8,  # noqa: E731
                               x_dtype="f32")
    rs = np.random.default_rng(4)
    e1, e2 = rs.standard_normal((9, 64)), rs.standard_normal((9, 64))
    off, ids, pf = np.array([0, 5, 6, 9]), np.array([0, 1, 2]), np.array([1, 0, 1])
    q1, L1 = mk().predict_step(e1, off, ids, pf)
    q2, L2 = mk().predict_step_layers([e1], off, ids, pf, [2.5])
    np.testing.assert_array_equal(q1, q2)
    q3, _ = mk().predict_step_layers([e1, e1, e1], off, ids, pf, [1.0, 7.0, 0.5])
    np.testing.assert_allclose(q3, q1, rtol=1e-12, atol=1e-15)
    q4, _ = mk().predict_step_layers([e1, e2], off, ids, pf, [1.0, 0.0])
    np.testing.assert_allclose(q4, q1, rtol=1e-12, atol=1e-15)
    # hand-computed 2-d example: request rows layer1 [[1,2],[3,6]], layer2 [[5,-2],[7,2]]
    o = R.TrailOracle(np.eye(2), np.zeros(2), np.zeros((3, 2)), np.zeros(3),
                      np.array([0.0, 2.0, 4.0, 6.0]), 0.8, 2, x_dtype="f32")
    X = o.mixed_inputs([np.array([[1.0, 2.0], [3.0, 6.0]]), np.array([[5.0, -2.0], [7.0, 2.0]])],
                       np.array([0, 2]), [3.0, 1.0])
    # layer means [2, 4] and [6, 0] -> 0.75 [2, 4] + 0.25 [6, 0] = [3, 3]
    np.testing.assert_array_equal(X, [[3.0, 3.0]])
    ob = R.TrailOracle(np.eye(2), np.zeros(2), np.zeros((3, 2)), np.zeros(3),
                       np.array([0.0, 2.0, 4.0, 6.0]), 0.8, 2, x_dtype="bf16")
    Xb = ob.mixed_inputs([np.array([[1.0, 1.0]]), np.array([[1.0 + 2.0 ** -7, 1.0]])], np.array([0, 1]),
                         [1.0, 1.0])
    # (1 + (1 + 2^-7)) / 2 = 1 + 2^-8: a bf16 tie, rounded once to even -> 1.0
    np.testing.assert_array_equal(Xb, [[1.0, 1.0]])
