"""Self-check of the policy (north_star: 'a discrete-event M/G/1 run of the policy
reproduces the paper's closed-form mean response time within Monte Carlo error').

The DES (oracle/mg1_des.c) runs SPRPT with limited preemption (rank r - a while a < C r,
-inf after).  It is pinned against textbook closed forms computed here with
scipy quadrature, independently of oracle/lemma1.py:
  * C = 0 literal (all ranks -inf) = FCFS: M/M/1 1/(1 - lam), Pollaczek-Khinchine;
  * C -> 0+ = non-preemptive SPJF with perfect predictions: Cobham/Phipps;
  * C >= 1 with perfect predictions = SRPT: Schrage-Miller;
and the corrected Lemma 1 (reading D-19) is checked against the DES at intermediate C."""
import numpy as np
import pytest
from scipy import integrate

from oracle import lemma1, mg1

N_JOBS = 1_000_000
SEEDS = (1, 2, 3)


def des_mean(lam, C, predictor, zero_plus=False):
    ms, ses = [], []
    for s in SEEDS:
        m, se, _ = mg1.mean_response(N_JOBS, lam, C, predictor, s, zero_plus=zero_plus)
        ms.append(m)
        ses.append(se)
    return float(np.mean(ms)), float(np.sqrt(np.sum(np.square(ses))) / len(ses))


def _rho(lam, x):                     # lam * int_0^x t e^{-t} dt
    return lam * (1.0 - (1.0 + x) * np.exp(-x))


def cobham_spjf_perfect(lam):
    """Non-preemptive SJF, continuous sizes (Phipps 1956): E[T] = int f(x) [lam E[X^2] /
    (2 (1 - rho(x))^2) + x] dx with E[X^2] = 2 for Exp(1)."""
    f = lambda x: np.exp(-x) * (lam * 2.0 / (2.0 * (1.0 - _rho(lam, x)) ** 2) + x)  # noqa: E731
    return integrate.quad(f, 0, np.inf, limit=200)[0]


def schrage_miller_srpt(lam):
    """SRPT (Schrage & Miller 1966): E[T(x)] = lam (int_0^x t^2 f + x^2 (1 - F(x))) /
    (2 (1 - rho(x))^2) + int_0^x dt / (1 - rho(t))."""
    def T(x):
        m2 = 2.0 - (x * x + 2 * x + 2) * np.exp(-x) + x * x * np.exp(-x)
        w = lam * m2 / (2.0 * (1.0 - _rho(lam, x)) ** 2)
        res = integrate.quad(lambda t: 1.0 / (1.0 - _rho(lam, t)), 0, x)[0]
        return w + res
    return integrate.quad(lambda x: np.exp(-x) * T(x), 0, 60, limit=200)[0]


@pytest.mark.parametrize("lam", [0.3, 0.5, 0.8])
def test_fcfs_mm1(lam):
    """SPEC acceptance 1: C = 0 (every rank -inf -> FCFS) within 2% of 1/(1 - lam)."""
    m, se = des_mean(lam, 0.0, "perfect")
    assert abs(m - 1.0 / (1.0 - lam)) <= max(0.02 / (1.0 - lam), 3 * se)
    assert lemma1.mean_response(lam, 0.0) == pytest.approx(1.0 / (1.0 - lam), rel=1e-12)


def test_c0_literal_is_fcfs_order():
    a, s, r = mg1.job_stream(20000, 0.7, "exponential", 9)
    out = mg1.simulate(a, s, r, 0.0)
    assert np.all(np.diff(out["completion"]) > 0) and out["preemptions"] == 0


def test_zero_plus_is_cobham_spjf():
    lam = 0.7
    exact = cobham_spjf_perfect(lam)
    assert lemma1.mean_response(lam, 0.0, "perfect", zero_plus=True) == pytest.approx(exact, rel=2e-4)
    m, se = des_mean(lam, 0.0, "perfect", zero_plus=True)
    assert abs(m - exact) <= 3 * se + 0.005 * exact


@pytest.mark.parametrize("C", [1.0, 2.0])
def test_perfect_predictor_C_ge_1_is_srpt(C):
    """P:402 'When C=1, the system becomes the same as SPRPT' = SRPT for perfect r."""
    lam = 0.7
    exact = schrage_miller_srpt(lam)
    assert exact == pytest.approx(1.87457, abs=2e-4)
    assert lemma1.mean_response(lam, C, "perfect") == pytest.approx(exact, rel=2e-4)
    m, se = des_mean(lam, C, "perfect")
    assert abs(m - exact) <= 3 * se + 0.005 * exact


@pytest.mark.parametrize("C,predictor", [(0.25, "perfect"), (0.5, "perfect"), (0.8, "perfect"),
                                         (0.5, "exponential"), (1.0, "exponential")])
def test_corrected_lemma1_matches_des(C, predictor):
    lam = 0.7
    m, se = des_mean(lam, C, predictor)
    f = lemma1.mean_response(lam, C, predictor, "corrected")
    assert abs(m - f) <= 3 * se + 0.005 * f


def test_printed_lemma1_is_refuted():
    """D-19: as printed, Lemma 1 at C = 1 with perfect predictions goes below the SRPT
    optimum, which no policy can beat; it disagrees with the DES by > 5%."""
    lam = 0.7
    printed = lemma1.mean_response(lam, 1.0, "perfect", "printed")
    assert printed < schrage_miller_srpt(lam) * 0.95


def test_trace_equivalence_c1_c2():
    """SPEC acceptance 6 / D-14: in M/G/1 any C >= 1 is SPRPT: identical traces."""
    a, s, r = mg1.job_stream(200_000, 0.8, "exponential", 4)
    o1, o2 = mg1.simulate(a, s, r, 1.0), mg1.simulate(a, s, r, 2.0)
    assert o1["completion"].tobytes() == o2["completion"].tobytes()


def test_burst_c08_equals_c1_and_spjf_beats_fcfs():
    """P:570 'since no new requests arrive during processing, preemption has no
    advantage, leading to similar performance between c = 0.8 and c = 1'."""
    for seed in range(5):
        a, s, r = mg1.job_stream(1000, 1.0, "exponential", seed, burst=True)
        o8, o1 = mg1.simulate(a, s, r, 0.8), mg1.simulate(a, s, r, 1.0)
        assert o8["completion"].tobytes() == o1["completion"].tobytes()
        assert o8["preemptions"] == 0
        sp = mg1.simulate(a, s, s, 0.0, zero_plus=True)["response"].mean()
        fc = mg1.simulate(a, s, s, 0.0)["response"].mean()
        assert sp < fc


def test_limited_preemption_memory_tradeoff():
    """App. D: limiting preemption lowers peak memory (SPEC acceptance 5 shape)."""
    peaks = {}
    for C in (0.5, 1.0):
        ps = []
        for seed in range(4):
            a, s, r = mg1.job_stream(200_000, 0.9, "exponential", 100 + seed)
            ps.append(mg1.simulate(a, s, r, C)["peak_memory"])
        peaks[C] = np.mean(ps)
    assert peaks[0.5] < peaks[1.0]


def test_theory_sweep_small_grid():
    """§8(f)4 sweep harness (tests/theory_sweep.py) on a small grid: every point has a DES
    mean within 3 SE + 2 % of the corrected Lemma 1 where the lemma applies, mean response
    grows with lambda, and peak memory never rises when C shrinks from 2 to 0.25 (App. D:
    limiting preemption bounds the memory held by preempted jobs)."""
    import theory_sweep as TS
    rows = TS.sweep(lams=(0.5, 0.8), cs=("0", 0.25, 1.0, 2.0), predictors=("perfect",),
                    jobs=60_000, seeds=2)
    by = {(r["lambda"], r["C"]): r for r in rows}
    for r in rows:
        if r["lemma1_corrected"] is not None:
            tol = 3 * (r["des_se"] or 0.0) + 0.02 * r["lemma1_corrected"]
            assert abs(r["des_mean_response"] - r["lemma1_corrected"]) <= tol, r
    for C in ("0", 0.25, 1.0, 2.0):
        assert by[(0.8, C)]["des_mean_response"] > by[(0.5, C)]["des_mean_response"]
    for lam in (0.5, 0.8):
        assert by[(lam, 0.25)]["des_peak_memory"] <= by[(lam, 2.0)]["des_peak_memory"] * 1.0001
