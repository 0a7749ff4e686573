"""Pins of the oracle's limited-preemption SPRPT selection (oracle.trail_ref.select):
brute-force enumeration on tiny inputs, the D-15 worked example, and the c = 0 / c = inf /
unlimited-budget reductions named in BASELINE.json's north_star."""
import itertools
import math

import numpy as np
import pytest

from oracle import trail_ref as R
from synth import workload as W


def brute_force_run_set(key, forced, arrival, kv, budget, max_run):
    """Largest subset S with forced c S, sum kv <= budget, |S| <= max_run, that is
    priority-closed: any non-forced request ranked ahead of a non-forced member is a
    member.  Enumerated, not constructed greedily."""
    m = len(key)
    cap = max_run if max_run > 0 else m
    F = [j for j in range(m) if forced[j]]
    if sum(kv[j] for j in F) > budget or len(F) > cap:
        return set(F), R.STATUS_WARN_OVER_BUDGET
    rank = lambda j: (key[j], arrival[j])  # noqa: E731
    free = [j for j in range(m) if not forced[j]]
    best = None
    for r in range(len(free) + 1):
        for S in itertools.combinations(free, r):
            S = set(S)
            if sum(kv[j] for j in S) + sum(kv[j] for j in F) > budget or len(S) + len(F) > cap:
                continue
            closed = all((j in S) for j in free for s in S if rank(j) < rank(s))
            if closed and (best is None or len(S) > len(best)):
                best = S
    return set(F) | best, R.STATUS_OK


@pytest.mark.parametrize("trial", range(400))
def test_select_equals_brute_force(trial):
    rs = np.random.default_rng(1000 + trial)
    m = int(rs.integers(1, 10))
    key = rs.choice([25.6, 76.8, 128.0, 179.2, 256.0], size=m) + rs.choice([0.0, 0.5], size=m)
    forced = rs.random(m) < 0.3
    running = forced | (rs.random(m) < 0.5)
    arrival = rs.permutation(m) + 10
    kv = rs.integers(0, 8, size=m)
    budget = int(rs.integers(0, 30))
    max_run = int(rs.choice([0, 0, 2, 4]))
    ids = np.arange(m) + 100
    run, pre, adm, st = R.select(key, forced, arrival, kv, running, ids, budget, max_run)
    exp_set, exp_st = brute_force_run_set(key, forced, arrival, kv, budget, max_run)
    assert set(run - 100) == exp_set and st == exp_st
    assert set(pre - 100) == {j for j in range(m) if running[j] and j not in exp_set}
    assert set(adm - 100) == {j for j in range(m) if not running[j] and j in exp_set}
    # lists come in priority order: forced first, then (key, arrival)
    order = [(0 if forced[j] else 1, key[j], arrival[j]) for j in run - 100]
    assert order == sorted(order)


def test_strict_prefix_example_D15():
    """Keys A=10, B=20, C=30 with kv 5, 8, 2 and budget 9: strict prefix {A} (first-fit
    would give {A, C})."""
    run, pre, adm, st = R.select([10.0, 20.0, 30.0], [False] * 3, [0, 1, 2], [5, 8, 2],
                                 [0, 0, 0], np.array([0, 1, 2]), 9)
    assert list(run) == [0] and list(adm) == [0] and st == R.STATUS_OK


def test_forced_over_budget_warns():
    run, pre, adm, st = R.select([10.0, 20.0, 30.0], [True, True, False], [0, 1, 2], [5, 8, 2],
                                 [1, 1, 0], np.array([0, 1, 2]), 9)
    assert set(run) == {0, 1} and st == R.STATUS_WARN_OVER_BUDGET and len(pre) == 0


def _trajectory(c, budget_frac, steps=60, n=24, seed=3):
    """Run the oracle in closed loop on a small synthetic engine."""
    eng = W.EngineScript(n, 6, d=32, dtype="f32", seed=seed, temporal="iid",
                         budget_frac=budget_frac)
    w = W.make_weights(32, 16, 10, "f32", seed=seed)
    o = R.TrailOracle(w["W1"], w["b1"], w["W2"], w["b2"], w["edges"], c, eng.max_slots,
                      x_dtype="f32")
    out = []
    for _ in range(steps):
        b = eng.batch()
        emb = W.decode(b.emb, "f32")
        o.predict_step(emb, b.row_offsets, b.request_ids, b.is_prefill)
        res = o.schedule_step(b.sched_ids, b.arrival_seq, b.kv_blocks, b.is_running,
                              b.kv_budget if budget_frac < 10 else 1 << 60)
        key, forced = o.keys_and_forced(b.sched_ids, b.is_running)
        seen = o.state.seen[b.sched_ids.astype(np.int64)].copy()
        out.append((b, res, key, forced, seen))
        eng.advance(res[0])
    return out


def test_c_zero_never_preempts():
    """north_star / D-13: with c = 0 every observed running request is frozen (a >= 0),
    so the preempt list is always empty."""
    for b, (run, pre, adm, st), key, forced, seen in _trajectory(0.0, 0.8):
        assert len(pre) == 0
        assert np.array_equal(forced, (b.is_running == 1) & seen)


def test_c_inf_is_pure_sprpt_prefix():
    """c = inf: nothing is frozen; the run set is the shortest-predicted prefix (D-14)."""
    for b, (run, pre, adm, st), key, forced, seen in _trajectory(math.inf, 0.8):
        assert not forced.any()
        order = sorted(range(b.m), key=lambda j: (key[j], b.arrival_seq[j]))
        assert list(run) == [int(b.sched_ids[j]) for j in order[:len(run)]]


def test_unlimited_budget_runs_everything():
    for b, (run, pre, adm, st), key, forced, seen in _trajectory(0.8, 1e9):
        assert len(run) == b.m and len(pre) == 0


def brute_force_first_fit(key, forced, arrival, kv, budget, max_run):
    """First-fit by definition, enumerated: among all subsets S with forced c S, sum kv <=
    budget and |S| <= max_run, the one whose membership vector, read in priority order
    (forced first, then (key, arrival)), is lexicographically largest — a member ranked
    earlier always outweighs any set of later ones."""
    m = len(key)
    cap = max_run if max_run > 0 else m
    F = [j for j in range(m) if forced[j]]
    if sum(kv[j] for j in F) > budget or len(F) > cap:
        return set(F), R.STATUS_WARN_OVER_BUDGET
    free = sorted((j for j in range(m) if not forced[j]), key=lambda j: (key[j], arrival[j], j))
    best, best_vec = None, None
    for r in range(len(free) + 1):
        for S in itertools.combinations(free, r):
            if sum(kv[j] for j in S) + sum(kv[j] for j in F) > budget or len(S) + len(F) > cap:
                continue
            vec = tuple(1 if j in S else 0 for j in free)
            if best_vec is None or vec > best_vec:
                best, best_vec = set(S), vec
    return set(F) | best, R.STATUS_OK


@pytest.mark.parametrize("trial", range(300))
def test_first_fit_equals_brute_force(trial):
    """fill='first_fit' (the D-15 alternative) against its definition."""
    rs = np.random.default_rng(5000 + trial)
    m = int(rs.integers(1, 10))
    key = rs.choice([25.6, 76.8, 128.0, 179.2, 256.0], size=m) + rs.choice([0.0, 0.5], size=m)
    forced = rs.random(m) < 0.3
    running = forced | (rs.random(m) < 0.5)
    arrival = rs.permutation(m) + 10
    kv = rs.integers(0, 8, size=m)
    budget = int(rs.integers(0, 30))
    max_run = int(rs.choice([0, 0, 2, 4]))
    ids = np.arange(m) + 100
    run, pre, adm, st = R.select(key, forced, arrival, kv, running, ids, budget, max_run,
                                 fill="first_fit")
    exp_set, exp_st = brute_force_first_fit(key, forced, arrival, kv, budget, max_run)
    assert set(run - 100) == exp_set and st == exp_st
    assert set(pre - 100) == {j for j in range(m) if running[j] and j not in exp_set}
    assert set(adm - 100) == {j for j in range(m) if not running[j] and j in exp_set}
    order = [(0 if forced[j] else 1, key[j], arrival[j]) for j in run - 100]
    assert order == sorted(order)
    # first-fit contains the strict prefix
    run_p = R.select(key, forced, arrival, kv, running, ids, budget, max_run)[0]
    assert set(run_p) <= set(run)


def test_first_fit_example_D15():
    """Keys A=10, B=20, C=30 with kv 5, 8, 2 and budget 9: first-fit gives {A, C} (SURVEY
    §8(c) D-15 example)."""
    run, pre, adm, st = R.select([10.0, 20.0, 30.0], [False] * 3, [0, 1, 2], [5, 8, 2],
                                 [0, 0, 0], np.array([0, 1, 2]), 9, fill="first_fit")
    assert list(run) == [0, 2] and list(adm) == [0, 2] and st == R.STATUS_OK
