"""Regression test of the iteration-level batch simulator, which drives the
real library (every selection and every prediction is a C-ABI call) with SPEC's synthetic
observation model.  Small workloads, fixed seeds:
  * every job completes, results are deterministic (same seed -> same trace summary);
  * c = 0 never preempts an observed running request (D-13);
  * TRAIL (c = 0.8) has a lower mean latency than the vLLM-FCFS baseline under Poisson
    arrivals and under a burst;
  * burst arrivals with c = 0.8 and c = 1 are within a few percent ('c = 0.8 ~ c = 1')."""
import importlib.util
import os
import types

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sim():
    spec = importlib.util.spec_from_file_location("simulate", os.path.join(ROOT, "scripts", "simulate.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _args(**kw):
    a = dict(jobs=400, rate=2.0, slots=256, budget_frac=0.25, conc=2.0, mislabel=0.1,
             recompute_rate=0.0, seeds=1, max_iters=100000, arrivals="poisson")
    a.update(kw)
    return types.SimpleNamespace(**a)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.timeout(600)
def test_simulator_trail_vs_fcfs_poisson():
    sim = _sim()
    a = _args()
    tr = sim.run(0.8, a, 1000)
    tr2 = sim.run(0.8, a, 1000)
    ff = sim.run(0.0, a, 1000, fcfs=True)
    c0 = sim.run(0.0, a, 1000)
    assert tr["completed"] == ff["completed"] == c0["completed"] == a.jobs
    assert tr == tr2                                            # deterministic
    assert c0["preemptions"] == 0                               # D-13
    assert tr["mean_latency"] < ff["mean_latency"], (tr, ff)    # P:516 trend
    print("poisson", tr, ff, c0)


@pytest.mark.timeout(600)
def test_simulator_burst():
    sim = _sim()
    a = _args(arrivals="burst", jobs=300)
    tr = sim.run(0.8, a, 1001)
    t1 = sim.run(1.0, a, 1001)
    ff = sim.run(0.0, a, 1001, fcfs=True)
    assert tr["completed"] == t1["completed"] == ff["completed"] == a.jobs
    assert tr["mean_latency"] < ff["mean_latency"], (tr, ff)    # P:570 trend
    assert abs(tr["mean_latency"] - t1["mean_latency"]) <= 0.05 * t1["mean_latency"], (tr, t1)
    print("burst", tr, t1, ff)
