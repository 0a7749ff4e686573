"""Parity at the configs[4] sweep points (BASELINE.json: 1-65 536 requests x c in
{0, 0.5, 0.8, inf}; bench.py --sweep times them).  For each point, in the launch
configuration the sweep times (auto layer-1 kernel choice, steady-state decode step after a
first-observation step, n running + n/4 waiting): posteriors / expected lengths of a sample
of the requests within the BASELINE tolerance of the fp64 oracle fed the same rows, and the
run / preempt / admit lists bit-exact against oracle.select on the GPU's own keys."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import trail_ref as R  # noqa: E402
from synth import workload as W  # noqa: E402

from gpu_util import dev, gpu_keys_forced  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def weights():
    return W.make_weights(4096, 512, 10, "bf16", seed=W.MASTER_SEED)


def _sub(b, js):
    rows, off = [], [0]
    for j in js:
        r0, r1 = int(b.row_offsets[j]), int(b.row_offsets[j + 1])
        rows.append(b.emb[r0:r1])
        off.append(off[-1] + r1 - r0)
    return np.concatenate(rows), np.array(off, np.int32), b.request_ids[js], b.is_prefill[js]


@pytest.mark.timeout(900)
@pytest.mark.parametrize("n", [1, 16, 512, 4096, 16384, 65536])
def test_sweep_point_parity(n, weights):
    from paper_2410_01035_b200 import Trail
    eng = W.EngineScript(n, max(1, n // 4), d=4096, dtype="bf16", seed=W.MASTER_SEED + n,
                         burst_start=False)
    b0 = eng.batch()
    eng.advance()
    b1 = eng.batch()
    rs = np.random.default_rng(n)
    js = np.sort(rs.choice(b1.n, size=min(48, b1.n), replace=False))
    slots = set(int(v) for v in b1.request_ids[js])
    j0 = [j for j in range(b0.n) if int(b0.request_ids[j]) in slots]
    for c in (0.0, 0.5, 0.8, math.inf):
        t = Trail(weights, c, eng.max_slots, eng.max_slots, eng.max_slots, dtype="bf16")
        o = R.TrailOracle(W.decode(weights["W1"], "bf16"), weights["b1"], weights["W2"],
                          weights["b2"], weights["edges"], c, eng.max_slots, x_dtype="bf16")
        for b in (b0, b1):
            q, L = t.predict(dev(b.emb), dev(b.row_offsets), dev(b.request_ids), dev(b.is_prefill))
            run, pre, adm, cnt = t.schedule(dev(b.sched_ids), dev(b.arrival_seq), dev(b.kv_blocks),
                                            dev(b.is_running), b.kv_budget)
        torch.cuda.synchronize()
        if j0:
            e, of, ids, pf = _sub(b0, j0)
            o.predict_step(W.decode(e, "bf16"), of, ids, pf)
        e, of, ids, pf = _sub(b1, js)
        qo, Lo = o.predict_step(W.decode(e, "bf16"), of, ids, pf)
        qg, Lg = q.cpu().numpy()[js].astype(np.float64), L.cpu().numpy()[js].astype(np.float64)
        assert np.abs(qg - qo).max() <= 2e-3, (n, c)
        assert (np.abs(Lg - Lo) / Lo).max() <= 1e-3, (n, c)
        gk, gf, _ = gpu_keys_forced(t, b1.sched_ids, b1.is_running, o.prior_L)
        r2, p2, a2, s2 = R.select(gk, gf, b1.arrival_seq, b1.kv_blocks, b1.is_running,
                                  b1.sched_ids.astype(np.int64), b1.kv_budget)
        cc = cnt.cpu().numpy()
        assert cc[3] == s2
        np.testing.assert_array_equal(run[:cc[0]].cpu().numpy(), r2)
        np.testing.assert_array_equal(pre[:cc[1]].cpu().numpy(), p2)
        np.testing.assert_array_equal(adm[:cc[2]].cpu().numpy(), a2)
        if c == 0.0:
            assert cc[1] == 0          # c = 0: observed running requests are never preempted
        t.close()
