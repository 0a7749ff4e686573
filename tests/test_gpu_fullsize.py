"""GPU parity at BASELINE.json's full sizes in the launch configuration bench.py times, on
sampled outputs the oracle computes one request at a time (the oracle is per-request
independent), plus selection bit-exact on the GPU's own keys at the full record
count.  configs[3]: 16384 requests, d = 8192 (70B-shaped), 20 bins over [0, 1024]."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import trail_ref as R  # noqa: E402
from synth import workload as W  # noqa: E402

from gpu_util import assert_predict_close, dev, gpu_keys_forced, gpu_schedule  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2410_01035_b200 import load_library
    load_library()


def _sub_batch(b, sel, d):
    """Rows and offsets of the sampled requests only (their own CSR)."""
    rows, counts = [], []
    for j in sel:
        r0, r1 = int(b.row_offsets[j]), int(b.row_offsets[j + 1])
        rows.append(b.emb[r0:r1])
        counts.append(r1 - r0)
    off = np.zeros(len(sel) + 1, np.int32)
    np.cumsum(counts, out=off[1:])
    return np.concatenate(rows, 0), off


@pytest.mark.parametrize("n,waiting,d,k,total", [
    (16384, 4096, 8192, 20, 1024.0),    # configs[3] at one GPU
    (512, 128, 4096, 10, 512.0),        # configs[1] (the bench workload) through 3 steps
])
def test_full_size_sampled(n, waiting, d, k, total):
    from paper_2410_01035_b200 import Trail
    eng = W.EngineScript(n, waiting, d=d, dtype="bf16", seed=41, burst_start=(n <= 4096))
    w = W.make_weights(d, 512, k, "bf16", edges=W.paper_bin_edges(k, total), seed=41)
    t = Trail(w, 0.8, eng.max_slots, eng.max_slots, eng.max_slots, dtype="bf16")
    o = R.TrailOracle(W.decode(w["W1"], "bf16"), w["b1"], w["W2"], w["b2"], w["edges"], 0.8,
                      eng.max_slots, x_dtype="bf16")
    rs = np.random.default_rng(5)
    sample = None
    for step in range(3):
        b = eng.batch()
        if sample is None:   # the same requests are followed across steps (state carries)
            sample = np.sort(rs.choice(b.n, size=min(64, b.n), replace=False))
            sample_ids = b.request_ids[sample]
        pos = {int(s): i for i, s in enumerate(b.request_ids)}
        sel = np.array([pos[int(s)] for s in sample_ids if int(s) in pos])
        q, L = t.predict(dev(b.emb), dev(b.row_offsets), dev(b.request_ids), dev(b.is_prefill))
        torch.cuda.synchronize()
        qg, Lg = q.cpu().numpy().astype(np.float64), L.cpu().numpy().astype(np.float64)
        emb_s, off_s = _sub_batch(b, sel, d)
        qo, Lo = o.predict_step(W.decode(emb_s, "bf16"), off_s, b.request_ids[sel],
                                b.is_prefill[sel])
        assert_predict_close(qg[sel], Lg[sel], qo, Lo, f"n={n} step {step}")
        assert np.isfinite(Lg).all() and (Lg > 0).all()
        # selection over every live request, bit-exact on the GPU's own keys
        run, pre, adm, st = gpu_schedule(t, b)
        gk, gf, _ = gpu_keys_forced(t, b.sched_ids, b.is_running, o.prior_L)
        r2, p2, a2, s2 = R.select(gk, gf, b.arrival_seq, b.kv_blocks, b.is_running,
                                  b.sched_ids.astype(np.int64), b.kv_budget)
        np.testing.assert_array_equal(run, r2)
        np.testing.assert_array_equal(pre, p2)
        np.testing.assert_array_equal(adm, a2)
        assert st == s2
        eng.advance(run)
    t.close()
