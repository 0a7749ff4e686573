"""the paper's second workload, its theory (App. D): mean
response time and peak memory of the M/G/1 SPRPT-with-limited-preemption policy over a grid
of arrival rates lambda and preemption parameters C, for the perfect and the exponential
predictor, by many-replication discrete-event simulation (oracle/mg1_des.c) beside the
corrected Lemma 1 (oracle/lemma1.py, reading D-19).  Lives under tests/ because it runs the
oracle (test infrastructure).  Writes one JSON document:

    python tests/theory_sweep.py [--jobs 200000] [--seeds 3] [--out profiles/r02_theory_sweep.json]

Peak memory is the DES's max over time of the summed ages of started, unfinished jobs (the
KV a preempted job keeps, App. D); C = 0 is literal FCFS (rank -inf at every age, D-13) and
"0+" the non-preemptive SPJF limit."""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import lemma1, mg1  # noqa: E402

LAMS = (0.5, 0.6, 0.7, 0.8, 0.9)
CS = ("0", "0+", 0.25, 0.5, 0.8, 1.0, 2.0)


def point(lam, C, predictor, jobs, seeds):
    zp = C == "0+"
    Cv = 0.0 if C in ("0", "0+") else float(C)
    means, peaks, pre = [], [], []
    for s in range(seeds):
        a, x, r = mg1.job_stream(jobs, lam, predictor, seed=100 + s)
        out = mg1.simulate(a, x, r, Cv, zero_plus=zp)
        resp = out["response"][int(0.2 * jobs):]
        means.append(float(resp.mean()))
        peaks.append(out["peak_memory"])
        pre.append(out["preemptions"] / jobs)
    rec = {"lambda": lam, "C": C, "predictor": predictor,
           "des_mean_response": float(np.mean(means)),
           "des_se": float(np.std(means, ddof=1) / math.sqrt(seeds)) if seeds > 1 else None,
           "des_peak_memory": float(np.mean(peaks)),
           "des_preemptions_per_job": float(np.mean(pre)),
           "jobs": jobs, "seeds": seeds}
    try:
        rec["lemma1_corrected"] = lemma1.mean_response(lam, Cv, predictor, "corrected", zero_plus=zp)
    except Exception as e:   # noqa: BLE001 (report, keep sweeping)
        rec["lemma1_corrected"] = None
        rec["lemma1_error"] = str(e)
    return rec


def sweep(lams=LAMS, cs=CS, predictors=("perfect", "exponential"), jobs=200_000, seeds=3):
    return [point(lam, C, p, jobs, seeds) for p in predictors for lam in lams for C in cs]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=200_000)
    ap.add_argument("--seeds", type=int, default=3)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_theory_sweep.json"))
    args = ap.parse_args()
    t0 = time.time()
    rows = sweep(jobs=args.jobs, seeds=args.seeds)
    doc = {"what": "M/G/1 SPRPT-LP: mean response time and peak memory vs lambda x C "
                   "(App. D, P:946-1006), DES vs corrected Lemma 1; Exp(1) service",
           "seconds": time.time() - t0, "rows": rows}
    with open(args.out, "w") as f:
        json.dump(doc, f, indent=1)
    for r in rows:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
