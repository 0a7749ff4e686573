"""TEST INFRASTRUCTURE ONLY — the fp64 CPU oracle for the TRAIL predict+schedule path.

This package is the plain, slow, obviously-correct definition of what the CUDA path
computes, written from /root/reference/PAPER.md (cited as P:<line>) and the readings in
DESIGN.md §2 (D-<n>).  It shares no code with paper_2410_01035_b200/ and neither side
imports the other.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import, call, link or execute anything under oracle/.

Modules
  trail_ref  predict (pool, MLP probe, softmax, Bayes refinement, expected length) and
             schedule (limited-preemption SPRPT selection under a KV budget), fp64 numpy.
  mg1        M/G/1 discrete-event simulation of the SPRPT-LP rank policy (plain C,
             compiled on demand with gcc) — the policy's self-check.
  lemma1     Lemma 1 as printed and in the SOAP-consistent corrected form
             (reading D-19), evaluated by quadrature.

Parity status per function is listed in DESIGN.md §4 ("what pins each part").
"""
