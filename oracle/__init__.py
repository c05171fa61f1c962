"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the stage-discharge path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package, and only as the checker (or, for the reference
arm, as the timed CPU restatement). The product path
(paper_2506_15961_b200.verify / stages / engine) never routes through it.

Contents:
  m31.py        F_p (p = 2^31-1) arithmetic and the keyed hashes, numpy-vectorized.
  evaluator.py  the reference's concrete operator semantics
                (pkg/src/planeq/oracle.py:81-357 eval_node) restated over F_p
                with a witness batch as the trailing axis.
  stage_check.py  the reference's per-stage discharge semantics
                (pkg/src/planeq/stages.py:144-176 interface, :267-389 run_stage)
                restated as witness evaluation: same interface construction,
                same obligations, verdict per witness batch.
  gen_golden.py   (needs /root/reference, runs in the build container only)
                regenerates tests/golden/* from the reference implementation.

Pinning: tests/test_oracle_golden.py checks this oracle against the committed
golden vectors generated from the reference (exact-rational evaluations of
each operator through the reference's own oracle.eval_node, mapped into F_p,
and the reference's per-stage verdicts on a plan corpus).
"""
