"""CPU oracle for the CDMPP predictor hot path — TEST INFRASTRUCTURE ONLY.

This package is a float64 numpy restatement of the reference (`tpcost`,
`/root/reference/pkg/src/tpcost`) algorithms on the hot path.  Every function
cites the reference file:line it restates.  It exists to *check* the CUDA path:

* only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg
  (`cpu_baseline` / `--impl reference`) may import it;
* the product package `paper_2311_09690_b200` never imports it and has no CPU
  fallback — its ops fail loudly when the CUDA library is missing.

Pinning: the oracle is checked against golden vectors produced by running the
reference itself (`tests/golden/make_golden.py`, run in the build container
where `/root/reference` exists) and against the reference test-suite's own
known answers (PE row 0, CMD 0.3125, the k-means 5-point hand run, the
select_tasks hand example, loss_pretrain 1.001).  See
`tests/test_oracle_golden.py`.
"""
