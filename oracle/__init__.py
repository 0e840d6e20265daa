"""CPU oracle for the dense-mapping path — TEST INFRASTRUCTURE ONLY.

A float64 NumPy restatement of the reference algorithm (fisheyestereo,
pkg/src/fisheyestereo/{camera,fields,rasters,solver}.py), used exclusively by
tests/, `__graft_entry__.smoke()` and bench.py's CPU-baseline leg as the
checker. The product (paper_1909_07545_b200) never imports it.

Parity is pinned: tests/test_oracle_golden.py checks every oracle stage against
golden vectors produced by running the reference itself (oracle/make_golden.py
-> tests/golden/*.npz).
"""
