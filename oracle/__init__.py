"""CPU oracle for the citywalk env-side hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, in numpy / plain Python, the reference algorithms the
B200 kernels replace (scene sampling and the crowd dynamics step of
`/root/reference/pkg/src/citywalk`).  It exists to *check* the CUDA path:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import it;
* the product package ``paper_2505_00690_b200`` never imports it and has no
  CPU fallback (it raises when the CUDA library is missing).

Parity pinning: ``oracle/make_golden.py`` imports the real reference in the
build container and writes ``tests/golden/*.npz``; ``tests/test_oracle_golden.py``
checks this restatement against those fixtures bit-for-bit.  The reference's
third-party arithmetic dependency is numpy 2.3.5 (Generator/PCG64/SeedSequence,
pairwise sums, OpenBLAS fp32 GEMM / fp64 dot); where the reference calls BLAS
the oracle uses the explicit formula measured in DESIGN.md §3 instead, so the
oracle does not depend on which OpenBLAS kernel the host CPU selects.
"""
