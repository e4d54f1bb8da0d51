"""CPU oracle for the aliasing-filter sparse-FFT hot path — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference algorithms (/root/reference/pkg/src/aliasfft/),
each function citing the reference file:line it follows.  It exists to check the
CUDA path, never to be it: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import it.  The
product package (``paper_2011_05749_b200``) never imports this package.

Pinning: ``tests/test_oracle_golden.py`` checks every function here against
golden vectors produced by running the real reference in the build container
(``tests/golden/make_golden.py``, committed with its outputs), plus the
reference's own known-answer tests (N=20 census 3/3/3, plan KATs, Kay weights).
"""
