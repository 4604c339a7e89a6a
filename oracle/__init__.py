"""TEST INFRASTRUCTURE ONLY — the CPU oracle for parity checks.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg (``cpu_baseline`` / ``--impl reference``) may import this package, and
only as the checker or the timed CPU baseline — never on the product path
(``paper_2010_04868_b200`` has no CPU fallback and never imports it).

Contents
* ``oracle.py``  — NumPy restatement of the reference CPU path
  ``scalar_reference`` (tvstencil/baselines.py:43-49, 73-125) plus a
  row-major lexicographic Gauss-Seidel sweep (the loop of the reference test
  test_baselines.py:39-52, generalised to any radius-1 tap set).
* ``stencil_oracle.c`` — the same algorithms in C (compiled with
  -ffp-contract=off: every multiply and add separately rounded), OpenMP over
  axis 0 for Jacobi; bit-exact with the NumPy restatement and with the
  reference itself (tests/golden/, made by tests/golden/make_golden.py by
  importing the real reference package).  ``cref.py`` is its ctypes wrapper.

Pinning: the Jacobi, GS-1D and anti-diagonal ("reference" order) GS paths
are pinned against golden vectors produced by the reference package itself.
The lexicographic box-GS order (BASELINE config 4) has no counterpart in the
reference (its oracle uses the anti-diagonal order); it is
pinned only by (a) equality with the reference for star stencils, where the
two orders coincide, and (b) agreement of three independent restatements
(plain loop, NumPy hyperplane, C loop) — "partially pinned".
"""
