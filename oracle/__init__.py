"""oracle/ -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct CPU implementations of what the CUDA path
computes, written from PAPER.md (arXiv 2504.00480).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything under ``oracle/``.  The product
package ``paper_2504_00480_b200`` never imports it and shares no code with it.

Modules:
  dense.c / dense.py  float64 dense direct sums (eqs. 1.1, 2.1-2.3)
  fourier.py          eq. (3.2) coefficients, eq. (3.3) truncated-Fourier fast sum,
                      App. A NFFT step by step with the Kaiser-Bessel window,
                      window scaling (reading R2)
  bounds.py           Lemma 4.2/4.3, Theorems 4.4/4.5, eq. (A.3) closed forms
  krylov.py           CG / Lanczos-SLQ objective (eqs. 1.3-1.4) with dense MVMs

Parity status: every function is pinned by a ``-m "not gpu"`` test in
tests/test_oracle_*.py; none is "parity unpinned".
"""
from .dense import dense_apply, kernel_value  # noqa: F401
