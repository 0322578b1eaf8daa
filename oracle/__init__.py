"""CPU oracle for the rGSVD hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and
only as the checker or the timed CPU baseline. The product package
(``paper_2404_09459_b200``) never imports it and has no CPU fallback.

``oracle.rgsv_oracle`` restates, in numpy, the reference package ``rgsv``
0.1.0 (``/root/reference/pkg/src/rgsv``) for the hot path: fixed-width
Gaussian range finder + q power iterations, projection, stacked QR, L-block
singular values, spectrum completion/classification and the comparative
quantities. Every function cites the reference file:line it follows.

Pinning: at q = 0 the restatement reproduces the reference bit for bit on
the same numpy/OpenBLAS (checked by ``tests/test_oracle.py`` against the
golden vectors in ``tests/golden/`` that ``tests/golden/make_golden.py``
produced by importing the reference itself). For q >= 1 the reference has
no implementation: that leg is a restatement of the
standard subspace iteration built only from reference primitives, and is
"parity unpinned" beyond those primitives.
"""
