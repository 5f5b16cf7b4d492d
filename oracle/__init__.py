"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference DiscoMatch dual solver
(/root/reference/pkg/src/prodmatch: bdd.py, splitting.py, ilp.py,
kernels.py, dual.py, qn.py, primal.py:83-111).  It exists to check the
B200 product path and to serve as the timed CPU baseline; only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline / --impl
reference) may import it.  The product package never imports it.

Pinning: ``tests/golden/make_golden.py`` runs the real reference
(``prodmatch``) in the build container and records golden outputs;
``tests/test_oracle_golden.py`` checks this restatement against them
bit-for-bit (hybrid mode: within the OpenBLAS dot tolerance).
"""

from .clib import lib, build_oracle  # noqa: F401
