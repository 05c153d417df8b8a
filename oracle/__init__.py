"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the TAR+RHT hot path.

This package restates, in numpy, the reference ``ubar`` algorithm for the one
path this repo accelerates (RHT encode -> Transpose AllReduce with masked mean
-> masked RHT decode).  Every function cites the reference file:line it
follows (paths are relative to ``/root/reference/pkg/src/ubar/``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import it, and only as the checker or as the
timed CPU baseline.  The product package ``paper_2310_06993_b200`` never
imports it; the product fails loudly when its CUDA library is missing.

Parity pinning: the oracle is checked against golden vectors produced by the
real reference (``tests/golden/make_golden.py`` imports ``ubar`` from
``/root/reference`` in the build container) and, where the reference is
importable, against the reference live (``tests/test_oracle_vs_reference.py``).
"""

from .ubar_oracle import *  # noqa: F401,F403
