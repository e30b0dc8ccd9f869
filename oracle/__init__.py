"""CPU oracle for the sparse-contraction hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package, and only as the checker / the timed reference
arm. The product package (``paper_2405_16883_b200``) never imports it and has
no CPU execution path.

Two restatements of the reference engine's arithmetic
(/root/reference/pkg/src/sparsetc/engine.py), both float64 and both
bit-identical to ``sparsetc.execute`` on the same inputs:

* ``oracle.restate`` — vectorised numpy ("position-major": the p-th stored
  entry of every row is folded in one vector step, so each output element
  sees exactly the reference's left-to-right order from 0.0);
* ``oracle/stc_oracle.c`` — the same loops in plain C (OpenMP over rows,
  ``-ffp-contract=off``), loaded with ctypes by ``oracle.native``; used for
  configuration-scale parity and as the CPU baseline of bench.py.

Pinning: ``tests/golden/make_golden.py`` runs the real reference (imported
from /root/reference in the build container) on small seeded cases and stores
inputs, outputs and op counters under ``tests/golden/``; ``tests/test_oracle_pin.py``
checks both restatements against those fixtures bit for bit. The
reference has no softmax / scale / ReLU / dense GEMM symbols (its grammar has
only + and *); those restatements are plain float64 numpy
and are pinned only by their definitions.
"""

from . import restate  # noqa: F401
