"""CPU oracle for the batch-SOM epoch hot path -- TEST INFRASTRUCTURE ONLY.

This package is a plain numpy restatement of the reference `somkit` package's
per-epoch path (BMU search, influence rows, accumulation, blend, U-matrix,
schedules), each function citing the reference file:line it follows.  It is
the checker, never the product: only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s CPU-baseline / `--impl reference` legs may import it.  The
product path (`paper_1305_1422_b200`) never imports this package and fails
loudly when its CUDA library is missing.

Parity pinning: `tests/golden/make_golden.py` runs the *reference itself*
(importable in the build container from /root/reference/pkg/src) and commits
its outputs as fixtures; `tests/test_oracle_golden.py` checks this oracle
against them (bit-exact BMUs, fp64 accumulators to 1e-12, codebooks to
1 ulp).  The hexagonal grid / bubble neighbourhood / compact-support
extensions have no reference counterpart; they are builder definitions
(DESIGN.md section "Extensions") pinned by hand-computed known answers.
"""

from .somoracle import *  # noqa: F401,F403
from .somoracle import __all__  # noqa: F401
