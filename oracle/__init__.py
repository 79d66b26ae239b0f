"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the forward-solve hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline.  The product package ``paper_2212_00964_b200`` never
imports it and has no CPU fallback.

Parity status: PINNED.  ``tests/golden/*.npz`` were produced by running the
reference package itself (``tests/golden/make_golden.py`` imports gradfem from
/root/reference/pkg/src in the build container); ``tests/test_oracle_golden.py``
checks this oracle against every fixture (bit-exact for integer maps, FP64
within the tolerances written in the tests).
"""

from .gradfem_oracle import *  # noqa: F401,F403
