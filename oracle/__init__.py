"""TEST INFRASTRUCTURE ONLY — CPU oracle for the CHESS decode hot path.

This package is a NumPy restatement of the reference `pagesel` algorithms
(/root/reference/pkg/src/pagesel, cited file:line per function) plus the two
pieces the reference does not ship (sparse paged attention and entropy from
logits).  It exists to check the CUDA path and to time the CPU baseline.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
arm may import it.  The product package (paper_2602_20732_b200) never does.

Pinning: pagesel_ref is validated against golden vectors produced by running
the reference itself in the build container (tests/golden/make_golden.py ->
tests/golden/*.npz|json, checked by tests/test_oracle_golden.py).  The
attention restatement is NOT pinned by the reference (the reference only
counts attention ops, simulate.py:186); it is checked against an independent
dense formulation in tests/test_oracle_golden.py.
"""

from . import attention, pagesel_ref  # noqa: F401
