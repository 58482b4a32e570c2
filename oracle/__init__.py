"""CPU oracle for the SpeCache decode hot path -- TEST INFRASTRUCTURE ONLY.

This package is a vectorised numpy restatement of the reference's CPU
algorithm (``/root/reference/pkg/src/speckv``).  It exists to *check* the
B200 product path.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it,
and there only as the checker or the timed CPU baseline -- never as the thing
measured or shipped.  The product package ``paper_2503_16163_b200`` never
imports it and fails loudly when its CUDA library is missing.

Parity pinning: ``tests/golden/`` holds fixtures produced by importing the
reference itself (``tests/golden/gen_golden.py``); ``tests/test_oracle.py``
checks this restatement against them bit-for-bit (quantizer, snapshot,
materialize, select_topk) and to BLAS tolerance (attention).
"""
from .restate import *  # noqa: F401,F403
