"""CPU oracle for the ocmg hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import anything under
``oracle/``, and only as the checker or as the timed CPU baseline.  The
product package ``paper_1502_03917_b200`` never imports it; its device path
fails loudly when the CUDA library is missing instead of falling back here.

Parity pin: the reference (``ocmg``, pure Python + numba) ships no tests or
golden vectors.  The oracle is pinned against fixtures
produced by running the reference itself in the build container
(``tests/golden/gen_golden.py`` -> ``tests/golden/*.npz``), see
``tests/test_oracle_golden.py``.
"""
from .ocmg_oracle import *  # noqa: F401,F403
