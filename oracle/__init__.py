"""CPU oracle for the starm t-SVDM hot path -- TEST INFRASTRUCTURE ONLY.

This package is a numpy/scipy restatement of the reference algorithm
(``/root/reference/pkg/src/starm``) used as the parity checker for the
B200 CUDA path.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline / ``--impl reference`` arms may import it.
The product package ``paper_2605_16058_b200`` never imports it and has no
CPU fallback.

Parity pin: the restatement is checked against outputs of the reference
package itself, generated in the build container by
``tests/golden/make_golden.py`` (which imports the reference read-only) and
committed as ``tests/golden/*.npz``.  See ``tests/test_oracle_golden.py``.
"""

from .starm_oracle import *  # noqa: F401,F403
