"""CPU oracle for the incremental-SVD hot path — TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the reference `svdstream` per-tick
update path (arxiv/paper_2605_24514, `pkg/src/svdstream/`).  It exists so
that tests, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` leg of
``bench.py`` have a checker to compare the CUDA engine against.  Nothing in
``paper_2605_24514_b200`` imports it; the product path fails loudly when its
CUDA library is missing instead of falling back here.

Parity pin: ``tests/golden/*.npz`` hold outputs produced by the real
reference (imported from /root/reference by ``tests/golden/make_golden.py``);
``tests/test_oracle_golden.py`` checks this restatement against them.
"""

from .isvd_oracle import *  # noqa: F401,F403
