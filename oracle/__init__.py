"""oracle — TEST INFRASTRUCTURE ONLY: plain, slow, obviously-correct fp64 reference for the
TPA-SCD hot path of Parnell et al., arXiv 1702.07005 ("Large-Scale Stochastic Learning using
GPUs").  Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` leg and
``--impl reference`` arm may import it.  It shares no code with the CUDA product path
(``paper_1702_07005_b200``); neither imports the other.

Modules:
  ``ridge``   objectives, Fenchel maps, duality gaps, closed form, aggregation γ (numpy/scipy, fp64)
  ``solver``  sequential SCD/SDCA epochs (Alg. 1; C in ``oracle.c``), full solves, and the
              distributed Alg. 3/4 simulator
  ``_lib``    ctypes loader for ``liboracle.so`` (Feistel permutation, partition, transpose,
              norms, epochs)
  ``data``    data-layer references: frequency renumbering of the inner indices, LIBSVM parsing

Pinned by tests/test_oracle_pins.py against what the paper and mathematics fix (closed-form
normal equations, stationarity, monotone objective, strong duality, exact line search, SPEC
hand values).  Parity unpinned (no paper values; invariants only): the permutation, partition
and transpose artefacts — see DESIGN.md §5.
"""
from . import data, ridge, solver  # noqa: F401
from ._lib import block_order, permutation, partition, partition_balanced, transpose, sq_norms, perm_at  # noqa: F401
