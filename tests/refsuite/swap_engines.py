"""pytest plugin: run the reference's OWN test files with the GPU engines
swapped in (SURVEY §4 strategy 1).

Loaded with ``-p swap_engines`` before the reference's test modules are
imported, it rebinds ``slbm.sparse.SparseEngine`` / ``slbm.dense.DenseEngine``
(and the names ``slbm.domain`` imported at ``domain.py:29,33``) to this
package's CUDA engines and adopts the reference's error and Parity classes
(``errors.adopt``).  Nothing in the reference is edited.  At session end it
writes how many GPU engines the suite built to ``$SWAP_ENGINES_REPORT`` so
the caller can prove the swap took effect.
"""

from __future__ import annotations

import json
import os

import slbm.dense
import slbm.domain
import slbm.errors
import slbm.sparse

from paper_2408_06880_b200 import errors as gpu_errors
from paper_2408_06880_b200.engine import DenseEngine as _GpuDense
from paper_2408_06880_b200.engine import SparseEngine as _GpuSparse

_built = {"sparse": 0, "dense": 0}


class GpuSparseEngine(_GpuSparse):
    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        _built["sparse"] += 1


class GpuDenseEngine(_GpuDense):
    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        _built["dense"] += 1


REFERENCE_SPARSE = slbm.sparse.SparseEngine
REFERENCE_DENSE = slbm.dense.DenseEngine

gpu_errors.adopt(slbm.errors)
slbm.sparse.SparseEngine = GpuSparseEngine
slbm.domain.SparseEngine = GpuSparseEngine
if os.environ.get("SWAP_DENSE", "1") == "1":
    slbm.dense.DenseEngine = GpuDenseEngine
    slbm.domain.DenseEngine = GpuDenseEngine


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("SWAP_ENGINES_REPORT")
    if path:
        with open(path, "w") as f:
            json.dump(dict(_built, exitstatus=int(exitstatus)), f)
