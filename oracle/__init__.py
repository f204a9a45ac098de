"""TEST INFRASTRUCTURE ONLY — CPU oracle for the sparse LBM hot path.

A numpy restatement of the reference package's algorithm (paths relative
to ``/root/reference/pkg/src/slbm/``), used exclusively as the *checker*:

* by ``tests/`` (parity of the CUDA engine against it),
* by ``__graft_entry__.smoke()`` (one tiny parity check),
* by ``bench.py``'s ``cpu_baseline`` leg and ``--impl reference`` arm (the
  timed reference CPU path).

Nothing in ``paper_2408_06880_b200`` imports this package; the product
path raises when the CUDA library is missing instead of falling back here.

Parity of the oracle itself is pinned: ``tests/golden/*.npz``
were produced by running the unmodified reference in the build container
(``tools/make_golden.py``), and ``tests/test_oracle_golden.py`` checks this
restatement against every one of them bit for bit; when ``/root/reference``
is present, ``tests/test_oracle_vs_reference.py`` additionally compares
against the live reference on random cases.
"""

from .sparse_ref import OracleSparseEngine, build_lists, collide, equilibrium, moments  # noqa: F401
