import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"
# the unmodified reference installed by tools/install_reference.sh; it travels
# to the GPU box with the snapshot (git-ignored), /root/reference does not
REFERENCE_INSTALL = os.path.join(ROOT, "baseline", "_ref")


def reference_paths():
    """(package dir, tests dir) of an importable unmodified reference, or
    (None, None).  Prefers the in-tree install (present on the GPU box)."""
    inst = REFERENCE_INSTALL
    if os.path.isdir(os.path.join(inst, "slbm")):
        tests = os.path.join(inst, "slbm_tests")
        return inst, tests if os.path.isdir(tests) else None
    if os.path.isdir(REFERENCE_SRC):
        return REFERENCE_SRC, "/root/reference/pkg/tests"
    return None, None


def import_reference():
    """The reference package ``slbm`` (imported read-only), or skip."""
    src, _ = reference_paths()
    if src is None:
        pytest.skip("reference package not installed (tools/install_reference.sh)")
    sys.dont_write_bytecode = True
    if src not in sys.path:
        sys.path.insert(0, src)
    import slbm
    import slbm.core
    import slbm.dense
    import slbm.domain
    import slbm.errors
    import slbm.exchange
    import slbm.flags
    import slbm.geometry
    import slbm.sparse
    import slbm.stencil

    return slbm


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running")


def golden_files(prefix):
    return sorted(glob.glob(os.path.join(GOLDEN, f"{prefix}_*.npz")))


def load_golden(path):
    with np.load(path, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def golden_id(path):
    return os.path.basename(path)[:-4]


def flags_of(rec):
    from paper_2408_06880_b200.tags import FlagField

    return FlagField(
        dims=tuple(int(d) for d in rec["dims"]),
        tags=rec["tags"].astype(np.uint8),
        ubb_u=rec["ubb_u"].astype(np.float64),
        periodic=tuple(bool(p) for p in rec["periodic"]),
    )


def params_of(rec):
    from paper_2408_06880_b200.collision import CollisionParams

    lam = float(rec["lambda_odd"])
    model = str(rec["model"])
    return CollisionParams(omega=float(rec["omega"]), model=model,
                           lambda_odd=None if model == "srt" else lam)


def stencil_of(rec):
    from paper_2408_06880_b200.lattice import make_stencil

    return make_stencil(str(rec["stencil"]))


def drive(eng, steps, ghost_slot=None, ghost_fill=None):
    """tests/conftest.py:38-43 of the reference, plus fixed halo values."""
    for _ in range(steps):
        if ghost_slot is not None and len(ghost_slot):
            eng.write_slots(ghost_slot, ghost_fill)
        eng.refresh_boundary(eng.parity)
        eng.step()
        eng.finish_step()


def seed_values(flags, st, seed, amplitude=0.01):
    """reference tests/conftest.py:29-60 (values part), via the oracle's
    equilibrium (bit-identical to core.equilibrium_fields)."""
    from oracle.sparse_ref import equilibrium

    rng = np.random.default_rng(seed)
    shape = tuple(reversed(flags.dims))
    rho = 1.0 + amplitude * rng.standard_normal(shape)
    u = amplitude * rng.standard_normal((st.dim,) + shape)
    mask = flags.tags[tuple(slice(1, n + 1) for n in shape)] == 0
    return equilibrium(rho[mask], u.reshape(st.dim, -1)[:, mask.reshape(-1)], st)


@pytest.fixture(scope="session")
def gpu_lib():
    """The built CUDA library, or a loud failure (no fallback)."""
    from paper_2408_06880_b200 import _abi

    return _abi.load()
