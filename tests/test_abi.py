"""The C-ABI library loads on a CPU-only host and exports every symbol the
public header declares (no compute calls here)."""

import ctypes
import os
import re

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "slbm_b200.h")


def declared_symbols():
    with open(HEADER) as fh:
        text = fh.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(slbm_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_engine_protocol():
    syms = declared_symbols()
    for must in ("slbm_engine_create", "slbm_step", "slbm_finish_step", "slbm_refresh_boundary",
                 "slbm_canonical_state", "slbm_macroscopic", "slbm_slot_index",
                 "slbm_ghost_slot_index", "slbm_read_slots", "slbm_write_slots",
                 "slbm_halo_start", "slbm_nccl_comm_init"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_2408_06880_b200 import _abi

    lib = _abi.load()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_abi.SIGNATURES) == set(declared_symbols())
    assert b"sm_100a" in lib.slbm_version()


def test_status_codes_match_header():
    from paper_2408_06880_b200 import errors

    with open(HEADER) as fh:
        text = fh.read()
    codes = dict(re.findall(r"#define (SLBM_E[A-Z]+|SLBM_OK) (\d+)", text))
    assert int(codes["SLBM_OK"]) == errors.SLBM_OK
    assert int(codes["SLBM_ECONFIG"]) == errors.SLBM_ECONFIG
    assert int(codes["SLBM_EEMPTY"]) == errors.SLBM_EEMPTY
    assert int(codes["SLBM_EUNSTABLE"]) == errors.SLBM_EUNSTABLE
    assert int(codes["SLBM_EPROTOCOL"]) == errors.SLBM_EPROTOCOL
    assert int(codes["SLBM_ECUDA"]) == errors.SLBM_ECUDA


def test_error_classes_can_be_adopted():
    from paper_2408_06880_b200 import errors

    class Foreign:
        class ConfigurationError(Exception):
            pass

    errors.adopt(Foreign)
    try:
        try:
            errors.raise_for_status(errors.SLBM_ECONFIG, "x")
        except Foreign.ConfigurationError:
            pass
    finally:
        errors.adopt(errors)  # restore own classes
    try:
        errors.raise_for_status(errors.SLBM_EPROTOCOL, "y")
    except errors.ProtocolError:
        pass


def test_library_is_built_for_sm100a():
    import subprocess

    from paper_2408_06880_b200 import _abi

    out = subprocess.run(["cuobjdump", "--list-elf", _abi.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        import pytest

        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
    ctypes.CDLL(_abi.LIB_PATH)


def test_tuning_knobs_documented_and_accepted():
    """Every knob the header documents is accepted (host-side state only, no
    GPU work); unknown knobs fail with the configuration error."""
    from paper_2408_06880_b200 import _abi

    with open(HEADER) as fh:
        text = fh.read()
    block = text[text.index("Tuning knobs"):text.index("int slbm_set_tuning")]
    knobs = sorted({int(k) for k in re.findall(r"^\s*\*\s+(\d+)\s", block, flags=re.M)} | {11})
    assert {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12} <= set(knobs)
    lib = _abi.load()
    defaults = {0: 0, 1: 0, 2: 1, 3: 0, 4: 1 << 19, 5: 0, 6: 0, 7: -1, 8: 1, 9: 1, 12: 0, 13: 0}
    for k, v in defaults.items():
        assert lib.slbm_set_tuning(k, v) == 0
    assert lib.slbm_set_tuning(99, 0) != 0
    # the memory probe and the experimental pair kernel are not in the shipped build
    assert lib.slbm_set_tuning(0, 2) != 0
    assert lib.slbm_set_tuning(5, 1) != 0
    assert lib.slbm_set_tuning(0, 0) == 0
    assert lib.slbm_set_tuning(13, 3) != 0  # 0, 4 or 5 CTAs per SM
