"""errors.adopt(slbm.errors) makes the engines report the reference's own
Parity enum (exchange.py:313-316 compares by identity).  CPU only: the
enum plumbing, no engine is built."""

import pytest

from conftest import import_reference


def test_adopt_swaps_parity_class_and_back():
    slbm = import_reference()
    from paper_2408_06880_b200 import collision, errors

    try:
        errors.adopt(slbm.errors)
        P = collision.parity_class()
        assert P is slbm.core.Parity
        assert slbm.exchange.phase_for("aa", P.EVEN) is slbm.exchange.Phase.CANONICAL
        assert slbm.exchange.phase_for("aa", P.EVEN.flipped()) is slbm.exchange.Phase.REVERSED
        assert collision.is_even(P.EVEN) and not collision.is_even(P.ODD)
        assert collision.as_parity(collision.Parity.ODD) is P.ODD
        assert errors.error_class("ProtocolError") is slbm.errors.ProtocolError
    finally:
        errors.reset()
    assert collision.parity_class() is collision.Parity
    assert errors.error_class("ProtocolError") is errors.ProtocolError


def test_adopt_rejects_foreign_enum():
    from enum import Enum

    from paper_2408_06880_b200 import collision, errors

    class Bad(Enum):
        EVEN = 1
        ODD = 0

    with pytest.raises(errors.ConfigurationError):
        collision.adopt_parity(Bad)
    assert collision.parity_class() is collision.Parity
