"""Collision configuration and in-place storage parity.

``CollisionParams`` validates like the reference (``pkg/src/slbm/core.py:
50-74``) and adds the cumulant model the reference lacks (
its parity is *unpinned*).  The arithmetic itself lives in
the CUDA kernels (``csrc/collide.cuh``); there is deliberately no host
implementation of it in the product package.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

from . import errors
from .lattice import CS2

UBB_WALL_DENSITY = 1.0

MODELS = ("srt", "trt", "cumulant")
MODEL_CODE = {"srt": 0, "trt": 1, "cumulant": 2}


class Parity(Enum):
    """EVEN: slot (q, cell) holds the value moving along q.  ODD: the state
    left by the combined (index-list) AA step, values parked in the
    opposite-direction slots.  The reference names the combined step's
    input EVEN (``core.py:32-47``; the paper calls that step "odd")."""

    EVEN = 0
    ODD = 1

    def flipped(self) -> "Parity":
        return Parity.ODD if self is Parity.EVEN else Parity.EVEN


# The Parity class the engines report.  A host application that compares
# parities by identity (the reference's ``exchange.phase_for`` does
# ``parity is Parity.EVEN``, ``exchange.py:313-316``) adopts its own enum
# through :func:`adopt_parity` (``errors.adopt`` does this for the
# reference package); internally parities are compared by ``.value``.
_parity_cls = [Parity]


def parity_class():
    return _parity_cls[0]


def adopt_parity(cls) -> None:
    """Report parities as members of ``cls`` (an Enum with EVEN=0, ODD=1
    and ``flipped()``, e.g. ``slbm.core.Parity``) from now on."""
    if cls.EVEN.value != 0 or cls.ODD.value != 1:
        raise errors.make("ConfigurationError", f"{cls!r} is not an EVEN=0/ODD=1 parity enum")
    _parity_cls[0] = cls


def is_even(parity) -> bool:
    return getattr(parity, "value", parity) == 0


def as_parity(parity):
    """``parity`` (any EVEN/ODD enum or 0/1) as a member of the adopted class."""
    return parity_class()(getattr(parity, "value", parity))


@dataclass
class CollisionParams:
    """Reference fields (core.py:50-74) plus, for the cumulant model only
    (extension, unpinned; Geier et al. 2015 §4): ``bulk_omega`` = w2, the
    rate of the trace of the second-order cumulants (bulk viscosity
    zeta = 2/9 (1/w2 - 1/2)), and ``higher_omegas`` = (w3, ..., w10) for the
    third- to sixth-order cumulants (None: all 1, the closed-form kernel)."""

    omega: float
    model: str = "srt"
    lambda_odd: float | None = None
    bulk_omega: float = 1.0
    higher_omegas: tuple | None = None

    def __post_init__(self) -> None:
        if not (0.0 < self.omega < 2.0):
            raise errors.make("ConfigurationError", f"omega must lie in (0, 2), got {self.omega}")
        if self.model not in MODELS:
            raise errors.make("ConfigurationError", f"unknown collision model {self.model!r}")
        if self.model == "trt":
            if self.lambda_odd is None:
                raise errors.make("ConfigurationError", "trt requires lambda_odd")
            if not (0.0 < self.lambda_odd < 2.0):
                raise errors.make(
                    "ConfigurationError", f"lambda_odd must lie in (0, 2), got {self.lambda_odd}"
                )
        if self.model != "cumulant" and (self.bulk_omega != 1.0 or self.higher_omegas is not None):
            raise errors.make("ConfigurationError", "bulk / higher-order rates are cumulant-only")
        rates = [self.bulk_omega] + list(self.higher_omegas or [])
        if self.higher_omegas is not None and len(self.higher_omegas) != 8:
            raise errors.make("ConfigurationError", "higher_omegas needs 8 rates (w3..w10)")
        if not all(0.0 < float(w) < 2.0 for w in rates):
            raise errors.make("ConfigurationError", f"cumulant rates must lie in (0, 2), got {rates}")


def omega_from_viscosity(nu: float) -> float:
    if nu <= 0.0:
        raise errors.make("ConfigurationError", f"viscosity must be positive, got {nu}")
    return 1.0 / (nu / CS2 + 0.5)


def viscosity_from_omega(omega: float) -> float:
    if not (0.0 < omega < 2.0):
        raise errors.make("ConfigurationError", f"omega must lie in (0, 2), got {omega}")
    return CS2 * (1.0 / omega - 0.5)


def trt_magic_lambda(omega: float, magic: float = 3.0 / 16.0) -> float:
    """Odd rate giving the TRT "magic" parameter Lambda = (1/w_e - 1/2)(1/w_o - 1/2)."""
    even = 1.0 / omega - 0.5
    return 1.0 / (magic / even + 0.5)


def params_code(params) -> tuple[int, float, float]:
    """(model code, omega, lambda_odd) for the C-ABI; accepts the
    reference's CollisionParams too (duck-typed)."""
    model = getattr(params, "model", "srt")
    if model not in MODEL_CODE:
        raise errors.make("ConfigurationError", f"unknown collision model {model!r}")
    if model == "cumulant":  # the second rate word carries the bulk rate
        return MODEL_CODE[model], float(params.omega), float(getattr(params, "bulk_omega", 1.0))
    lam = getattr(params, "lambda_odd", None)
    return MODEL_CODE[model], float(params.omega), float(lam if lam is not None else params.omega)


def cumulant_rates(params):
    """(bulk, higher (8,) or None) of a cumulant CollisionParams (duck-typed)."""
    higher = getattr(params, "higher_omegas", None)
    return float(getattr(params, "bulk_omega", 1.0)), (None if higher is None else tuple(higher))
