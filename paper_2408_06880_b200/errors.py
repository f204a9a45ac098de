"""Error vocabulary of the drop-in engine.

The class names and hierarchy match the reference package
(``pkg/src/slbm/errors.py:4-29``) so callers written against it catch the
same things.  The C-ABI reports failures as integer status codes
(``include/slbm_b200.h``); :func:`raise_for_status` turns a status plus
the library's last message into the matching exception.

Integrators that already import the reference's own exception classes can
call :func:`adopt` with that module; the engine then raises *those*
classes, so ``except slbm.errors.NumericalInstabilityError`` keeps working
when the engine is swapped in.
"""

from __future__ import annotations


class SlbmError(Exception):
    """Root of every error the solver raises."""


class ConfigurationError(SlbmError):
    """Bad parameter, shape, phase name, or a geometry the solver cannot use."""


class NumericalInstabilityError(SlbmError):
    """A collision saw a density that is <= 0 or not finite."""


class FormatError(SlbmError):
    """A mask or message byte stream is malformed."""


class ProtocolError(SlbmError):
    """Halo exchange addressed a slot or route the receiver does not have."""


class EmptyBlockError(SlbmError):
    """The block holds no fluid cell."""


class UnreachablePorosityError(SlbmError):
    """A geometry generator cannot reach the requested porosity."""


# status codes shared with the C-ABI (include/slbm_b200.h)
SLBM_OK = 0
SLBM_ECONFIG = 1
SLBM_EEMPTY = 2
SLBM_EUNSTABLE = 3
SLBM_EPROTOCOL = 4
SLBM_ECUDA = 5

_BY_STATUS = {
    SLBM_ECONFIG: "ConfigurationError",
    SLBM_EEMPTY: "EmptyBlockError",
    SLBM_EUNSTABLE: "NumericalInstabilityError",
    SLBM_EPROTOCOL: "ProtocolError",
}

_classes = {
    name: globals()[name]
    for name in (
        "SlbmError",
        "ConfigurationError",
        "NumericalInstabilityError",
        "FormatError",
        "ProtocolError",
        "EmptyBlockError",
        "UnreachablePorosityError",
    )
}


def adopt(module) -> None:
    """Raise the exception classes of ``module`` (e.g. ``slbm.errors``)
    from now on, instead of this package's own.

    When ``module`` belongs to a package with a ``core.Parity`` enum (the
    reference: ``slbm.core.Parity``, ``core.py:32-47``), the engines also
    report their parity as members of that enum, so host code comparing
    parities by identity -- the reference's ``exchange.phase_for``
    (``exchange.py:313-316``) -- takes the right halo phase."""
    import importlib

    for name in list(_classes):
        cls = getattr(module, name, None)
        if cls is not None:
            _classes[name] = cls
    pkg = getattr(module, "__package__", None) or getattr(module, "__name__", "").rpartition(".")[0]
    if pkg:
        try:
            core = importlib.import_module(pkg + ".core")
        except ImportError:
            core = None
        parity = getattr(core, "Parity", None)
        if parity is not None:
            from .collision import adopt_parity

            adopt_parity(parity)


def reset() -> None:
    """Back to this package's own exception and Parity classes."""
    from .collision import Parity, adopt_parity

    for name in list(_classes):
        _classes[name] = globals()[name]
    adopt_parity(Parity)


def error_class(name: str) -> type:
    return _classes[name]


def make(name: str, message: str) -> Exception:
    """Instance of the (possibly adopted) class ``name``; use as
    ``raise errors.make("ConfigurationError", "...")``."""
    return _classes[name](message)


def raise_for_status(status: int, message: str) -> None:
    if status == SLBM_OK:
        return
    name = _BY_STATUS.get(status)
    if name is None:
        raise RuntimeError(f"slbm_b200 CUDA failure: {message}")
    raise _classes[name](message)
