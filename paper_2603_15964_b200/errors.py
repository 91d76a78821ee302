"""Error types of the drop-in API, tied to the C-ABI status codes.

The class names are the reference's (localexp/errors.py:4-50) so existing
``except`` clauses keep working; each class also records the lmep_status it
stands for (include/lmep.h), and ``for_status`` is the single place a status
code becomes an exception type.
"""

from __future__ import annotations


class LocalExpError(Exception):
    """Root of every error raised by this package."""

    status = -1


class NonFinite(LocalExpError):
    """NaN/Inf met in an input, an exponential or a time integration.

    From the run loop ``state`` is the last finite snapshot and ``time`` its
    time (reference errors.py:24-34); both are None elsewhere.
    """

    status = 1

    def __init__(self, message, state=None, time=None):
        super().__init__(message)
        self.state, self.time = state, time


class DimensionMismatch(LocalExpError):
    status = 2


class InvalidConfig(LocalExpError):
    status = 3


class OrderTooHigh(LocalExpError):
    status = 5


class DuplicateNodes(LocalExpError):
    status = 6


class InvalidGrid(LocalExpError):
    """Grid/stencil geometry rejected (host-side validation only)."""


class StencilTooLarge(LocalExpError):
    """Stencil wider than the grid (host-side validation only)."""


class NoConvergence(LocalExpError):
    """Kept for API compatibility; the device expm always terminates."""


class NotWarmedUp(LocalExpError):
    """Multistep update called with too short a nonlinear history."""


_BY_STATUS = {c.status: c for c in (NonFinite, DimensionMismatch, InvalidConfig, OrderTooHigh,
                                    DuplicateNodes)}


def for_status(code: int) -> type[LocalExpError]:
    return _BY_STATUS.get(int(code), LocalExpError)
