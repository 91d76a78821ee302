"""Dense matrix exponentials on the device (reference: localexp/expm.py:24-42).

``expm`` keeps the reference contract -- finiteness guard, diagonal
balancing, Pade scaling-and-squaring, overflow guard raising NonFinite -- but
runs as one warp per matrix in lmep_expm and accepts a batch [B, d, d].
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native as nat
from . import _ops
from .errors import NoConvergence, NonFinite

PHI_SERIES_RADIUS = 0.5      # expm.py:21


def expm(a):
    """exp(A) of a square fp64 matrix, or of each matrix of a [B, d, d] batch.
    numpy in -> numpy out; torch in -> torch (device) out."""
    as_torch = isinstance(a, torch.Tensor)
    A = a if as_torch else np.asarray(a, dtype=np.float64)
    if A.ndim not in (2, 3) or A.shape[-1] != A.shape[-2]:
        raise NonFinite(f"expected a square matrix, got shape {tuple(A.shape)}")
    batch = A.ndim == 3
    At = _ops.dev_f64(A if batch else A[None])
    E, status, ms = _ops.expm_batched(At)
    flag = torch.zeros(1, dtype=torch.int32, device=At.device)
    nat.check(nat.lib().lmep_status_any(nat.ptr(status), int(status.numel()), nat.ptr(flag),
                                        nat.stream_handle()), "lmep_status_any")
    if int(flag.item()):
        raise NonFinite("matrix exponential input contains NaN/Inf or overflowed")
    E = E if batch else E[0]
    return E if as_torch else _ops.to_host(E)


def expm_with_stats(A: torch.Tensor):
    """Batched device expm returning (E, status, pade_degree, squarings)."""
    E, status, ms = _ops.expm_batched(_ops.dev_f64(A))
    return E, status, ms & 0xFF, ms >> 8


# ---------------------------------------------------------------------------
# The reference's scalar / plain-series helpers (expm.py:45-83).  They are its
# own cross-check oracles for tests, not part of the harvest or stepping path,
# and are kept host-side with the reference's exact arithmetic so code that
# imports them from the package keeps working.
# ---------------------------------------------------------------------------
def expm_taylor_oracle(a, tol: float = 1e-16, max_terms: int = 200) -> np.ndarray:
    """Plain-series exp(A) for cross-checking expm (expm.py:45-56)."""
    A = np.asarray(a, dtype=float)
    n = A.shape[0]
    result = np.eye(n)
    term = np.eye(n)
    for k in range(1, max_terms + 1):
        term = term @ A / k
        result = result + term
        if np.abs(term).max() <= tol * max(1.0, np.abs(result).max()):
            return result
    raise NoConvergence(f"exp series did not converge in {max_terms} terms")


def phi_scalar(j: int, z):
    """phi_j(z), phi_0 = e^z, phi_{j+1}(z) = (phi_j(z) - 1/j!)/z: the recursion for
    |z| >= 0.5, the series sum_m z^m/(m+j)! below it (expm.py:59-83)."""
    if not 0 <= j <= 8:
        raise ValueError(f"phi order must be in [0, 8], got {j}")
    if j == 0:
        return np.exp(z)
    if abs(z) >= PHI_SERIES_RADIUS:
        phi = np.exp(z)
        for i in range(j):
            phi = (phi - 1.0 / math.factorial(i)) / z
        return phi
    acc = 1.0 / math.factorial(j)
    term = acc
    m = 0
    while True:
        m += 1
        term = term * z / (m + j)
        acc = acc + term
        if abs(term) < 1e-18 * max(1.0, abs(acc)):
            return acc
