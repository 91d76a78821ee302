"""Dense matrix exponentials on the device (reference: localexp/expm.py:24-42).

``expm`` keeps the reference contract -- finiteness guard, diagonal
balancing, Pade scaling-and-squaring, overflow guard raising NonFinite -- but
runs as one warp per matrix in lmep_expm and accepts a batch [B, d, d].
"""

from __future__ import annotations

import numpy as np
import torch

from . import _ops
from .errors import NonFinite


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
    bad = int((status != 0).sum().item())
    if bad:
        raise NonFinite("matrix exponential input contains NaN/Inf or overflowed")
    E = E if batch else E[0]
    return E if as_torch else _ops.to_host(E)


def expm_with_stats(A: torch.Tensor):
    """Batched device expm returning (E, status, pade_degree, squarings)."""
    E, status, ms = _ops.expm_batched(_ops.dev_f64(A))
    return E, status, ms & 0xFF, ms >> 8
