"""Local finite-difference operators (reference: localexp/localop.py:19-128).

Weights come from the device Fornberg kernel (lmep_fornberg), which keeps the
reference recursion's evaluation order and roundings, so tables are
bit-identical to ``localexp.fornberg_weights``.  Node-set validation runs on
the host (it inspects at most 32 numbers).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _ops
from .errors import OrderTooHigh


@dataclass(frozen=True)
class LinearOperatorSpec:
    """Constant-coefficient operator sum_k c_k d^k/dx^k (localop.py:19-49)."""

    terms: tuple[tuple[int, float], ...]

    def __post_init__(self):
        terms = tuple((int(k), float(c)) for k, c in self.terms)
        object.__setattr__(self, "terms", terms)
        if not terms:
            raise ValueError("operator needs at least one term")
        orders = [k for k, _ in terms]
        if len(set(orders)) != len(orders):
            raise ValueError("derivative orders must be distinct")
        if min(orders) < 0:
            raise ValueError("derivative orders must be >= 0")

    @property
    def max_order(self) -> int:
        return max(k for k, _ in self.terms)

    @property
    def reaction(self) -> float:
        return next((c for k, c in self.terms if k == 0), 0.0)


@dataclass(frozen=True)
class VariableCoefficientSpec:
    """Per-node coefficients.  Default (frozen at the target node, SURVEY
    Appendix B.3): node i's local operator is sum_t coef[i, t] * D^(orders[t])
    (+ reaction[i] * I), equal to ``LinearOperatorSpec(tuple(zip(orders,
    coef[i])))`` bit for bit (M12).  row_scaled=True: the stencil restriction
    of sum_t diag(coef[:, t]) D^(orders[t]) + diag(reaction), i.e. local row j
    of node i's operator uses the coefficients of the stencil member m_j
     -- a different discretisation.
    Extension of the reference API for BASELINE config 5."""

    orders: tuple[int, ...]
    coef: np.ndarray            # (N, len(orders))
    reaction: np.ndarray | None = None
    row_scaled: bool = False

    def __post_init__(self):
        orders = tuple(int(k) for k in self.orders)
        object.__setattr__(self, "orders", orders)
        if not orders or min(orders) < 1 or len(set(orders)) != len(orders):
            raise ValueError("orders must be distinct and >= 1 (use `reaction` for order 0)")
        c = self.coef if isinstance(self.coef, torch.Tensor) else np.asarray(self.coef, float)
        if c.ndim != 2 or c.shape[1] != len(orders):
            raise ValueError("coef must be (N, len(orders))")

    @property
    def max_order(self) -> int:
        return max(self.orders)


@dataclass(frozen=True)
class DiffMatrix:
    order: int
    nodes: np.ndarray
    entries: np.ndarray


def fornberg_weights(z: float, nodes, max_order: int) -> np.ndarray:
    """(max_order+1, n) weights for d^k/dx^k at z from samples at nodes
    (localop.py:61-96), computed by lmep_fornberg."""
    x = np.asarray(nodes, dtype=np.float64)
    _ops.check_nodes(x, max_order)
    xt = _ops.dev_f64(x[None, :])
    zt = _ops.dev_f64([float(z)])
    return _ops.to_host(_ops.fornberg_dev(zt, xt, int(max_order))[0])


def diff_matrix(nodes, k: int) -> DiffMatrix:
    """D^(k) with row i differentiating at nodes[i] (localop.py:99-108)."""
    x = np.asarray(nodes, dtype=np.float64)
    n = x.size
    if not 1 <= k <= n - 1:
        raise OrderTooHigh(f"order {k} not representable on {n} nodes")
    _ops.check_nodes(x, k)
    tab = _ops.derivative_tables(_ops.dev_f64(x[None, :]), k)[0]   # [i, k, j]
    return DiffMatrix(order=k, nodes=x, entries=_ops.to_host(tab[:, k, :]))


def local_operator(nodes, spec: LinearOperatorSpec) -> np.ndarray:
    """Dense c_0 I + sum_k c_k D^(k) on the nodes (localop.py:111-128): rows
    accumulated in term order from zeros, reaction added last."""
    x = np.asarray(nodes, dtype=np.float64)
    n = x.size
    if spec.max_order > n - 1:
        raise OrderTooHigh(f"operator order {spec.max_order} not representable on {n} nodes")
    _ops.check_nodes(x, spec.max_order)
    L = torch.zeros((n, n), dtype=torch.float64, device=_ops.nat.device())
    if spec.max_order > 0:
        tab = _ops.derivative_tables(_ops.dev_f64(x[None, :]), spec.max_order)[0]
        for k, c in spec.terms:
            if k > 0:
                L = L + c * tab[:, k, :]
    c0 = spec.reaction
    if c0 != 0.0:
        idx = torch.arange(n, device=L.device)
        L[idx, idx] = L[idx, idx] + c0
    return _ops.to_host(L)
