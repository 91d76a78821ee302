"""1D grids and stencil windows (reference: localexp/grid.py:21-175).

The reference materialises one ``Stencil`` object per node (an O(N) Python
loop, 6-9 s at N=2^20) and later stacks their member indices
into an (N, n) int64 array.  Here a stencil assignment is a ``StencilSet``:
the four numbers (N, n, row, periodic) that determine every window
arithmetically,

    periodic:      members(t) = (t - row + j) mod N,      target_row = row
    non-periodic:  start = clamp(t - row, 0, N - n),      target_row = t - start

It still behaves as the reference's list (``len``, indexing and iteration
yield ``Stencil`` objects on demand), so code written against the reference
keeps working, while the device kernels derive windows from the numbers.
"""

from __future__ import annotations

from collections.abc import Sequence
from dataclasses import dataclass
from enum import Enum

import numpy as np

from .errors import InvalidGrid, StencilTooLarge


class Topology(Enum):
    PERIODIC_UNIFORM = "periodic-uniform"
    NON_PERIODIC = "non-periodic"


class StencilPolicy(Enum):
    CENTERED = "centered"
    ONE_SIDED_UPWIND = "upwind"


@dataclass(frozen=True)
class Grid:
    """Sorted 1D nodes on [x_min, x_max] with a topology (grid.py:31-70)."""

    nodes: np.ndarray
    x_min: float
    x_max: float
    topology: Topology
    # Set by make_uniform_grid: stencil coordinates are then offsets * h
    # exactly (as on periodic grids) instead of nodes[m] - nodes[t].
    uniform_spacing: float | None = None

    def __post_init__(self):
        x = np.ascontiguousarray(np.asarray(self.nodes, dtype=np.float64))
        x.setflags(write=False)
        object.__setattr__(self, "nodes", x)
        if x.ndim != 1 or x.size < 2:
            raise InvalidGrid("a grid needs at least two nodes")
        gaps = np.diff(x)
        if (gaps <= 0).any():
            raise InvalidGrid("nodes must increase strictly")
        if not self.x_max > self.x_min:
            raise InvalidGrid("x_max must exceed x_min")
        if self.topology is Topology.PERIODIC_UNIFORM:
            h = (self.x_max - self.x_min) / x.size
            if (np.abs(gaps - h) > 1e-14 * abs(h) * x.size).any():
                raise InvalidGrid("a periodic grid must be uniform")
        elif self.uniform_spacing is None and x.size >= 3:
            # a reference-style uniform grid, Grid(nodes=np.linspace(a, b, N)):
            # equispaced to the rounding of its own construction -> stencil
            # coordinates offsets * h (position classes, shardable), as
            # make_uniform_grid's (DESIGN 5.5)
            h = (x[-1] - x[0]) / (x.size - 1)
            tol = 8.0 * np.finfo(np.float64).eps * max(abs(x[0]), abs(x[-1]), abs(h))
            ideal = x[0] + h * np.arange(x.size, dtype=np.float64)
            if np.abs(x - ideal).max() <= tol:
                object.__setattr__(self, "uniform_spacing", float(h))

    @property
    def size(self) -> int:
        return int(self.nodes.size)

    @property
    def periodic(self) -> bool:
        return self.topology is Topology.PERIODIC_UNIFORM

    @property
    def h_min(self) -> float:
        return float(np.diff(self.nodes).min())

    @property
    def spacing(self) -> float:
        if not self.periodic:
            raise InvalidGrid("spacing is defined for uniform periodic grids only")
        return (self.x_max - self.x_min) / self.size


@dataclass(frozen=True)
class Stencil:
    """Window of node indices feeding one node (grid.py:73-103)."""

    target: int
    members: np.ndarray
    target_row: int

    def __post_init__(self):
        m = np.ascontiguousarray(np.asarray(self.members, dtype=np.int64))
        m.setflags(write=False)
        object.__setattr__(self, "members", m)
        if np.unique(m).size != m.size:
            raise InvalidGrid("stencil members must be distinct")
        if not 0 <= self.target_row < m.size:
            raise InvalidGrid("target_row out of range")
        if int(m[self.target_row]) != int(self.target):
            raise InvalidGrid("members[target_row] must be the target")

    @property
    def n(self) -> int:
        return int(self.members.size)

    @property
    def offsets(self) -> np.ndarray:
        return np.arange(self.n, dtype=np.int64) - self.target_row


class StencilSet(Sequence):
    """Structured stencil assignment of a whole grid (see module docstring)."""

    def __init__(self, N: int, n: int, row: int, periodic: bool):
        self.N, self.n, self.row, self.periodic = int(N), int(n), int(row), bool(periodic)

    # window arithmetic ----------------------------------------------------
    def starts(self, t) -> np.ndarray:
        t = np.asarray(t, dtype=np.int64)
        if self.periodic:
            return t - self.row
        return np.clip(t - self.row, 0, self.N - self.n)

    def target_rows(self, t=None) -> np.ndarray:
        t = np.arange(self.N, dtype=np.int64) if t is None else np.asarray(t, dtype=np.int64)
        return t - self.starts(t)

    def members_array(self) -> np.ndarray:
        """The reference's stacked (N, n) int64 member array (harvest.py:172)."""
        t = np.arange(self.N, dtype=np.int64)
        m = self.starts(t)[:, None] + np.arange(self.n, dtype=np.int64)[None, :]
        return m % self.N if self.periodic else m

    # boundary classes (non-periodic): nodes whose window is clamped
    @property
    def n_left(self) -> int:
        return 0 if self.periodic else self.row

    @property
    def n_right(self) -> int:
        return 0 if self.periodic else self.n - 1 - self.row

    # Sequence protocol ----------------------------------------------------
    def __len__(self) -> int:
        return self.N

    def __getitem__(self, t):
        if isinstance(t, slice):
            return [self[i] for i in range(*t.indices(self.N))]
        t = int(t)
        if t < 0:
            t += self.N
        if not 0 <= t < self.N:
            raise IndexError(t)
        s = int(self.starts(t))
        m = s + np.arange(self.n, dtype=np.int64)
        if self.periodic:
            m %= self.N
        return Stencil(target=t, members=m, target_row=t - s)

    def __repr__(self) -> str:
        kind = "periodic" if self.periodic else "clamped"
        return f"StencilSet(N={self.N}, n={self.n}, row={self.row}, {kind})"


def make_periodic_grid(N: int, x_min: float, x_max: float) -> Grid:
    """Uniform periodic nodes x_j = x_min + j*h, right end excluded (grid.py:106-114)."""
    if N < 3:
        raise InvalidGrid(f"periodic grid needs N >= 3, got {N}")
    if not x_max > x_min:
        raise InvalidGrid("x_max must exceed x_min")
    h = (x_max - x_min) / N
    return Grid(nodes=x_min + h * np.arange(N), x_min=x_min, x_max=x_max,
                topology=Topology.PERIODIC_UNIFORM)


def make_uniform_grid(N: int, x_min: float, x_max: float) -> Grid:
    """Uniform non-periodic nodes including both ends (np.linspace), the grid
    of BASELINE config 4."""
    if N < 3:
        raise InvalidGrid(f"grid needs N >= 3, got {N}")
    return Grid(nodes=np.linspace(x_min, x_max, N), x_min=x_min, x_max=x_max,
                topology=Topology.NON_PERIODIC, uniform_spacing=(x_max - x_min) / (N - 1))


def make_chebyshev_grid(N: int, x_min: float, x_max: float) -> Grid:
    """Chebyshev-Gauss-Lobatto nodes, ascending, exact ends (grid.py:117-133)."""
    if N < 3:
        raise InvalidGrid(f"Chebyshev grid needs N >= 3, got {N}")
    if not x_max > x_min:
        raise InvalidGrid("x_max must exceed x_min")
    m = N - 1
    ref = -np.sin((m - 2 * np.arange(N)) * np.pi / (2 * m))
    x = 0.5 * (x_min + x_max) + 0.5 * (x_max - x_min) * ref
    x[0], x[-1] = x_min, x_max
    return Grid(nodes=x, x_min=x_min, x_max=x_max, topology=Topology.NON_PERIODIC)


def select_stencils(grid: Grid, n: int, policy: StencilPolicy, upwind_sign: int = 1) -> StencilSet:
    """Assign an n-node window to every node (grid.py:136-175).  Returns a
    StencilSet, which iterates like the reference's list of Stencils."""
    N = grid.size
    if n > N:
        raise StencilTooLarge(f"stencil size {n} exceeds grid size {N}")
    if n < 1:
        raise StencilTooLarge("stencil size must be positive")
    if policy is StencilPolicy.CENTERED and n % 2 == 0 and n != N:
        raise InvalidGrid("centered stencils require odd n")
    if policy is StencilPolicy.CENTERED:
        row = (n - 1) // 2
    else:
        row = n - 1 if upwind_sign >= 0 else 0
    return StencilSet(N, n, row, grid.periodic)


def as_stencil_set(grid: Grid, stencils) -> StencilSet:
    """Accept a StencilSet or a reference-style list of Stencils and return the
    structured description.  Only contiguous windows (the reference's
    select_stencils output) have a device path; anything else raises."""
    from .errors import InvalidConfig

    if isinstance(stencils, StencilSet):
        if stencils.N != grid.size or stencils.periodic != grid.periodic:
            raise InvalidConfig("stencil set does not belong to this grid")
        return stencils
    st = list(stencils)
    N = grid.size
    if len(st) != N:
        raise InvalidConfig("one stencil per node required")
    n = st[0].n
    mid = st[N // 2]
    row = int(mid.target_row)
    cand = StencilSet(N, n, row, grid.periodic)
    members = np.array([s.members for s in st], dtype=np.int64)
    rows = np.array([s.target_row for s in st], dtype=np.int64)
    if not (np.array_equal(members, cand.members_array()) and
            np.array_equal(rows, cand.target_rows())):
        raise InvalidConfig("only contiguous select_stencils windows have a device path")
    return cand
