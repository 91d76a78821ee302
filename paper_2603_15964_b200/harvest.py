"""Weight harvesting on the device (reference: localexp/harvest.py:31-235).

Reference flow per node (Python loop, harvest.py:135-159):
    coords -> local_operator (Fornberg) -> build_augmented (sn x sn)
           -> expm -> target row(s)
Here the whole set is one batched launch of lmep_harvest: each warp
assembles its node's (or stencil class's) operator from Fornberg tables in
shared memory, exponentiates the reduced (n+s-1) x (n+s-1) transposed
augmentation and writes the target rows.  Which items exist is decided by
the stencil geometry instead of a byte-level cache:

  periodic uniform grid               1 shared item            (W_SHARED)
  uniform non-periodic grid,          row(+1) left classes,     (W_CLASS)
    frozen nodes within {0, N-1}      1 interior, right classes
  anything else (non-uniform grids,   one item per node         (W_PERNODE)
    variable coefficients, ...)

``BandedPropagator`` keeps the reference's fields; its (N, n) arrays are
materialised only when someone reads them.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from . import _ops
from .errors import DimensionMismatch, InvalidConfig
from .grid import Grid, StencilSet, as_stencil_set
from .localop import LinearOperatorSpec, VariableCoefficientSpec

PERNODE_CHUNK = 1 << 20          # nodes per harvest launch on the per-node path


@dataclass(frozen=True)
class PhiWeightSet:
    """w_lin plus the raw dt^j phi_j rows of one node (harvest.py:31-42)."""

    delta_t: float
    w_lin: np.ndarray
    w_phi: tuple[np.ndarray, ...]


class BandedPropagator:
    """Global banded operator (harvest.py:45-70).

    Construct it like the reference, ``BandedPropagator(weights, members,
    periodic, delta_t)``, or internally from device rows.  ``weights`` and
    ``members`` are read-only (N, n) numpy arrays produced on demand;
    ``rows()`` is the compact device form the kernels consume.
    """

    def __init__(self, weights=None, members=None, periodic: bool = False, delta_t: float = 0.0,
                 *, _rows: _ops.CompactRows | None = None):
        self.periodic = bool(periodic)
        self.delta_t = float(delta_t)
        self._rows = _rows
        self._w = self._m = None
        if _rows is None:
            w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
            m = np.ascontiguousarray(np.asarray(members, dtype=np.int64))
            if w.shape != m.shape or w.ndim != 2:
                raise DimensionMismatch("weights and members must share an (N, n) shape")
            w.setflags(write=False)
            m.setflags(write=False)
            self._w, self._m = w, m

    @property
    def weights(self) -> np.ndarray:
        if self._w is None:
            w = _ops.to_host(self._rows.dense()[0])
            w.setflags(write=False)
            self._w = w
        return self._w

    @property
    def members(self) -> np.ndarray:
        if self._m is None:
            m = self._rows.layout.members_array()
            m.setflags(write=False)
            self._m = m
        return self._m

    @property
    def layout(self) -> StencilSet:
        if self._rows is not None:
            return self._rows.layout
        return _ops.validate_members(self._m, self._w.shape)

    def rows(self) -> _ops.CompactRows:
        if self._rows is None:
            lay = _ops.validate_members(self._m, self._w.shape)
            self._rows = _ops.compress(_ops.dev_f64(self._w), lay)
        return self._rows

    @property
    def N(self) -> int:
        return self.layout.N if self._w is None else self._w.shape[0]

    @property
    def n(self) -> int:
        return self.layout.n if self._w is None else self._w.shape[1]

    def __repr__(self) -> str:
        return f"BandedPropagator(N={self.N}, n={self.n}, periodic={self.periodic}, dt={self.delta_t})"


# ---------------------------------------------------------------------------
# single-operator API (harvest.py:73-121)
# ---------------------------------------------------------------------------
def _explicit(L_n, delta_t, s, target_row, frozen_rows=()):
    L = np.asarray(L_n, dtype=np.float64)
    if L.ndim != 2 or L.shape[0] != L.shape[1]:
        raise DimensionMismatch(f"expected a square operator, got shape {L.shape}")
    n = L.shape[0]
    if not 0 <= target_row < n:
        raise DimensionMismatch(f"target row {target_row} out of range for n={n}")
    if not 1 <= s <= 6:
        raise ValueError(f"augmentation depth must be in [1, 6], got {s}")
    if n + s - 1 > nat.MAX_DIM:
        raise DimensionMismatch(f"n + s - 1 must be <= {nat.MAX_DIM}")
    mask = 0
    for j in frozen_rows:
        mask |= 1 << int(j)
    h = _ops.harvest(n, s, delta_t, 1, L=_ops.dev_f64(L[None]), row_default=int(target_row),
                     frozen_default=mask)
    _ops.raise_on_status(h)
    return _ops.to_host(h.rows[0])


def harvest_propagator(L_n, delta_t: float, target_row: int) -> np.ndarray:
    """Row target_row of exp(delta_t L_n) (harvest.py:73-79)."""
    return _explicit(L_n, delta_t, 1, target_row)[0].copy()


def build_augmented(L_n, s: int) -> np.ndarray:
    """The reference's sn x sn block companion matrix (harvest.py:82-94).
    Kept for API parity; the device harvest uses the reduced form."""
    if not 1 <= s <= 6:
        raise ValueError(f"augmentation depth must be in [1, 6], got {s}")
    L = torch.as_tensor(np.asarray(L_n, dtype=np.float64))
    n = L.shape[0]
    A = torch.zeros((s * n, s * n), dtype=torch.float64)
    A[:n, :n] = L
    eye = torch.eye(n, dtype=torch.float64)
    for i in range(s - 1):
        A[i * n:(i + 1) * n, (i + 1) * n:(i + 2) * n] = eye
    return A.numpy()


def harvest_phi_weights(L_n, delta_t: float, s: int, target_row: int,
                        frozen_rows=()) -> PhiWeightSet:
    """w_lin and the raw dt^j phi_j rows from one exponential (harvest.py:97-121)."""
    w = _explicit(L_n, delta_t, s, target_row, frozen_rows)
    return PhiWeightSet(delta_t=delta_t, w_lin=w[0].copy(),
                        w_phi=tuple(w[j].copy() for j in range(1, s)))


# ---------------------------------------------------------------------------
# grid-wide harvest (harvest.py:135-210)
# ---------------------------------------------------------------------------
@dataclass
class _Plan:
    mode: int
    coords: torch.Tensor          # [T, n] local coordinates (T=1 shared, classes, or N)
    rows: np.ndarray              # [T] target rows
    masks: np.ndarray             # [T] frozen bitmasks (uint64)
    nleft: int = 0
    nright: int = 0
    uniform_rows: bool = False    # every item has target row sset.row and no frozen rows


def _frozen_masks(sset: StencilSet, t: np.ndarray, frozen: list[int]) -> np.ndarray:
    masks = np.zeros(t.size, dtype=np.uint64)
    if not frozen:
        return masks
    start = sset.starts(t)
    for f in frozen:
        off = (f - start) % sset.N if sset.periodic else f - start
        hit = (off >= 0) & (off < sset.n)
        masks[hit] |= (np.uint64(1) << off[hit].astype(np.uint64))
    return masks


# Stencil-geometry constants of uniform / periodic grids (window coordinates and
# their derivative tables, a few n x n doubles per geometry), keyed by exactly what
# determines them (spacing, n, target rows, operator terms) -- the analogue of the
# reference's exact-match cache (harvest.py:135-159), which keys whole harvested rows.
# Harvested weights themselves are never cached.
_GEOMETRY: dict = {}


def _geometry(key, make):
    """The memoised value; a later use waits (on the device, stream order) for
    the kernels that produced it."""
    hit = _GEOMETRY.get(key)
    if hit is None:
        if len(_GEOMETRY) >= 64:
            _GEOMETRY.clear()
        v = make()
        _GEOMETRY[key] = (v, torch.cuda.current_stream().record_event(), nat.stream_handle())
        return v
    v, ev, made_on = hit
    if nat.stream_handle() != made_on:       # (same stream: its own order is enough)
        cur = torch.cuda.current_stream()
        cur.wait_event(ev)
        t = v[0] if isinstance(v, tuple) else v
        if t.numel():
            t.record_stream(cur)           # stays allocated for this stream's readers
    return v


def _uniform_h(grid: Grid):
    if grid.periodic:
        return grid.spacing
    return grid.uniform_spacing


def _tables_for(grid: Grid, sset: StencilSet, plan, terms):
    """operator_tables of the plan's windows; memoised for uniform / periodic
    geometries with few windows (shared and class plans, periodic per-node)."""
    h = _uniform_h(grid)
    if h is None or plan.coords.shape[0] > 64:
        return _ops.operator_tables(plan.coords, terms)
    key = ("tables", str(plan.coords.device), sset.n, float(h), np.asarray(plan.rows).tobytes(),
           tuple((int(k), float(c)) for k, c in terms))
    return _geometry(key, lambda: _ops.operator_tables(plan.coords, terms))


_CHECKED: set = set()


def _checked_nodes(grid: Grid, sset: StencilSet, plan, kmax: int) -> None:
    """localop.py:69-74 node checks on the first window; a uniform / periodic
    geometry that passed once is not re-checked (the check raises, it never
    changes anything)."""
    h = _uniform_h(grid)
    key = None if h is None else (sset.n, float(h), int(plan.rows[0]), int(kmax))
    if key is not None and key in _CHECKED:
        return
    _ops.check_nodes(_coords0_host(grid, sset, plan), kmax)
    if key is not None:
        _CHECKED.add(key)


def _coords_for(grid: Grid, sset: StencilSet, t: np.ndarray) -> torch.Tensor:
    """Local coordinates of the windows of nodes t (harvest.py:124-132)."""
    trow = sset.target_rows(t)
    off = np.arange(sset.n, dtype=np.int64)[None, :] - trow[:, None]
    if grid.periodic or grid.uniform_spacing is not None:
        h = grid.spacing if grid.periodic else grid.uniform_spacing
        if trow.size <= 64:
            key = ("coords", str(nat.device()), sset.n, float(h), trow.tobytes())
            return _geometry(key, lambda: _ops.dev_f64(off.astype(np.float64) * h))
        return _ops.dev_f64(off.astype(np.float64) * h)
    nodes = _ops.dev_f64(grid.nodes)
    tt = torch.as_tensor(t, device=nodes.device)
    start = torch.as_tensor(sset.starts(t), device=nodes.device)
    m = start[:, None] + torch.arange(sset.n, device=nodes.device)[None, :]
    return (nodes[m] - nodes[tt][:, None]).contiguous()


def _coords0_host(grid: Grid, sset: StencilSet, plan) -> np.ndarray:
    """The first window's local coordinates on the host (for the node checks):
    computed directly on uniform / periodic grids (the same values _coords_for
    uploads), else read back."""
    if grid.periodic or grid.uniform_spacing is not None:
        h = grid.spacing if grid.periodic else grid.uniform_spacing
        return (np.arange(sset.n, dtype=np.int64) - int(plan.rows[0])).astype(np.float64) * h
    return _ops.to_host(plan.coords[0])


_PLANS: dict = {}


def _plan(grid: Grid, sset: StencilSet, frozen_nodes=(), force_pernode=False) -> _Plan:
    N, n, row = sset.N, sset.n, sset.row
    if grid.periodic and len(frozen_nodes) == 0:
        # one window geometry for the whole ring: the plan depends on (n, row, h) only
        key = (bool(force_pernode), n, row, float(grid.spacing), torch.cuda.current_device())
        hit = _PLANS.get(key)
        if hit is None:
            hit = _PLANS[key] = _plan_uncached(grid, sset, (), force_pernode)
        return hit
    return _plan_uncached(grid, sset, frozen_nodes, force_pernode)


def _plan_uncached(grid: Grid, sset: StencilSet, frozen_nodes=(), force_pernode=False) -> _Plan:
    N, n, row = sset.N, sset.n, sset.row
    frozen = sorted({int(i) for i in frozen_nodes})
    if grid.periodic and not frozen and not force_pernode:
        t = np.array([0])
        return _Plan(nat.W_SHARED, _coords_for(grid, sset, t), np.array([row]),
                     np.zeros(1, np.uint64))
    if (not grid.periodic and grid.uniform_spacing is not None and set(frozen) <= {0, N - 1}
            and not force_pernode and N >= 2 * n + 2):
        nl = row + (1 if 0 in frozen else 0)
        nr = (n - 1 - row) + (1 if N - 1 in frozen else 0)
        t = np.concatenate([np.arange(nl), [N // 2], np.arange(N - nr, N)]).astype(np.int64)
        return _Plan(nat.W_CLASS, _coords_for(grid, sset, t), sset.target_rows(t),
                     _frozen_masks(sset, t, frozen), nl, nr)
    if grid.periodic and not frozen:
        # variable coefficients on a periodic grid: one window geometry for all nodes
        coords = _coords_for(grid, sset, np.array([0]))
        return _Plan(nat.W_PERNODE, coords, np.array([row]), np.zeros(1, np.uint64),
                     uniform_rows=True)
    t = np.arange(N, dtype=np.int64)
    coords = _coords_for(grid, sset, np.array([0]) if grid.periodic else t)
    return _Plan(nat.W_PERNODE, coords, sset.target_rows(t), _frozen_masks(sset, t, frozen))


def _rows_from(plan: _Plan, sset: StencilSet, out: torch.Tensor) -> _ops.CompactRows:
    if plan.mode == nat.W_SHARED:
        return _ops.CompactRows(sset, nat.W_SHARED, out[0].contiguous())
    if plan.mode == nat.W_CLASS:
        nl = plan.nleft
        return _ops.CompactRows(sset, nat.W_CLASS, out[nl].contiguous(), out.contiguous(), nl,
                                plan.nright)
    return _ops.CompactRows(sset, nat.W_PERNODE, pernode=out.contiguous())


def harvest_compact(grid: Grid, sset: StencilSet, spec, delta_t: float, s: int,
                    frozen_nodes=(), stats: dict | None = None,
                    node_range: tuple[int, int] | None = None,
                    pad: int = 0, half: bool = False):
    """Harvest w_lin and the raw dt^j phi_j rows (R = s) for the whole grid.
    node_range=(off, nloc): per-node rows only for the shard's nodes (the
    shared / class modes are grid-wide by construction); pad > 0 (periodic
    per-node only) also harvests the `pad` halo nodes on each side, so a shard
    can fuse several steps per halo exchange.  half=True (s >= 2) returns
    (rows, half_rows): also w_lin and the raw dt/2 phi_1 row at delta_t / 2, the
    ETDRK4 half-step set (timestep.py:294-299), from the same launch
    (lmep_harvest_ex half_out) on the shared / class paths."""
    if not 1 <= s <= 6:
        raise ValueError(f"augmentation depth must be in [1, 6], got {s}")
    n = sset.n
    if n + s - 1 > nat.MAX_DIM:
        raise DimensionMismatch(f"n + s - 1 must be <= {nat.MAX_DIM}")
    varcoef = isinstance(spec, VariableCoefficientSpec)
    plan = _plan(grid, sset, frozen_nodes, force_pernode=varcoef)
    if half and (plan.mode == nat.W_PERNODE or s < 2):
        full = harvest_compact(grid, sset, spec, delta_t, s, frozen_nodes, stats, node_range, pad)
        return full, harvest_compact(grid, sset, spec, delta_t / 2, 2, frozen_nodes, stats,
                                     node_range, pad)
    terms = tuple((k, 1.0) for k in spec.orders) if varcoef else spec.terms
    if max(k for k, _ in terms) > n - 1:
        from .errors import OrderTooHigh
        raise OrderTooHigh(f"operator order {max(k for k, _ in terms)} not representable on {n} nodes")
    _checked_nodes(grid, sset, plan, max(k for k, _ in terms))
    d = nat.device()
    if plan.mode != nat.W_PERNODE:
        tables, cf, c0 = _tables_for(grid, sset, plan, terms)
        T = plan.coords.shape[0]
        h = _ops.harvest(n, s, delta_t, T, tables=tables,
                         table_idx=_ops.dev_i32(np.arange(T)), coef=_ops.dev_f64(cf or [0.0]),
                         coef_stride=0, c0=_ops.dev_f64([c0]), c0_stride=0,
                         rows=_ops.dev_i32(plan.rows),
                         frozen=torch.as_tensor(plan.masks.view(np.int64), device=d), layout=0,
                         half=half)
        _ops.raise_on_status(h)
        if stats is not None:
            stats.setdefault("ms", []).append(h.ms)
        if half:
            return _rows_from(plan, sset, h.rows), _rows_from(plan, sset, h.half)
        return _rows_from(plan, sset, h.rows)
    # per-node path: one item per node (of the shard, plus its halo nodes)
    off, N = (0, sset.N) if node_range is None else (int(node_range[0]), int(node_range[1]))
    if pad and not (grid.periodic and plan.uniform_rows):
        raise InvalidConfig("padded per-node tables are supported on periodic grids only")
    shared_coords = plan.coords.shape[0] == 1
    uniform_rows = plan.uniform_rows
    if pad:
        idx = _wrapped_segments(off - pad, N + 2 * pad, sset.N)
        N += 2 * pad
    else:
        idx = None
    sl = slice(off, off + N)
    rs = varcoef and spec.row_scaled
    if rs:
        # row-scaled: the kernel reads member nodes' coefficients from the
        # whole-grid arrays (lmep_harvest_mapped); item b is node node0 + b
        coef_all = _ops.dev_f64(spec.coef).contiguous()
        react = None if spec.reaction is None else _ops.dev_f64(spec.reaction).contiguous()
        node0 = off - pad
    elif varcoef and idx is None and shared_coords and uniform_rows and \
            _ops.is_host(spec.coef) and N >= PIPELINE_MIN:
        # host coefficients: upload in chunks on the copy stream, each chunk's
        # harvest starting as soon as its slice has landed
        h = _harvest_pipelined(spec, sl, N, n, s, delta_t,
                               lambda: _tables_for(grid, sset, plan, terms)[0], sset.row, sset)
        _ops.raise_on_status(h)
        if stats is not None:
            stats.setdefault("ms", []).append(h.ms)
        return _ops.CompactRows(sset, nat.W_PERNODE, pernode=h.rows)
    elif varcoef:
        if idx is not None:
            cdev = _ops.dev_f64(spec.coef)
            coef_all = torch.cat([cdev[a:b] for a, b in idx], 0).contiguous()
            react = None
            if spec.reaction is not None:
                rdev = _ops.dev_f64(spec.reaction)
                react = torch.cat([rdev[a:b] for a, b in idx], 0).contiguous()
        else:
            coef_all = _ops.dev_f64(spec.coef[sl])
            react = None if spec.reaction is None else _ops.dev_f64(spec.reaction[sl])
    if node_range is not None and not uniform_rows:
        plan = _Plan(plan.mode, plan.coords if shared_coords else plan.coords[sl],
                     plan.rows[sl], plan.masks[sl])
    if shared_coords:
        # one launch writes the SoA [s][n][N] table directly
        tables, cf, c0 = _tables_for(grid, sset, plan, terms)
        if varcoef:
            coef, cs = coef_all, len(spec.orders)
            c0t, c0s = (None, 0) if react is None else (react, 1)
        else:
            coef, cs = _ops.dev_f64(cf or [0.0]), 0
            c0t, c0s = _ops.dev_f64([c0]), 0
        kw = dict(row_default=sset.row, frozen_default=0) if uniform_rows else \
            dict(rows=_ops.dev_i32(plan.rows),
                 frozen=torch.as_tensor(plan.masks.view(np.int64), device=d))
        if rs:
            kw["coef_map"] = (node0, sset.N, grid.periodic)
        h = _ops.harvest(n, s, delta_t, N, tables=tables, coef=coef, coef_stride=cs, c0=c0t,
                         c0_stride=c0s, layout=1, **kw)
        _ops.raise_on_status(h)
        if stats is not None:
            stats.setdefault("ms", []).append(h.ms)
        return _ops.CompactRows(sset, nat.W_PERNODE, pernode=h.rows, pernode_pad=int(pad))
    # per-node coordinates (non-uniform grids): chunked to bound the table memory
    out = torch.empty((s, n, N), dtype=torch.float64, device=d)
    rows_all = _ops.dev_i32(plan.rows)
    masks_all = torch.as_tensor(plan.masks.view(np.int64), device=d)
    for a in range(0, N, PERNODE_CHUNK):
        b = min(N, a + PERNODE_CHUNK)
        B = b - a
        tables, cf, c0 = _ops.operator_tables(plan.coords[a:b], terms)
        tidx = _ops.dev_i32(np.arange(B))
        cmap = None
        if rs:
            coef, cs = coef_all, len(spec.orders)
            c0t, c0s = (None, 0) if react is None else (react, 1)
            cmap = (node0 + a, sset.N, grid.periodic)
        elif varcoef:
            coef, cs = coef_all[a:b].contiguous(), len(spec.orders)
            c0t, c0s = (None, 0) if react is None else (react[a:b].contiguous(), 1)
        else:
            coef, cs = _ops.dev_f64(cf or [0.0]), 0
            c0t, c0s = _ops.dev_f64([c0]), 0
        h = _ops.harvest(n, s, delta_t, B, tables=tables, table_idx=tidx, coef=coef,
                         coef_stride=cs, c0=c0t, c0_stride=c0s, rows=rows_all[a:b].contiguous(),
                         frozen=masks_all[a:b].contiguous(), layout=1, coef_map=cmap)
        _ops.raise_on_status(h)
        if stats is not None:
            stats.setdefault("ms", []).append(h.ms)
        out[:, :, a:b] = h.rows
    return _ops.CompactRows(sset, nat.W_PERNODE, pernode=out)


def _wrapped_segments(start: int, count: int, N: int) -> list[tuple[int, int]]:
    """Nodes start .. start+count-1 taken mod N, as contiguous [a, b) slices in order."""
    out = []
    a = start % N
    while count > 0:
        b = min(N, a + count)
        out.append((a, b))
        count -= b - a
        a = 0
    return out


PIPELINE_MIN = 1 << 18      # nodes; smaller host tables go up in one copy
# growing slices (fractions of N): only the first, small upload is exposed, each
# upload is hidden behind the previous slice's harvest (the harvest runs ~1.8x
# slower than PCIe per item), and few launches keep the persistent harvest
# kernel's per-launch tail small
PIPELINE_FRACTIONS = (1 / 16, 1 / 8, 3 / 16, 1 / 4, 3 / 8)


def _pipeline_bounds(N: int):
    if N < 1 << 16:
        return [(0, N)] if N > 0 else []
    out, a, acc = [], 0, 0.0
    for f in PIPELINE_FRACTIONS:
        acc += f
        b = N if f is PIPELINE_FRACTIONS[-1] else min(N, -(-int(acc * N) // 1024) * 1024)
        if b > a:
            out.append((a, b))
            a = b
    return out


def _harvest_pipelined(spec, sl: slice, N: int, n: int, s: int, delta_t: float,
                       tables_fn, row: int, sset: StencilSet | None = None) -> _ops.HarvestOut:
    """Per-node harvest (one shared window geometry) from HOST coefficients:
    the [N, K] coefficient table goes up in growing slices (_pipeline_bounds;
    multiples of 1024 items, so the block-balanced kernel's superblocks and
    their representative balancing are those of a resident harvest; the
    constant-table kernel keeps the first slice's prepared tables for the later
    slices, lmep_harvest_reuse_prep, so its rows equal a one-launch harvest's bit
    for bit whatever the slicing) on the copy
    stream, and the harvest of slice i (lmep_harvest_chunk into the shared SoA
    output) overlaps the upload of slice i+1.  Every slice is queued before
    tables_fn() builds the derivative tables, so PCIe starts at once."""
    d = nat.device()
    cur = torch.cuda.current_stream(d)
    cp = _ops.copy_stream()
    K = len(spec.orders)
    hc = _ops.host_f64(spec.coef)[sl]
    hr = None if spec.reaction is None else _ops.host_f64(spec.reaction)[sl]
    dr = None if hr is None else torch.empty(N, dtype=torch.float64, device=d)
    out = _ops.HarvestOut(torch.empty((s, n, N), dtype=torch.float64, device=d),
                          torch.empty(N, dtype=torch.int32, device=d),
                          torch.empty(N, dtype=torch.int32, device=d))
    bounds = _pipeline_bounds(N)
    # a streamed linear run (timestep.run): its steps follow the harvest slice by
    # slice, and it sizes the slices for its launch levels
    ls = _ops.take_stream_consumer()
    if ls is not None and (s != 1 or sset is None or sl.start != 0 or N != ls.N or N != sset.N):
        ls = None
    if ls is not None:
        bounds = ls.begin(sset, out.rows, bounds)
    # prefixes the streamed run already sent up from its constructor (same host table)
    eager = ls is not None and ls.eager and hr is None and ls.coef_src is not None and \
        ls.coef_src.data_ptr() == hc.data_ptr() and tuple(ls.coef_dev.shape) == (N, K)
    dc = ls.coef_dev if eager else torch.empty((N, K), dtype=torch.float64, device=d)
    cp.wait_stream(cur)                      # dc / dr (and the stream's buffers) were allocated on cur

    def upload(i):
        """Queue slice i's transfers; returns (coefficients landed, everything landed):
        the harvest of a slice starts behind the first, while its initial state is
        still on the link."""
        a, b = bounds[i]
        if eager:
            ev = ls.eager_event(b)
            if ev is not None:
                return ev
            a = max(a, ls.eager_end())
        if ls is not None and dr is None:
            return ls.send(dc, hc, a, b, cp)         # one library call per slice
        with torch.cuda.stream(cp):
            dc[a:b].copy_(hc[a:b], non_blocking=True)
            if dr is not None:
                dr[a:b].copy_(hr[a:b], non_blocking=True)
            ec = cp.record_event()
            if ls is None:
                return ec, ec
            ls.upload(a, b)
            ev = cp.record_event()
        return ec, ev

    # streamed run: the harvests run on a side stream (they depend on the uploads
    # only), so the harvest of slice i+1 overlaps the step launches of slice i on
    # the compute stream; the steps of a slice wait for its harvest's event
    hs = _ops.copy_stream(2) if ls is not None and ls.active else cur
    if hs is not cur:
        hs.wait_stream(cur)

    def harvest_slice(i, evs):
        a, b = bounds[i]
        ec, ev = evs
        _ops.stream_wait(hs, ec)
        # later slices keep the first slice's prepared tables (lmep_harvest_reuse_prep):
        # the rows are those of a one-launch harvest whatever the slicing
        nat.lib().lmep_harvest_reuse_prep(1 if i > 0 else 0)
        with torch.cuda.stream(hs):
            _ops.harvest(n, s, delta_t, b - a, tables=tables, coef=dc[a:b], coef_stride=K,
                         c0=None if dr is None else dr[a:b], c0_stride=0 if dr is None else 1,
                         row_default=row, frozen_default=0, layout=1, into=out, item0=a)
        if ls is not None:
            if hs is not cur:
                cur.wait_event(hs.record_event())
                _ops.stream_wait(cur, ev)        # (the slice of the initial state)
            ls.ready(b)

    def _run_slices():
        nonlocal tables
        if ls is None:
            # every slice is queued before the tables are built, so PCIe starts at once
            landed = [upload(i) for i in range(len(bounds))]
            _ops.issue_deferred(cp)              # e.g. run()'s initial state, behind the slices
            tables = tables_fn()                 # overlaps the first slices' transfer
            for i, ev in enumerate(landed):
                harvest_slice(i, ev)
        else:
            # streamed run: the host's own enqueue time is on the critical path until
            # the first harvest is queued, so the uploads stay just two slices ahead of
            # the harvests (PCIe never idles: a slice takes longer to land than the
            # host needs to queue a harvest and its step launches)
            # With an eager prefix already on its way (LinearStream's constructor) the
            # first harvest is queued before anything else (its slice is covered by
            # the prefix) and every later slice goes up right behind it, at once: the
            # upload stream never idles and the compute stream starts ~75 us earlier.
            if eager:
                landed = []
                while len(landed) < len(bounds) and ls.eager_event(bounds[len(landed)][1]) is not None:
                    landed.append(upload(len(landed)))           # (events only, nothing to copy)
                tables = tables_fn()
                for i in range(len(bounds)):
                    if i >= len(landed):
                        landed.extend(upload(j) for j in range(len(landed), len(bounds)))
                    harvest_slice(i, landed[i])
                    if i == 0:
                        landed.extend(upload(j) for j in range(len(landed), len(bounds)))
            else:
                landed = [upload(i) for i in range(min(2, len(bounds)))]
                tables = tables_fn()
                for i in range(len(bounds)):
                    harvest_slice(i, landed[i])
                    if i + 2 < len(bounds):
                        landed.append(upload(i + 2))
            ls.uploaded(cp)

    tables = None
    try:
        _run_slices()
    finally:
        nat.lib().lmep_harvest_reuse_prep(0)
    dc.record_stream(cp)
    if dr is not None:
        dr.record_stream(cp)
    if hs is not cur:
        cur.wait_stream(hs)
        for t in (dc, dr, out.rows, out.status, out.ms, out.flag, tables):
            if isinstance(t, torch.Tensor) and t.is_cuda:
                t.record_stream(hs)
    return out


def derivative_compact(grid: Grid, sset: StencilSet, k: int) -> _ops.CompactRows:
    """Banded k-th derivative rows: fornberg_weights(0, coords, k)[k] per stencil
    (timestep.assemble_derivative, timestep.py:218-237)."""
    plan = _plan(grid, sset, ())
    T, n = plan.coords.shape
    _ops.check_nodes(_ops.to_host(plan.coords[0]), k)
    z = torch.zeros(T, dtype=torch.float64, device=plan.coords.device)
    tab = _ops.fornberg_dev(z, plan.coords, k)[:, k, :]          # [T, n]
    if plan.mode == nat.W_PERNODE:
        if T == 1:
            tab = tab.expand(sset.N, n)
        return _ops.CompactRows(sset, nat.W_PERNODE, pernode=tab.t().contiguous()[None])
    return _rows_from(plan, sset, tab[:, None, :].contiguous())


def assemble_global(grid: Grid, stencils, spec, delta_t: float,
                    frozen_nodes=()) -> BandedPropagator:
    """Banded linear propagator for one time step (harvest.py:162-178)."""
    sset = as_stencil_set(grid, stencils)
    rows = harvest_compact(grid, sset, spec, delta_t, 1, frozen_nodes)
    return BandedPropagator(periodic=grid.periodic, delta_t=delta_t, _rows=rows)


def assemble_global_phi(grid: Grid, stencils, spec, delta_t: float, s: int,
                        frozen_nodes=()) -> list[BandedPropagator]:
    """[exp, dt*phi_1, ..., dt^(s-1)*phi_(s-1)] banded operators (harvest.py:181-210)."""
    sset = as_stencil_set(grid, stencils)
    rows = harvest_compact(grid, sset, spec, delta_t, s, frozen_nodes)
    return [BandedPropagator(periodic=grid.periodic, delta_t=delta_t, _rows=rows.row(j))
            for j in range(s)]


def apply(prop: BandedPropagator, u):
    """out[i] = sum_j w[i, j] u[members[i, j]] (harvest.py:213-222), on the
    device in ascending order.  Complex vectors are applied part by part."""
    as_torch = isinstance(u, torch.Tensor)
    if as_torch and u.is_complex() or (not as_torch and np.iscomplexobj(u)):
        ur = u.real if as_torch else np.real(u)
        ui = u.imag if as_torch else np.imag(u)
        re, im = apply(prop, ur), apply(prop, ui)
        return torch.complex(re, im) if as_torch else re + 1j * im
    shape = tuple(u.shape)
    if shape != (prop.N,):
        raise DimensionMismatch(f"expected a vector of length {prop.N}, got shape {shape}")
    rows = prop.rows()
    ut = _ops.dev_f64(u)
    out = torch.empty_like(ut)
    import ctypes as C
    g = _ops.c_grid(rows.layout)
    w = rows.c_weights()
    st = nat.lib().lmep_banded_matvec(C.byref(g), C.byref(w), None, nat.ptr(ut), nat.ptr(out),
                                      nat.FLAG_EXACT, nat.stream_handle())
    nat.check(st, "lmep_banded_matvec")
    return out if as_torch else _ops.to_host(out)


def combine(props: list[BandedPropagator], coeffs) -> BandedPropagator:
    """sum_i coeffs[i] props[i] from zeros in list order (harvest.py:225-235)."""
    base = props[0]
    lay = base.layout
    for p in props[1:]:
        pl = p.layout
        if (pl.N, pl.n, pl.row, pl.periodic) != (lay.N, lay.n, lay.row, lay.periodic):
            raise DimensionMismatch("cannot combine operators with different stencils")
    rows = _ops.combine_rows([p.rows() for p in props], list(coeffs))
    return BandedPropagator(periodic=base.periodic, delta_t=base.delta_t, _rows=rows)


def weight_table_json(stencils, rows: list[PhiWeightSet]) -> str:
    """Weight table as JSON with 17 significant digits, one record per node
    (harvest.py:238-265); the text is the reference's byte for byte."""
    st = list(stencils)
    if len(st) != len(rows):
        raise DimensionMismatch("one weight set per stencil required")

    def num(x):
        return format(float(x), ".17g")

    def vec(v):
        return "[" + ", ".join(num(x) for x in v) + "]"

    recs = ['{"index": %d, "target_row": %d, "members": [%s], "w_lin": %s, "w_phi": [%s]}'
            % (int(s_.target), int(s_.target_row), ", ".join(str(int(m)) for m in s_.members),
               vec(r.w_lin), ", ".join(vec(v) for v in r.w_phi)) for s_, r in zip(st, rows)]
    head = '{"delta_t": %s, "N": %d, "n": %d, "s": %d, "nodes": [' % (
        num(rows[0].delta_t), len(st), st[0].n, len(rows[0].w_phi) + 1)
    return head + ", ".join(recs) + "]}"
