"""Time integration on the device (reference: localexp/timestep.py:38-394).

``run`` keeps the reference contract -- validation, harvest/step split
timers, snapshot chunks, NonFinite with the last finite snapshot -- and
runs every phase on the GPU: one batched harvest launch per operator set,
then the fused step kernels (linear / ETDRK4 / ETD2), which keep the
operator rows in compact form and never materialise (N, n) arrays.

Extensions beyond the reference API (each documented where it is used):
  * ``Boundary.neumann()``: zero-gradient closure with frozen boundary rows
    (BASELINE config 4);
  * ``SemiLinearProblem.nonlinear_scale``: N(u) = -scale * u * D1 u
    (KdV's 6 u u_x, BASELINE config 3);
  * ``VariableCoefficientSpec`` as ``problem.linear`` (config 5);
  * ``run(..., exact=..., tuning=...)``: arithmetic mode and launch shape.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable

import numpy as np
import torch

from . import _native as nat
from . import _ops
from .errors import DimensionMismatch, InvalidConfig, NonFinite, NotWarmedUp
from .grid import Grid, StencilSet, as_stencil_set
from .harvest import BandedPropagator, combine, derivative_compact, harvest_compact
from .localop import LinearOperatorSpec, VariableCoefficientSpec, fornberg_weights


@dataclass(frozen=True)
class Boundary:
    """Boundary handling (timestep.py:38-63) plus the "neumann" extension.

    dirichlet: u[0], u[-1] pinned after every stage and step; neumann: the
    end values are set from the zero one-sided first derivative at the same
    points.  With ``freeze_rows`` the two end nodes are held constant inside
    the local operators during harvesting.
    """

    kind: str  # "periodic" | "dirichlet" | "neumann"
    left: float = 0.0
    right: float = 0.0
    freeze_rows: bool = True

    @staticmethod
    def periodic() -> "Boundary":
        return Boundary(kind="periodic")

    @staticmethod
    def dirichlet(left: float, right: float, freeze_rows: bool = True) -> "Boundary":
        return Boundary(kind="dirichlet", left=left, right=right, freeze_rows=freeze_rows)

    @staticmethod
    def neumann(freeze_rows: bool = True) -> "Boundary":
        return Boundary(kind="neumann", freeze_rows=freeze_rows)

    @property
    def pinned(self) -> bool:
        return self.kind == "dirichlet"

    @property
    def closed(self) -> bool:
        return self.kind in ("dirichlet", "neumann")


@dataclass(frozen=True)
class SemiLinearProblem:
    """u_t = L u + N(u) (timestep.py:66-84)."""

    linear: object                       # LinearOperatorSpec | VariableCoefficientSpec
    nonlinear: Callable | None
    initial: np.ndarray
    boundary: Boundary
    nonlinear_kind: str = "callable"     # none | convective | cubic | callable
    nonlinear_scale: float = 1.0         # convective: N(u) = -scale * u * D1 u

    def __post_init__(self):
        u0 = self.initial
        if not isinstance(u0, torch.Tensor):
            u0 = np.ascontiguousarray(np.asarray(u0, dtype=np.float64))
            u0.setflags(write=False)
        object.__setattr__(self, "initial", u0)
        if self.nonlinear_kind not in ("none", "convective", "cubic", "callable"):
            raise InvalidConfig(f"unknown nonlinearity kind {self.nonlinear_kind!r}")
        if self.boundary.pinned:
            a, b = float(u0[0]), float(u0[-1])
            if abs(a - self.boundary.left) > 1e-12 or abs(b - self.boundary.right) > 1e-12:
                raise InvalidConfig("Dirichlet initial data must satisfy the pinned values")


@dataclass(frozen=True)
class StepperState:
    u: np.ndarray
    t: float
    history: tuple = ()


@dataclass(frozen=True)
class SchemeConfig:
    kind: str  # "linear" | "etdrk4" | "etd-multistep"
    s: int = 4

    def __post_init__(self):
        if self.kind not in ("linear", "etdrk4", "etd-multistep"):
            raise InvalidConfig(f"unknown scheme {self.kind!r}")
        if self.s < 1:
            raise InvalidConfig("scheme order must be >= 1")


@dataclass(frozen=True)
class SimulationResult:
    times: np.ndarray
    snapshots: np.ndarray
    steps: int
    harvest_ns: int
    step_ns: int

    @property
    def u_final(self) -> np.ndarray:
        return self.snapshots[-1]

    @property
    def t_final(self) -> float:
        return float(self.times[-1])


def _steps_for(span: float, delta_t: float, what: str) -> int:
    """timestep.py:240-244."""
    steps = int(round(span / delta_t))
    if steps < 0 or abs(steps * delta_t - span) > 1e-9 * max(abs(span), delta_t):
        raise InvalidConfig(f"dt={delta_t} does not divide the {what} {span}")
    return steps


_NL = {"none": nat.NL_NONE, "convective": nat.NL_CONVECTIVE, "cubic": nat.NL_CUBIC}


def _nl_kind(problem: SemiLinearProblem) -> int:
    k = problem.nonlinear_kind
    if k == "callable":
        if problem.nonlinear is not None:
            raise InvalidConfig("a Python callable nonlinearity has no device path; use the "
                                "structured kinds 'none', 'convective' or 'cubic'")
        return nat.NL_NONE
    return _NL[k]


def etdrk4_operators(ops_full: list[BandedPropagator], ops_half: list[BandedPropagator]):
    """alpha, beta, gamma precomposition (timestep.py:141-156)."""
    if len(ops_full) < 4:
        raise InvalidConfig("etdrk4 needs phi rows up to phi_3 at the full step")
    if len(ops_half) < 2:
        raise InvalidConfig("etdrk4 needs the phi_1 row at the half step")
    w, p1, p2, p3 = ops_full[:4]
    dt = w.delta_t
    alpha = combine([p1, p2, p3], [1.0, -3.0 / dt, 4.0 / dt**2])
    beta = combine([p2, p3], [2.0 / dt, -4.0 / dt**2])
    gamma = combine([p3, p2], [4.0 / dt**2, -1.0 / dt])
    return w, alpha, beta, gamma, ops_half[0], ops_half[1]


_ABG = ((nat.ROW_ALPHA, (1, 2, 3), lambda dt: (1.0, -3.0 / dt, 4.0 / dt**2)),
        (nat.ROW_BETA, (2, 3), lambda dt: (2.0 / dt, -4.0 / dt**2)),
        (nat.ROW_GAMMA, (3, 2), lambda dt: (4.0 / dt**2, -1.0 / dt)))


def _etdrk4_bank(full: _ops.CompactRows, half: _ops.CompactRows, dt: float,
                 d1: _ops.CompactRows | None) -> _ops.CompactRows:
    """The fused ETDRK4 bank [w, alpha, beta, gamma, w_half, p1_half(, d1)]:
    alpha / beta / gamma (timestep.py:141-156, combine's ordered sums,
    harvest.py:225-235) are composed by the library's combine kernel straight
    from the harvested phi rows into their slots of the bank."""
    p0 = full.row(0)
    if p0.mode == nat.W_PERNODE:
        zero = _ops.CompactRows(p0.layout, nat.W_PERNODE, pernode=torch.zeros_like(p0.pernode),
                                pernode_pad=p0.pernode_pad)
    else:
        zero = _ops.CompactRows(p0.layout, p0.mode, torch.zeros_like(p0.interior),
                                None if p0.classes is None else torch.zeros_like(p0.classes),
                                p0.nleft, p0.nright)
    parts = [p0, zero, zero, zero, half.row(0), half.row(1)] + ([d1] if d1 is not None else [])
    bank = _ops.stack_rows(parts)
    fb = full if bank.mode == nat.W_PERNODE else full.with_classes(bank.nleft, bank.nright)
    R = bank.R
    n = bank.n
    for slot, terms, cof in _ABG:
        c = cof(dt)
        if bank.mode == nat.W_PERNODE:
            blk = fb.pernode[0].numel()
            _ops.combine_into(bank.pernode[slot], [fb.pernode[t] for t in terms], c, 1, blk, blk,
                              [blk] * len(terms))
            continue
        _ops.combine_into(bank.interior[slot], [fb.interior[t] for t in terms], c, 1, n, n,
                          [n] * len(terms))
        if bank.classes is not None:
            Cn = bank.classes.shape[0]
            _ops.combine_into(bank.classes[:, slot], [fb.classes[:, t] for t in terms], c, Cn, n,
                              R * n, [fb.R * n] * len(terms))
    bank._host_interior = None
    return bank


def assemble_derivative(grid: Grid, stencils, k: int) -> BandedPropagator:
    """Banded k-th derivative operator, no dt factor (timestep.py:218-237)."""
    sset = as_stencil_set(grid, stencils)
    return BandedPropagator(periodic=grid.periodic, delta_t=0.0,
                            _rows=derivative_compact(grid, sset, k))


def _scaled(rows: _ops.CompactRows, c: float) -> _ops.CompactRows:
    if c == 1.0:
        return rows
    return _ops.combine_rows([rows], [c])


def _closure_rows(grid: Grid, n: int):
    """One-sided first-derivative rows at both ends."""
    N = grid.size
    if grid.uniform_spacing is not None:
        h = grid.uniform_spacing
        xl = np.arange(n) * h
        xr = (np.arange(n) - (n - 1)) * h
    else:
        xl = grid.nodes[:n] - grid.nodes[0]
        xr = grid.nodes[N - n:] - grid.nodes[N - 1]
    return fornberg_weights(0.0, xl, 1)[1], fornberg_weights(0.0, xr, 1)[1]


def _bc_for(grid: Grid, sset: StencilSet, boundary: Boundary) -> _ops.BC:
    if boundary.kind == "periodic":
        if not grid.periodic:
            raise InvalidConfig("periodic boundary on a non-periodic grid")
        return _ops.BC()
    if grid.periodic:
        raise InvalidConfig(f"{boundary.kind} boundary on a periodic grid")
    if boundary.kind == "dirichlet":
        return _ops.BC(nat.BC_DIRICHLET, boundary.left, boundary.right)
    dl, dr = _closure_rows(grid, sset.n)
    return _ops.BC(nat.BC_NEUMANN, dl=dl, dr=dr)


def close_initial(u: torch.Tensor, sset: StencilSet, bc: _ops.BC) -> torch.Tensor:
    """Apply the boundary closure to initial data (timestep.py:310-311) with the
    step kernel itself: one linear step with unit-vector rows copies u exactly
    and applies the closure at the ends."""
    if bc.kind == nat.BC_NONE:
        return u.clone()
    e = torch.zeros((1, sset.n), dtype=torch.float64, device=u.device)
    e[0, sset.row] = 1.0
    cl = _ops.CompactRows(sset, nat.W_CLASS if not sset.periodic else nat.W_SHARED, e, None, 0, 0)
    if not sset.periodic:
        # clamped windows near the ends: unit vector on the node itself
        nl, nr = sset.n_left, sset.n_right
        t = np.concatenate([np.arange(nl), [sset.N // 2], np.arange(sset.N - nr, sset.N)])
        rows = sset.target_rows(t)
        C = torch.zeros((t.size, 1, sset.n), dtype=torch.float64, device=u.device)
        C[torch.arange(t.size), 0, torch.as_tensor(rows, device=u.device)] = 1.0
        cl = _ops.CompactRows(sset, nat.W_CLASS, e, C, nl, nr)
    return _ops.step(nat.SCH_LIN, cl, u, 1, bc=bc, exact=True, tuning={"ksteps": 1})


@dataclass
class Prepared:
    """Harvested operator banks of one run (device resident)."""

    sset: StencilSet
    scheme: str
    nl: int
    bc: _ops.BC
    bank: _ops.CompactRows
    warm: _ops.CompactRows | None
    delta_t: float
    s: int


def prepare(grid: Grid, stencils, problem: SemiLinearProblem, scheme: SchemeConfig,
            delta_t: float, stats: dict | None = None) -> Prepared:
    """Harvest phase of ``run`` (timestep.py:284-308), on the device."""
    sset = as_stencil_set(grid, stencils)
    nl = _nl_kind(problem)
    bc = _bc_for(grid, sset, problem.boundary)
    frozen = (0, grid.size - 1) if problem.boundary.closed and problem.boundary.freeze_rows else ()
    d1 = None
    if nl == nat.NL_CONVECTIVE:
        d1 = _scaled(derivative_compact(grid, sset, 1), float(problem.nonlinear_scale))
    spec = problem.linear
    warm = None
    if scheme.kind == "linear":
        bank = harvest_compact(grid, sset, spec, delta_t, 1, frozen, stats)
    elif scheme.kind == "etdrk4":
        full, half = harvest_compact(grid, sset, spec, delta_t, 4, frozen, stats, half=True)
        bank = _etdrk4_bank(full, half, delta_t, d1)
    else:
        s = scheme.s
        if s > 5:
            raise InvalidConfig("etd-multistep supports s <= 5 (phi rows up to phi_5)")
        ops = harvest_compact(grid, sset, spec, delta_t, s + 1, frozen, stats)
        parts = {nat.ROW_W + j: ops.row(j) for j in range(s + 1)}
        if s >= 2:
            full, half = harvest_compact(grid, sset, spec, delta_t, 4, frozen, stats, half=True)
            warm = _etdrk4_bank(full, half, delta_t, d1)
        if d1 is not None:
            parts[nat.ROW_D1] = d1
        bank = _ops.rows_bank_for(sset, parts, max(parts) + 1)
    return Prepared(sset, scheme.kind, nl, bc, bank, warm, float(delta_t), scheme.s)


class Stepper:
    """Device state of a run: u (and the multistep history) plus the operator
    banks; ``advance(k)`` performs k steps without leaving the GPU."""

    def __init__(self, prep: Prepared, u0: torch.Tensor, exact: bool = True, tuning=None):
        self.p = prep
        self.exact = exact
        self.tuning = tuning
        self.u = close_initial(u0, prep.sset, prep.bc)
        self.hist = None
        self.done = 0
        self.flag = torch.zeros(1, dtype=torch.int32, device=u0.device)
        N = prep.sset.N
        self._out = torch.empty(N, dtype=torch.float64, device=u0.device)
        self._scr = torch.empty(max(prep.s, 2) * N, dtype=torch.float64, device=u0.device)
        self._hout = None

    @classmethod
    def resumed(cls, prep: Prepared, u: torch.Tensor, spare: torch.Tensor, scratch: torch.Tensor,
                flag: torch.Tensor, done: int, exact: bool = True, tuning=None) -> "Stepper":
        """A linear stepper whose first `done` steps already ran elsewhere (the
        streamed pipeline): u is the state after them, spare / scratch its buffers."""
        self = cls.__new__(cls)
        self.p, self.exact, self.tuning = prep, exact, tuning
        self.u, self._out, self._scr, self.flag = u, spare, scratch, flag
        self.hist, self._hout, self.done = None, None, done
        return self

    def advance(self, k: int, host_out: torch.Tensor | None = None,
                copy_stream: int | None = None) -> None:
        """k more steps.  host_out (linear scheme): a page-locked host vector that
        also receives the result through copy_stream (a raw stream handle), copied
        range by range behind the last launch (lmep_step_linear_host)."""
        p = self.p
        kw = dict(bc=p.bc, nl=p.nl, exact=self.exact, tuning=self.tuning, flag=self.flag,
                  scratch=self._scr)
        if k <= 0:
            return
        if p.scheme == "linear":
            out = _ops.step(nat.SCH_LIN, p.bank, self.u, k, out=self._out, host_out=host_out,
                            copy_stream=copy_stream, **kw)
            self._out, self.u = self.u, out
        elif p.scheme == "etdrk4":
            out = _ops.step(nat.SCH_ETDRK4, p.bank, self.u, k, out=self._out, **kw)
            self._out, self.u = self.u, out
        else:
            s = p.s
            if self.hist is None:
                self.hist = torch.zeros((max(s - 1, 1), self.u.numel()), dtype=torch.float64,
                                        device=self.u.device)
                self._hout = torch.empty_like(self.hist)
                self._warm = 0
            # warm-up: s-1 ETDRK4 steps, each storing N(u) in front of the
            # history (timestep.py:375-378); may straddle advance() calls.  The
            # history is newest first, so warm-up step i's N(u_i) lands in slot
            # s-2-i directly (no shifting of the older entries)
            while self._warm < s - 1 and k > 0:
                i = self._warm
                out = _ops.step(nat.SCH_ETDRK4, p.warm, self.u, 1, out=self._out,
                                nl0_out=self.hist[s - 2 - i], **kw)
                self._out, self.u = self.u, out
                self._warm += 1
                self.done += 1
                k -= 1
            if k == 0:
                return
            u, q = _ops.step(nat.SCH_ETD2, p.bank, self.u, k, hist=self.hist,
                             delta_t=p.delta_t, out=self._out, hist_out=self._hout,
                             etd_order=s, **kw)
            self._out, self.u = self.u, u
            if s > 1:
                self._hout, self.hist = self.hist, q
        self.done += k

    def nonfinite(self) -> bool:
        return bool(self.flag.item())


def run(grid: Grid, stencils, problem: SemiLinearProblem, scheme: SchemeConfig,
        delta_t: float, t_final: float, snapshot_stride: float | None = None, *,
        exact: bool = True, tuning=None, stats: dict | None = None,
        stream: bool = True) -> SimulationResult:
    """Integrate to t_final with snapshots (timestep.py:255-394), on the GPU.
    stream=True: a linear run from host coefficients and host initial data on a
    periodic grid runs upload, harvest, the first chunk of steps and the
    snapshot download as one pipeline (csrc/step_stream.cu), bit-identical to
    the phase-by-phase order on the same rows."""
    if t_final <= 0:
        raise InvalidConfig("t_final must be positive")
    if delta_t <= 0:
        raise InvalidConfig("dt must be positive")
    steps_total = _steps_for(t_final, delta_t, "final time")
    if snapshot_stride is None:
        snap_every = steps_total
    else:
        snap_every = _steps_for(snapshot_stride, delta_t, "snapshot stride")
        if snap_every == 0:
            raise InvalidConfig("snapshot stride must be at least one step")
    dev = nat.device()
    u0 = problem.initial
    if tuple(u0.shape) != (grid.size,):
        raise DimensionMismatch(f"initial data must have shape ({grid.size},)")
    N = grid.size
    cur = torch.cuda.current_stream(dev)
    cp, cp1 = _ops.copy_stream(0), _ops.copy_stream(1)

    torch.cuda.synchronize(dev)
    # harvest_ns / step_ns are device intervals between CUDA events on the compute
    # stream, so the host never waits between the harvest and the steps: it
    # enqueues the steps while the coefficients stream up and the harvest runs
    ev_start = torch.cuda.Event(enable_timing=True)
    ev_start.record(cur)
    # The initial data goes up while the harvest runs.  When the harvest
    # streams host coefficients (copy stream 0), u0 is queued behind them so
    # the slices the harvest waits on get the PCIe bandwidth first; otherwise
    # it goes up at once on its own copy stream.
    lin = problem.linear
    deferred = None
    ls = None
    nsnap = 1 + (-(-steps_total // snap_every) if snap_every else 0)
    # snapshots land straight in one page-locked [S, N] block (returned as is)
    snaps = torch.empty((nsnap, N), dtype=torch.float64, pin_memory=True)
    k_first = min(snap_every, steps_total)
    host_in = isinstance(lin, VariableCoefficientSpec) and _ops.is_host(lin.coef) and _ops.is_host(u0)
    if host_in and stream and scheme.kind == "linear" and grid.periodic and k_first >= 1 and \
            problem.boundary.kind == "periodic":
        # one pipeline: upload || harvest || steps || download, slice by slice
        # (_ops.LinearStream); the initial state rides up with the coefficients
        ls = _ops.LinearStream(_ops.host_f64(u0), k_first, exact, tuning, snaps[0], snaps[1], cp1,
                               coef_host=_ops.host_f64(lin.coef) if lin.reaction is None else None)
        _ops.set_stream_consumer(ls)
    elif host_in:
        src = _ops.host_f64(u0)
        deferred = _ops.DeferredUpload(src, torch.empty(N, dtype=torch.float64, device=dev))
        _ops.defer_upload(deferred)
    else:
        with torch.cuda.stream(cp1):
            u0d = _ops.dev_f64(u0)
        ev_u0 = cp1.record_event()
    try:
        # the harvest's status is checked once it has finished (below), so the
        # host runs ahead and prepares the stepping while the device harvests
        with _ops.deferred_status_checks() as pending:
            prep = prepare(grid, stencils, problem, scheme, delta_t, stats)
    except BaseException:
        if ls is not None:
            ls.active = False
            ls.close()
        raise
    finally:
        _ops.take_stream_consumer()
        if deferred is not None:
            _ops.drop_deferred(deferred)
    if deferred is not None:
        if deferred.event is None:           # the harvest did not pipeline: upload now
            deferred.issue(cp1)
        u0d, ev_u0 = deferred.dst, deferred.event
    if ls is not None:
        if not ls.began:                     # the harvest did not pipeline: upload now
            cp.wait_stream(cur)
            with torch.cuda.stream(cp):
                ls.upload(0, N)
            ls.uploaded(cp)
        u0d, ev_u0 = ls.u0, ls.last_landed
    ev_harvest = torch.cuda.Event(enable_timing=True)
    ev_harvest.record(cur)
    harvest_ns = None
    times = [0.0]
    step_ns = 0
    done = 0

    if ls is not None and ls.active:
        # the first chunk's steps were queued slice by slice behind the harvest and
        # both snapshots are on their way down (copy stream 1)
        ls.close()
        st = Stepper.resumed(prep, ls.out, ls.u0, ls.scr, ls.flag, k_first, exact=exact, tuning=tuning)
        cp1.wait_event(ls.snap0_event)
        snap_ev = prev_ev = cp1.record_event()
        cur.synchronize()
        t_prev, harvest_ms, step_ms = ev_start, 0.0, 0.0
        for eh, es in ls.marks:
            harvest_ms += t_prev.elapsed_time(eh)
            step_ms += eh.elapsed_time(es)
            t_prev = es
        harvest_ns, step_ns = int(harvest_ms * 1e6), int(step_ms * 1e6)
        _ops.check_deferred(pending)
        done = k_first
        if st.nonfinite():
            cp1.synchronize()
            raise NonFinite("time integration blew up", state=snaps[0].numpy().copy(), time=0.0)
        times.append(done * delta_t)
    else:
        cur.wait_event(ev_u0)
        u0d.record_stream(cur)
        st = Stepper(prep, u0d, exact=exact, tuning=tuning)
        snap_ev = None

    def snapshot(i):
        # D2H on the copy stream, overlapping the next chunk of steps; the
        # next advance() waits for it before it may reuse st.u's buffer
        cp.wait_stream(cur)
        with torch.cuda.stream(cp):
            snaps[i].copy_(st.u, non_blocking=True)
        st.u.record_stream(cp)
        return cp.record_event()

    if done == 0 and ls is not None and ls.began:
        snap_ev, prev_ev = ls.snap0_event, None          # snapshot 0 is already on its way down
    elif done == 0:
        snap_ev, prev_ev = snapshot(0), None
    ev_a, ev_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    while done < steps_total:
        k = min(snap_every, steps_total - done)
        ev_a.record(cur)
        # a linear / ETDRK4 advance() reads st.u and writes the other buffers:
        # it may overwrite the buffer the PREVIOUS snapshot was read from, never
        # the latest.  Multistep warm-up swaps buffers between single steps.
        wait = prev_ev if prep.scheme in ("linear", "etdrk4") else snap_ev
        if wait is not None:
            cur.wait_event(wait)
        if prep.scheme == "linear":
            # the library copies the snapshot itself, range by range behind the last
            # launch (its tail overlaps the copy), straight into the page-locked row
            st.advance(k, host_out=snaps[len(times)], copy_stream=cp.cuda_stream)
            ev_b.record(cur)
            st.u.record_stream(cp)
            new_ev = cp.record_event()
        else:
            st.advance(k)
            ev_b.record(cur)
            # the snapshot's D2H is queued behind the steps at once (its row of snaps
            # is only reported when the checks below pass), so the copy starts the
            # moment the last launch ends instead of after the host has read the flags
            new_ev = snapshot(len(times))
        cur.synchronize()
        if harvest_ns is None:
            # the harvest's status first: a failed exponential surfaces as the
            # harvest's NonFinite (timestep.py:284-308), not as a blown-up step
            harvest_ns = int(ev_start.elapsed_time(ev_harvest) * 1e6)
            _ops.check_deferred(pending)
        step_ns += int(ev_a.elapsed_time(ev_b) * 1e6)
        done += k
        if st.nonfinite():
            cp.synchronize()
            raise NonFinite("time integration blew up", state=snaps[len(times) - 1].numpy().copy(),
                            time=times[-1])
        times.append(done * delta_t)
        prev_ev, snap_ev = snap_ev, new_ev
    if harvest_ns is None:
        # zero steps (t_final below the dt rounding tolerance, _steps_for): the
        # harvest still ran and its status and time are reported (timestep.py:284)
        cur.synchronize()
        harvest_ns = int(ev_start.elapsed_time(ev_harvest) * 1e6)
        _ops.check_deferred(pending)
    cp.synchronize()
    if ls is not None:
        cp1.synchronize()
        ls.snap0_event.synchronize()
    return SimulationResult(times=np.array(times), snapshots=snaps.numpy(), steps=steps_total,
                            harvest_ns=harvest_ns, step_ns=step_ns)


# ---------------------------------------------------------------------------
# single-step API (timestep.py:136-215) for structured nonlinearities
# ---------------------------------------------------------------------------
def step_linear(prop: BandedPropagator, state: StepperState) -> StepperState:
    """u <- P u, t <- t + dt (timestep.py:136-138)."""
    from .harvest import apply
    return StepperState(u=apply(prop, state.u), t=state.t + prop.delta_t, history=state.history)


def etdrk4_step(ops_full, ops_half, problem: SemiLinearProblem, state: StepperState, *,
                d1: BandedPropagator | None = None, exact: bool = True) -> StepperState:
    """One ETDRK4 step (timestep.py:159-184) through the fused kernel."""
    w, al, be, ga, wh, p1h = etdrk4_operators(ops_full, ops_half)
    nl = _nl_kind(problem)
    parts = [x.rows() for x in (w, al, be, ga, wh, p1h)]
    if nl == nat.NL_CONVECTIVE:
        if d1 is None:
            raise InvalidConfig("convective nonlinearity needs the banded D1 operator (d1=)")
        parts.append(_scaled(d1.rows(), float(problem.nonlinear_scale)))
    bank = _ops.stack_rows(parts)
    bc = _ops.BC()
    if problem.boundary.pinned:
        bc = _ops.BC(nat.BC_DIRICHLET, problem.boundary.left, problem.boundary.right)
    flag = torch.zeros(1, dtype=torch.int32, device=nat.device())
    out = _ops.step(nat.SCH_ETDRK4, bank, _ops.dev_f64(state.u), 1, bc=bc, nl=nl, exact=exact,
                    flag=flag)
    if flag.item():
        raise NonFinite("etdrk4 step produced non-finite values", state=state.u, time=state.t)
    u = out if isinstance(state.u, torch.Tensor) else _ops.to_host(out)
    return StepperState(u=u, t=state.t + w.delta_t, history=state.history)


def etd_multistep_step(ops, problem: SemiLinearProblem, state: StepperState, s: int, *,
                       d1: BandedPropagator | None = None, exact: bool = True) -> StepperState:
    """One exponential multistep update of order s <= 5 (timestep.py:187-215)."""
    if len(ops) < s + 1:
        raise InvalidConfig(f"order {s} needs phi rows up to phi_{s}")
    if len(state.history) < s - 1:
        raise NotWarmedUp(f"order {s} needs {s - 1} stored evaluations, have {len(state.history)}")
    if s > 5:
        raise InvalidConfig("etd-multistep supports s <= 5")
    nl = _nl_kind(problem)
    slots = {nat.ROW_W + j: ops[j].rows() for j in range(s + 1)}
    if nl == nat.NL_CONVECTIVE:
        if d1 is None:
            raise InvalidConfig("convective nonlinearity needs the banded D1 operator (d1=)")
        slots[nat.ROW_D1] = _scaled(d1.rows(), float(problem.nonlinear_scale))
    lay = slots[nat.ROW_W].layout
    bank = _ops.rows_bank_for(lay, slots, max(slots) + 1)
    bc = _ops.BC()
    if problem.boundary.pinned:
        bc = _ops.BC(nat.BC_DIRICHLET, problem.boundary.left, problem.boundary.right)
    u = _ops.dev_f64(state.u)
    hist = torch.stack([_ops.dev_f64(h) for h in state.history[:s - 1]]) if s > 1 else None
    flag = torch.zeros(1, dtype=torch.int32, device=u.device)
    un, q = _ops.step(nat.SCH_ETD2, bank, u, 1, bc=bc, nl=nl, exact=exact, hist=hist,
                      delta_t=ops[0].delta_t, flag=flag, etd_order=s)
    if flag.item():
        raise NonFinite("multistep update produced non-finite values", state=state.u, time=state.t)
    conv = (lambda x: x) if isinstance(state.u, torch.Tensor) else _ops.to_host
    nk = q[0] if s > 1 else _nl_eval_device(u, d1, problem, nl)
    history = (conv(nk),) + tuple(state.history[:max(s - 2, 0)])
    return StepperState(u=conv(un), t=state.t + ops[0].delta_t, history=history)


def _nl_eval_device(u: torch.Tensor, d1: BandedPropagator | None, problem: SemiLinearProblem,
                    nl: int) -> torch.Tensor:
    """N(u) at the step start (the history entry), computed by the step kernel:
    one 0-step-ahead ETDRK4 launch would advance u, so evaluate through apply."""
    if nl == nat.NL_NONE:
        return torch.zeros_like(u)
    if nl == nat.NL_CUBIC:
        return -u * u * u
    from .harvest import apply
    du = apply(BandedPropagator(periodic=d1.periodic, delta_t=0.0,
                                _rows=_scaled(d1.rows(), float(problem.nonlinear_scale))), u)
    return -u * du


__all__ = ["Boundary", "SemiLinearProblem", "StepperState", "SchemeConfig", "SimulationResult",
           "etdrk4_operators", "etdrk4_step", "etd_multistep_step", "assemble_derivative",
           "step_linear", "run", "prepare", "Stepper", "LinearOperatorSpec", "math"]
