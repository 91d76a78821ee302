"""Device-side building blocks shared by the public modules.

Everything here drives liblmep.so on CUDA tensors; torch is used only for
allocation, streams and tiny elementwise glue (e.g. the ordered linear
combination of harvested rows that ``harvest.combine`` defines).
"""

from __future__ import annotations

from contextlib import contextmanager

import ctypes as C
import threading
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from .errors import DimensionMismatch, DuplicateNodes, InvalidConfig, OrderTooHigh
from .grid import StencilSet

F64 = torch.float64


def dev_f64(a) -> torch.Tensor:
    """Contiguous float64 tensor on the product device.  Host data is copied
    once (asynchronously from pinned torch tensors); read-only numpy arrays
    are wrapped without a host-side copy (the wrapper is never written)."""
    d = nat.device()
    if isinstance(a, torch.Tensor):
        if a.device.type == "cpu":
            a = a.to(dtype=F64).contiguous()
            return a.to(device=d, non_blocking=a.is_pinned())
        return a.to(device=d, dtype=F64).contiguous()
    h = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)     # read-only source, copied to device
        t = torch.from_numpy(h)
    return t.to(device=d)


def dev_i32(a) -> torch.Tensor:
    return torch.as_tensor(np.ascontiguousarray(np.asarray(a, dtype=np.int32)), device=nat.device())


_COPY_STREAMS: dict = {}


def copy_stream(which: int = 0) -> torch.cuda.Stream:
    """Side streams host<->device transfers overlap on (per device): 0 carries
    harvest inputs and snapshots, 1 the initial state; 2 is the side stream a
    streamed run's harvests are queued on, 3 the one its snapshot 0 goes down on."""
    d = nat.device()
    key = (d.index if d.index is not None else torch.cuda.current_device(), which)
    if key not in _COPY_STREAMS:
        # stream 2 (harvests beside a streamed run's step launches) has priority: its
        # CTAs go first whenever a persistent step kernel hands SMs back
        _COPY_STREAMS[key] = torch.cuda.Stream(device=d, priority=-1 if which == 2 else 0)
    return _COPY_STREAMS[key]


class DeferredUpload:
    """A host->device copy that a pipelined harvest queues on copy stream 0
    right after its coefficient slices (timestep.run's initial state): both
    directions of PCIe then serve the harvest inputs first.  ``event`` is set
    once the copy is queued."""

    def __init__(self, src: torch.Tensor, dst: torch.Tensor):
        self.src, self.dst, self.event = src, dst, None

    def issue(self, stream: torch.cuda.Stream) -> None:
        with torch.cuda.stream(stream):
            self.dst.copy_(self.src, non_blocking=self.src.is_pinned())
        self.event = stream.record_event()


# per host thread: uploads waiting for a pipelined harvest, and the harvest
# status checks a pipeline defers to its own sync point
_TLS = threading.local()


def _deferred() -> list:
    if not hasattr(_TLS, "deferred"):
        _TLS.deferred = []
    return _TLS.deferred


def defer_upload(up: DeferredUpload) -> None:
    _deferred().append(up)


def issue_deferred(stream: torch.cuda.Stream) -> None:
    q = _deferred()
    while q:
        q.pop(0).issue(stream)


def drop_deferred(up: DeferredUpload) -> None:
    q = _deferred()
    if up in q:
        q.remove(up)


_EVENT_POOL: dict = {}


def stream_wait(stream: torch.cuda.Stream, ev) -> None:
    """stream waits for ev: a torch event or a raw one (lmep_event_create)."""
    if isinstance(ev, torch.cuda.Event):
        stream.wait_event(ev)
    else:
        nat.check(nat.lib().lmep_stream_wait_event(stream.cuda_stream, ev), "lmep_stream_wait_event")


class LinearStream:
    """Consumer of a pipelined per-node harvest: timestep.run's linear scheme
    from host arrays as one pipeline (lmep_lin_stream, csrc/step_stream.cu).
    The harvest pipeline (harvest._harvest_pipelined) calls, in order,
    ``begin`` (the row table exists, nothing harvested yet: the library plans
    the launch levels and this object sizes the slices), ``upload`` per slice on
    the upload stream (the slice of the initial state rides with its
    coefficients), ``ready`` after each slice's harvest is queued (every k-step launch
    whose inputs are complete is queued behind it; the last slice finishes the
    ring), and ``uploaded`` once every slice is queued (snapshot 0 goes back
    down).  The result and its host copy (``host_out``) are bit-identical to
    Stepper.advance on the same rows.  When the library declines the plan
    (LMEP_INVALID_CONFIG: not the persistent per-node kernels' case) the object
    only uploads the initial state and the caller steps afterwards."""

    # slices in waves of (SM count) level-1 tiles: a small first slice (its upload
    # is the only exposed one), wide middle slices (few launches), a small last
    # slice (its download is the only exposed one)
    WAVES = (1.0, 3.0, 6.0, 6.0, 4.0)
    LAST_MIN = 2.0
    # prefixes (nodes) of the coefficient table and the initial state that go up
    # from the constructor, before the harvest is planned: PCIe works while the
    # host plans (the first covers the first slice, multiples of 1024)
    EAGER = (192 * 1024, 1024 * 1024)

    def __init__(self, u0_host: torch.Tensor, steps: int, exact: bool, tuning, snap0: torch.Tensor,
                 host_out: torch.Tensor, down: torch.cuda.Stream, coef_host: torch.Tensor | None = None):
        d = nat.device()
        self.N = int(u0_host.numel())
        self.src = u0_host
        self.u0 = torch.empty(self.N, dtype=F64, device=d)
        self.snap0, self.host_out, self.down = snap0, host_out, down
        # eager prefixes: [(end, event)] in rising order; coef_dev is the device
        # table the pipelined harvest then fills (harvest._harvest_pipelined)
        self.coef_src, self.coef_dev, self.eager = coef_host, None, []
        self._snapped = 0
        self._nev = 0
        # snapshot 0 goes down on its own stream: on the result's stream its slices
        # (queued with the uploads, up front) would sit in front of every result copy
        self.snap_stream = copy_stream(3)
        if coef_host is not None and coef_host.dim() == 2 and coef_host.shape[0] == self.N and self.EAGER:
            self.coef_dev = torch.empty(tuple(coef_host.shape), dtype=F64, device=d)
            up = copy_stream()
            up.wait_stream(torch.cuda.current_stream(d))
            a = 0
            for e in self.EAGER:
                b = min(self.N, int(e))
                if b <= a:
                    break
                self.eager.append((b, self.send(self.coef_dev, coef_host, a, b, up)))
                a = b
        self.out = torch.empty(self.N, dtype=F64, device=d)
        self.scr = torch.empty(self.N, dtype=F64, device=d)
        self.flag = torch.zeros(1, dtype=torch.int32, device=d)
        self.steps, self.exact, self.tuning = int(steps), bool(exact), tuning
        self.snap0, self.host_out, self.down = snap0, host_out, down
        self.handle = None
        self.active = False
        self.began = False
        self.last_landed = None
        self.snap0_event = None
        self.marks = []                      # (harvest queued, steps queued) events per slice
        self.launches = 0
        self.bounds = None

    def begin(self, layout: StencilSet, rows: torch.Tensor, default_bounds):
        self.began = True
        self.rows = rows
        if rows.shape[0] != 1 or rows.shape[2] != self.N or self.steps < 1:
            return default_bounds
        g = c_grid(layout, 0, None)
        w = nat.LmepWeights(nat.W_PERNODE, 1, 0, 0, None, None, rows.data_ptr(), 0)
        tun = _tuning(self.tuning)
        h = C.c_void_p()
        L = nat.lib()
        st = L.lmep_lin_stream_begin(C.byref(g), C.byref(w), self.u0.data_ptr(), self.out.data_ptr(),
                                     self.scr.data_ptr(), self.steps, nat.FLAG_EXACT if self.exact else 0,
                                     C.byref(tun) if tun is not None else None, self.flag.data_ptr(),
                                     self.host_out.data_ptr(), self.down.cuda_stream,
                                     nat.stream_handle(), C.byref(h))
        if st == nat.LMEP_INVALID_CONFIG:
            return default_bounds
        nat.check(st, "lmep_lin_stream_begin")
        self.handle, self.active = h, True
        tile, margin, lev, sms = C.c_int64(), C.c_int64(), C.c_int32(), C.c_int32()
        nat.check(L.lmep_lin_stream_info(h, C.byref(tile), C.byref(margin), C.byref(lev), C.byref(sms)),
                  "lmep_lin_stream_info")
        self.bounds = self.slice_bounds(self.N, tile.value, margin.value, sms.value)
        return self.bounds

    @classmethod
    def slice_bounds(cls, N: int, tile: int, margin: int, sms: int):
        """Prefix ends (multiples of 1024 nodes, the harvest's superblock) that give
        every launch level whole waves of tiles: margin + c * sms * tile."""
        wave = sms * tile
        out, a, c = [], 0, 0.0
        for wv in cls.WAVES:
            c += wv
            b = -(-int(margin + c * wave) // 1024) * 1024
            if b + cls.LAST_MIN * wave >= N:
                break
            out.append((a, b))
            a = b
        out.append((a, N))
        return out

    def upload(self, a: int, b: int) -> None:
        """(on the upload stream) the slice of the initial state."""
        self.u0[a:b].copy_(self.src[a:b], non_blocking=True)

    def eager_end(self) -> int:
        return self.eager[-1][0] if self.eager else 0

    def eager_event(self, b: int):
        """The events (coefficients, coefficients + initial state) behind which nodes
        [0, b) have landed, if an eager prefix covers them."""
        for end, ev in self.eager:
            if b <= end:
                return ev
        return None

    def send(self, coef_dev: torch.Tensor, coef_host: torch.Tensor, a: int, b: int,
             up: torch.cuda.Stream):
        """Queue nodes [a, b) on the link in one library call (lmep_upload_slice):
        their coefficients and their part of the initial state go up on `up`, that
        part of snapshot 0 (timestep.py:313) goes back down at once on the snapshot
        stream while the uploads keep the other direction busy (behind all the
        uploads it would hold the result's download up at the end).  Returns the
        raw events (coefficients landed, everything landed)."""
        ec, ev = self._event(), self._event()
        cb = coef_host.stride(0) * 8
        nat.check(nat.lib().lmep_upload_slice(
            coef_dev.data_ptr() + a * cb, coef_host.data_ptr() + a * cb, (b - a) * cb,
            self.u0.data_ptr() + 8 * a, self.src.data_ptr() + 8 * a, self.snap0.data_ptr() + 8 * a,
            8 * (b - a), up.cuda_stream, self.snap_stream.cuda_stream, ec, ev), "lmep_upload_slice")
        self._snapped += b - a
        return ec, ev

    def _event(self):
        """A raw event of the per-device pool (re-recorded run after run: a run ends
        synchronised, and a wait keeps the state it was queued behind)."""
        pool = _EVENT_POOL.setdefault(self.u0.device.index, [])
        if self._nev == len(pool):
            h = C.c_void_p()
            nat.check(nat.lib().lmep_event_create(C.byref(h)), "lmep_event_create")
            pool.append(h)
        self._nev += 1
        return pool[self._nev - 1]

    def uploaded(self, up: torch.cuda.Stream) -> None:
        """Every slice is queued on the upload stream `up`; snapshot 0 is complete
        behind snap0_event."""
        self.last_landed = up.record_event()
        if self._snapped != self.N:                      # (not sent slice by slice)
            self.snap_stream.wait_event(self.last_landed)
            with torch.cuda.stream(self.snap_stream):
                self.snap0.copy_(self.u0, non_blocking=True)
        self.snap0_event = self.snap_stream.record_event()

    def ready(self, b: int) -> None:
        """The harvest of nodes [0, b) is queued on the current stream."""
        if not self.active:
            return
        cur = torch.cuda.current_stream()
        eh = torch.cuda.Event(enable_timing=True)
        es = torch.cuda.Event(enable_timing=True)
        eh.record(cur)
        nat.check(nat.lib().lmep_lin_stream_advance(self.handle, int(b), cur.cuda_stream),
                  "lmep_lin_stream_advance")
        es.record(cur)
        self.marks.append((eh, es))

    def close(self) -> None:
        if self.handle is not None:
            n = C.c_int64()
            st = nat.lib().lmep_lin_stream_end(self.handle, C.byref(n))
            self.handle = None
            self.launches = n.value
            if self.active:
                nat.check(st, "lmep_lin_stream_end")


def set_stream_consumer(ls) -> None:
    _TLS.stream = ls


def take_stream_consumer():
    ls = getattr(_TLS, "stream", None)
    _TLS.stream = None
    return ls


def is_host(a) -> bool:
    """True for data that lives in host memory (numpy / CPU tensors)."""
    return not (isinstance(a, torch.Tensor) and a.device.type == "cuda")


def host_f64(a) -> torch.Tensor:
    """Contiguous float64 CPU tensor view of host data (no copy when possible;
    pinned tensors stay pinned)."""
    if isinstance(a, torch.Tensor):
        return a.to(dtype=F64).contiguous()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64)))


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def to_host_pinned(t: torch.Tensor) -> np.ndarray:
    """D2H through a page-locked buffer (torch caches pinned blocks), then a numpy view."""
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return h.numpy()


# ---------------------------------------------------------------------------
# node-set validation (localop.py:69-74) -- host checks on n <= 32 numbers
# ---------------------------------------------------------------------------
def check_nodes(x: np.ndarray, max_order: int) -> None:
    n = x.size
    if not 0 <= max_order <= n - 1:
        raise OrderTooHigh(f"derivative order {max_order} needs > {max_order} nodes, got {n}")
    if n > nat.MAX_N:
        raise DimensionMismatch(f"stencils larger than {nat.MAX_N} nodes are not supported")
    if n > 1:
        spread = float(x.max() - x.min())
        if np.min(np.diff(np.sort(x))) <= 1e-14 * spread:
            raise DuplicateNodes("two stencil nodes coincide within 1e-14 of the spread")


def fornberg_dev(z: torch.Tensor, x: torch.Tensor, m: int) -> torch.Tensor:
    """Batched Fornberg tables on the device: z [B], x [B, n] -> [B, m+1, n]."""
    B, n = x.shape
    out = torch.empty((B, m + 1, n), dtype=F64, device=x.device)
    st = nat.lib().lmep_fornberg(nat.ptr(z), nat.ptr(x), n, n, m, B, nat.ptr(out),
                                 nat.stream_handle())
    nat.check(st, "lmep_fornberg")
    return out


def derivative_tables(coords: torch.Tensor, kmax: int) -> torch.Tensor:
    """D^(k) matrices on each coordinate set: coords [T, n] -> [T, n(i), kmax+1, n(j)]
    with row i evaluated at z = coords[t, i] (localop.diff_matrix, localop.py:99-108)."""
    T, n = coords.shape
    x = coords.repeat_interleave(n, dim=0).contiguous()        # item t*n+i uses coords[t]
    z = coords.reshape(-1).contiguous()
    return fornberg_dev(z, x, kmax).reshape(T, n, kmax + 1, n)


def operator_tables(coords: torch.Tensor, terms) -> tuple[torch.Tensor, list, float]:
    """Tables [T, nterms, n, n] of the spec's k>0 terms (in term order), their
    coefficients and the reaction coefficient (localop.py:111-128)."""
    kmax = max(k for k, _ in terms)
    pos = [(k, c) for k, c in terms if k > 0]
    c0 = 0.0
    for k, c in terms:
        if k == 0:
            c0 = float(c)
            break
    T, n = coords.shape
    if kmax == 0 or not pos:
        return torch.zeros((T, 0, n, n), dtype=F64, device=coords.device), [], c0
    tab = derivative_tables(coords, kmax)                       # [T, i, k, j]
    sel = torch.stack([tab[:, :, k, :] for k, _ in pos], dim=1)  # [T, t, i, j]
    return sel.contiguous(), [float(c) for _, c in pos], c0


# ---------------------------------------------------------------------------
# harvest (K1)
# ---------------------------------------------------------------------------
@dataclass
class HarvestOut:
    rows: torch.Tensor           # layout 0: [B, s, n]; layout 1: [s, n, B]
    ms: torch.Tensor             # [B] int32: pade degree | squarings << 8
    status: torch.Tensor         # [B] int32
    flag: torch.Tensor | None = None   # [1] int32, set by the library if any status failed
    half: torch.Tensor | None = None   # (w_lin, dt/2 phi_1) at delta_t / 2: [B, 2, n] / [2, n, B]


def harvest(n: int, s: int, delta_t: float, B: int, *, tables=None, table_idx=None, coef=None,
            coef_stride=0, c0=None, c0_stride=0, L=None, rows=None, row_default=0,
            frozen=None, frozen_default=0, layout=0, coef_map=None,
            into: HarvestOut | None = None, item0: int = 0, half: bool = False) -> HarvestOut:
    """One lmep_harvest_ex call.  coef_map = (node0, nnodes, periodic): row-scaled
    coefficients; coef / c0 then index the whole grid.  into / item0 (layout 1):
    write items [item0, item0 + B) of a larger HarvestOut; coef / c0 / rows /
    frozen are then the slice's own (already offset) arrays.  half: also the
    half-step set (s >= 2).  The per-item status is reduced on the device into
    HarvestOut.flag (no host synchronisation)."""
    d = nat.device()
    if into is None:
        out = torch.empty((B, s, n) if layout == 0 else (s, n, B), dtype=F64, device=d)
        ms = torch.empty(B, dtype=torch.int32, device=d)
        status = torch.empty(B, dtype=torch.int32, device=d)
        flag = torch.zeros(1, dtype=torch.int32, device=d)
        hv = None
        if half:
            hv = torch.empty((B, 2, n) if layout == 0 else (2, n, B), dtype=F64, device=d)
        res, ld, optr = HarvestOut(out, ms, status, flag, hv), B, nat.ptr(out)
        hptr = nat.ptr(hv)
    else:
        if layout != 1:
            raise InvalidConfig("chunked harvests write the SoA layout")
        res, ld = into, int(into.rows.shape[2])
        optr = into.rows.data_ptr() + 8 * int(item0)
        ms, status = into.ms[item0:item0 + B], into.status[item0:item0 + B]
        if into.flag is None:
            into.flag = torch.zeros(1, dtype=torch.int32, device=d)
        flag = into.flag
        hptr = None
        if half:
            if into.half is None:
                raise InvalidConfig("the target HarvestOut holds no half-step rows")
            hptr = into.half.data_ptr() + 8 * int(item0)
    a = nat.LmepHarvestArgs()
    a.n, a.s, a.layout = int(n), int(s), int(layout)
    a.nterms = 0 if tables is None else int(tables.shape[1])
    a.tables, a.table_idx, a.coef = nat.ptr(tables), nat.ptr(table_idx), nat.ptr(coef)
    a.coef_stride, a.c0, a.c0_stride = int(coef_stride), nat.ptr(c0), int(c0_stride)
    a.L, a.delta_t = nat.ptr(L), float(delta_t)
    a.target_row, a.row_default = nat.ptr(rows), int(row_default)
    a.frozen, a.frozen_default = nat.ptr(frozen), int(frozen_default)
    a.B, a.out_ld, a.w_out = int(B), int(ld), optr
    a.status, a.ms, a.half_out, a.status_any = nat.ptr(status), nat.ptr(ms), hptr, nat.ptr(flag)
    m = None
    if coef_map is not None:
        m = nat.LmepCoefMap(int(coef_map[0]), int(coef_map[1]), int(bool(coef_map[2])), 0)
        a.map = C.addressof(m)
    st = nat.lib().lmep_harvest_ex(C.byref(a), nat.stream_handle())
    nat.check(st, "lmep_harvest")
    return res


@contextmanager
def deferred_status_checks():
    """Within the block (this host thread), harvests queue their status flag
    instead of synchronising on it; the caller runs check_deferred(list) at its
    own sync point (a pipeline that enqueues harvest + steps back to back)."""
    prev = getattr(_TLS, "pending", None)
    _TLS.pending = []
    try:
        yield _TLS.pending
    finally:
        _TLS.pending = prev


def check_deferred(pending: list) -> None:
    for flag, what in pending:
        if int(flag.item()) != 0:
            pending.clear()
            nat.check(nat.LMEP_NONFINITE, what)
    pending.clear()


def raise_on_status(h: HarvestOut, what="matrix exponential overflowed") -> None:
    """NonFinite if any item failed: reads the library's device flag (4 bytes)."""
    pending = getattr(_TLS, "pending", None)
    if pending is not None:
        pending.append((h.flag, what))
        return
    if h.flag is not None and int(h.flag.item()) != 0:
        nat.check(nat.LMEP_NONFINITE, what)


def expm_batched(A: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """exp of A [B, d, d] on the device -> (E, status, ms)."""
    B, d, _ = A.shape
    if d > nat.MAX_DIM:
        raise DimensionMismatch(f"expm supports d <= {nat.MAX_DIM}, got {d}")
    E = torch.empty_like(A)
    status = torch.empty(B, dtype=torch.int32, device=A.device)
    ms = torch.empty(B, dtype=torch.int32, device=A.device)
    st = nat.lib().lmep_expm(nat.ptr(A), d, B, nat.ptr(E), nat.ptr(status), nat.ptr(ms),
                             nat.stream_handle())
    nat.check(st, "lmep_expm")
    return E, status, ms


# ---------------------------------------------------------------------------
# compact operator rows: the device form of one or more BandedPropagators
# ---------------------------------------------------------------------------
@dataclass
class CompactRows:
    """R operator rows on a StencilSet layout.

    SHARED : interior [R, n] serves every node (periodic uniform grids)
    CLASS  : interior [R, n] + classes [nleft+1+nright, R, n] (clamped ends)
    PERNODE: pernode SoA [R, n, N]
    """

    layout: StencilSet
    mode: int
    interior: torch.Tensor | None = None
    classes: torch.Tensor | None = None
    nleft: int = 0
    nright: int = 0
    pernode: torch.Tensor | None = None
    pernode_pad: int = 0                 # halo-node columns on each side of a shard's table
    _host_interior: np.ndarray | None = field(default=None, repr=False)

    @property
    def R(self) -> int:
        if self.mode == nat.W_PERNODE:
            return int(self.pernode.shape[0])
        return int(self.interior.shape[0])

    @property
    def n(self) -> int:
        return self.layout.n

    def host_interior(self) -> np.ndarray:
        if self._host_interior is None and self.interior is not None:
            self._host_interior = np.ascontiguousarray(to_host(self.interior))
        return self._host_interior

    def row(self, r: int) -> "CompactRows":
        """The single-operator view of row r."""
        if self.mode == nat.W_PERNODE:
            return CompactRows(self.layout, self.mode, pernode=self.pernode[r:r + 1].contiguous(),
                               pernode_pad=self.pernode_pad)
        cl = None if self.classes is None else self.classes[:, r:r + 1].contiguous()
        return CompactRows(self.layout, self.mode, self.interior[r:r + 1].contiguous(), cl,
                           self.nleft, self.nright)

    def dense(self) -> torch.Tensor:
        """Per-node rows [R, N, n] (the reference's (N, n) arrays, stacked)."""
        N, n = self.layout.N, self.n
        if self.mode == nat.W_PERNODE:
            return self.pernode.permute(0, 2, 1).contiguous()
        out = self.interior[:, None, :].expand(self.R, N, n).clone()
        if self.mode == nat.W_CLASS:
            if self.nleft:
                out[:, :self.nleft] = self.classes[:self.nleft].permute(1, 0, 2)
            if self.nright:
                out[:, N - self.nright:] = self.classes[self.nleft + 1:].permute(1, 0, 2)
        return out

    def to_pernode(self) -> "CompactRows":
        if self.mode == nat.W_PERNODE:
            return self
        return CompactRows(self.layout, nat.W_PERNODE,
                           pernode=self.dense().permute(0, 2, 1).contiguous())

    def with_classes(self, nleft: int, nright: int) -> "CompactRows":
        """Widen the class table (extra boundary classes repeat interior rows)."""
        if self.mode == nat.W_PERNODE:
            return self
        if self.mode == nat.W_CLASS and self.nleft == nleft and self.nright == nright:
            return self
        full = self.dense()                                   # [R, N, n]
        N = self.layout.N
        left = full[:, :nleft].permute(1, 0, 2)
        right = full[:, N - nright:].permute(1, 0, 2)
        mid = self.interior[None]
        cl = torch.cat([left, mid, right], dim=0).contiguous()
        return CompactRows(self.layout, nat.W_CLASS, self.interior, cl, nleft, nright)

    # ctypes views -----------------------------------------------------------
    def c_weights(self) -> nat.LmepWeights:
        w = nat.LmepWeights()
        w.mode = self.mode
        w.nrows = self.R
        w.nleft, w.nright = self.nleft, self.nright
        if self.mode != nat.W_PERNODE:
            w.interior = self.host_interior().ctypes.data
        w.classes = nat.ptr(self.classes) if self.classes is not None else None
        w.pernode = nat.ptr(self.pernode) if self.pernode is not None else None
        w.pernode_pad = int(self.pernode_pad)
        return w


def stack_rows(parts: list[CompactRows]) -> CompactRows:
    """Concatenate single/multi-row CompactRows (same layout) into one bank."""
    lay = parts[0].layout
    if any(p.mode == nat.W_PERNODE for p in parts):
        pads = {p.pernode_pad for p in parts if p.mode == nat.W_PERNODE}
        if len(pads) > 1 or (pads != {0} and any(p.mode != nat.W_PERNODE for p in parts)):
            raise InvalidConfig("cannot stack per-node tables with different halo padding")
        pn = [p.to_pernode().pernode for p in parts]
        return CompactRows(lay, nat.W_PERNODE, pernode=torch.cat(pn, 0).contiguous(),
                           pernode_pad=pads.pop())
    if any(p.mode == nat.W_CLASS for p in parts):
        nl = max(p.nleft for p in parts)
        nr = max(p.nright for p in parts)
        parts = [p.with_classes(nl, nr) for p in parts]
        interior = torch.cat([p.interior for p in parts], 0).contiguous()
        cl = torch.cat([p.classes for p in parts], 1).contiguous()
        return CompactRows(lay, nat.W_CLASS, interior, cl, nl, nr)
    return CompactRows(lay, nat.W_SHARED, torch.cat([p.interior for p in parts], 0).contiguous())


def compress(dense: torch.Tensor, layout: StencilSet, max_classes: int = 64) -> CompactRows:
    """(N, n) per-node rows -> the most compact exact representation.  The rows
    equal to the middle one are located by the library (lmep_rows_classify:
    first / last equal row and their count, 24 bytes back to the host)."""
    N = layout.N
    w = dense.to(dtype=F64).contiguous()
    out3 = torch.empty(3, dtype=torch.int64, device=w.device)
    st = nat.lib().lmep_rows_classify(w.data_ptr(), N, layout.n, N // 2, out3.data_ptr(),
                                      nat.stream_handle())
    nat.check(st, "lmep_rows_classify")
    first, last, count = (int(x) for x in out3.tolist())
    mid = w[N // 2]
    if count == N and layout.periodic:
        return CompactRows(layout, nat.W_SHARED, mid[None].clone())
    if not layout.periodic:
        nl, nr = first, N - 1 - last
        if count == last - first + 1 and nl + nr <= max_classes and nl + nr < N:
            cl = torch.cat([w[:nl], mid[None], w[N - nr:]], 0)[:, None, :].contiguous()
            return CompactRows(layout, nat.W_CLASS, mid[None].clone(), cl, nl, nr)
    return CompactRows(layout, nat.W_PERNODE, pernode=w.t().contiguous()[None])


def combine_into(out: torch.Tensor, ins: list[torch.Tensor], coeffs, rows: int, cols: int,
                 ld_out: int, ld_in: list[int]) -> None:
    """out(r, j) = sum_t coeffs[t] * ins[t](r, j) from zeros in list order
    (harvest.combine, harvest.py:225-235) on the library's combine kernel; the
    tensors are strided row arrays (row r at r * ld)."""
    k = len(ins)
    ptrs = (C.c_void_p * k)(*[t.data_ptr() for t in ins])
    lds = (C.c_int64 * k)(*[int(x) for x in ld_in])
    cs = (C.c_double * k)(*[float(c) for c in coeffs])
    st = nat.lib().lmep_combine(k, ptrs, lds, cs, int(rows), int(cols), out.data_ptr(), int(ld_out),
                                nat.stream_handle())
    nat.check(st, "lmep_combine")


def combine_rows(parts: list[CompactRows], coeffs) -> CompactRows:
    """sum_i coeffs[i] * parts[i], accumulated from zeros in list order
    (harvest.combine, harvest.py:225-235): two roundings per term like numpy."""
    bank = stack_rows(parts)                      # aligns modes / classes
    R = parts[0].R
    K = len(parts)
    if bank.mode == nat.W_PERNODE:
        src = bank.pernode                        # [K*R, n, N]
        blk = src[0].numel() * R
        out = torch.empty_like(src[:R])
        combine_into(out, [src[i * R:(i + 1) * R] for i in range(K)], coeffs, 1, blk, blk,
                     [blk] * K)
        return CompactRows(bank.layout, nat.W_PERNODE, pernode=out, pernode_pad=bank.pernode_pad)
    n = bank.n
    it = torch.empty((R, n), dtype=F64, device=bank.interior.device)
    combine_into(it, [bank.interior[i * R:(i + 1) * R] for i in range(K)], coeffs, 1, R * n, R * n,
                 [R * n] * K)
    cl = None
    if bank.classes is not None:
        Cn = bank.classes.shape[0]
        cl = torch.empty((Cn, R, n), dtype=F64, device=it.device)
        ldi = K * R * n
        combine_into(cl, [bank.classes[:, i * R:(i + 1) * R] for i in range(K)], coeffs, Cn, R * n,
                     R * n, [ldi] * K)
    return CompactRows(bank.layout, bank.mode, it, cl, bank.nleft, bank.nright)


# ---------------------------------------------------------------------------
# stepping (K3-K5)
# ---------------------------------------------------------------------------
def c_halo(halo) -> nat.LmepHalo | None:
    """halo = (left, right, hist_left, hist_right, width[, push_left, push_right,
    push_width]): device tensors, raw device pointers (mailbox slots of the
    communicator) or None."""
    if halo is None:
        return None

    def ptr(x):
        return x if (x is None or isinstance(x, int)) else x.data_ptr()

    h = nat.LmepHalo()
    h.left, h.right = ptr(halo[0]), ptr(halo[1])
    h.hist_left, h.hist_right = ptr(halo[2]), ptr(halo[3])
    h.width = int(halo[4])
    if len(halo) > 5:
        h.push_left, h.push_right, h.push_width = ptr(halo[5]), ptr(halo[6]), int(halo[7])
    return h


def c_grid(layout: StencilSet, off: int = 0, nloc: int | None = None) -> nat.LmepGrid:
    g = nat.LmepGrid()
    g.N = layout.N
    g.off = off
    g.nloc = layout.N if nloc is None else nloc
    g.n = layout.n
    g.row = layout.row
    g.periodic = 1 if layout.periodic else 0
    return g


class BC:
    """Boundary closure description for the step kernels."""

    def __init__(self, kind: int = nat.BC_NONE, lo: float = 0.0, hi: float = 0.0, dl=None,
                 dr=None):
        self.kind, self.lo, self.hi = kind, float(lo), float(hi)
        self.dl = None if dl is None else np.ascontiguousarray(np.asarray(dl, dtype=np.float64))
        self.dr = None if dr is None else np.ascontiguousarray(np.asarray(dr, dtype=np.float64))

    def c(self) -> nat.LmepBC:
        b = nat.LmepBC()
        b.kind = self.kind
        b.lo, b.hi = self.lo, self.hi
        b.dl = None if self.dl is None else self.dl.ctypes.data
        b.dr = None if self.dr is None else self.dr.ctypes.data
        return b


def _tuning(tuning) -> nat.LmepTuning | None:
    if tuning is None:
        return None
    t = nat.LmepTuning()
    t.tile = int(tuning.get("tile", 0))
    t.ksteps = int(tuning.get("ksteps", 0))
    t.ring = int(tuning.get("ring", 0))
    t.threads = int(tuning.get("threads", 0))
    return t


def step(scheme: int, rows: CompactRows, u: torch.Tensor, steps: int, *, bc: BC | None = None,
         nl: int = nat.NL_NONE, exact: bool = True, hist: torch.Tensor | None = None,
         delta_t: float = 0.0, nl0_out: torch.Tensor | None = None, tuning=None,
         flag: torch.Tensor | None = None, out: torch.Tensor | None = None,
         hist_out: torch.Tensor | None = None, scratch: torch.Tensor | None = None,
         off: int = 0, nloc: int | None = None, halo=None, etd_order: int = 2,
         host_out: torch.Tensor | None = None, copy_stream: int | None = None, host_parts: int = 4):
    """Run `steps` steps of a scheme on the whole grid, or on the shard
    [off, off+nloc) with ghost cells `halo` (see c_halo).
    Returns the new u (and the new history for ETD2)."""
    lay = rows.layout
    g = c_grid(lay, off, nloc)
    hc = c_halo(halo)
    hp = C.byref(hc) if hc is not None else None
    w = rows.c_weights()
    b = (bc or BC()).c()
    u = u.contiguous()
    out = torch.empty_like(u) if out is None else out
    flags = nat.FLAG_EXACT if exact else 0
    tun = _tuning(tuning)
    tp = C.byref(tun) if tun is not None else None
    L = nat.lib()
    s = nat.stream_handle()
    fp = nat.ptr(flag)
    if scheme == nat.SCH_LIN:
        if host_out is not None and steps > 0:
            # the result also lands in (page-locked) host memory through copy_stream,
            # range by range behind the last launch (lmep_step_linear_host)
            st = L.lmep_step_linear_host(C.byref(g), C.byref(w), C.byref(b), hp, nat.ptr(u),
                                         nat.ptr(out), nat.ptr(scratch), int(steps), flags, tp, fp,
                                         s, host_out.data_ptr(), int(host_parts), copy_stream)
            nat.check(st, "lmep_step_linear_host")
            return out
        st = L.lmep_step_linear(C.byref(g), C.byref(w), C.byref(b), hp, nat.ptr(u),
                                nat.ptr(out), nat.ptr(scratch), int(steps), flags, tp, fp, s)
        nat.check(st, "lmep_step_linear")
        return out
    if scheme == nat.SCH_ETDRK4:
        st = L.lmep_step_etdrk4(C.byref(g), C.byref(w), C.byref(b), hp, nl, nat.ptr(u),
                                nat.ptr(out), nat.ptr(scratch), int(steps), nat.ptr(nl0_out),
                                flags, tp, fp, s)
        nat.check(st, "lmep_step_etdrk4")
        return out
    order = int(etd_order)
    if order > 1:
        hist = hist.contiguous()
        hist_out = torch.empty_like(hist) if hist_out is None else hist_out
    st = L.lmep_step_etds(C.byref(g), C.byref(w), C.byref(b), hp, nl, order, float(delta_t),
                          nat.ptr(u), nat.ptr(hist) if order > 1 else None, nat.ptr(out),
                          nat.ptr(hist_out) if order > 1 else None, nat.ptr(scratch), int(steps),
                          flags, tp, fp, s)
    nat.check(st, "lmep_step_etds")
    return out, hist_out


def rows_bank_for(layout: StencilSet, slots: dict[int, CompactRows], nrows: int) -> CompactRows:
    """Operator bank with rows placed at their LMEP_ROW_* slots (missing = 0)."""
    parts = []
    proto = next(iter(slots.values()))
    for r in range(nrows):
        if r in slots:
            parts.append(slots[r])
        else:
            z = CompactRows(layout, nat.W_SHARED, torch.zeros_like(proto.row(0).interior)) \
                if proto.mode != nat.W_PERNODE else \
                CompactRows(layout, nat.W_PERNODE, pernode=torch.zeros_like(proto.row(0).pernode))
            parts.append(z)
    return stack_rows(parts)


def validate_members(members, weights_shape) -> StencilSet:
    """Recognise the reference's (N, n) int64 member array as a StencilSet
    (periodic wrap or clamped windows); anything else has no device path."""
    m = members.detach().cpu().numpy() if isinstance(members, torch.Tensor) else np.asarray(members)
    m = np.asarray(m, dtype=np.int64)
    if m.ndim != 2 or tuple(m.shape) != tuple(weights_shape):
        raise DimensionMismatch("weights and members must share an (N, n) shape")
    N, n = m.shape
    t = N // 2
    row = int(t - m[t, 0])
    for periodic in (True, False):
        if not 0 <= row < n:
            continue
        cand = StencilSet(N, n, row, periodic)
        if np.array_equal(cand.members_array(), m):
            return cand
    # periodic windows whose interior start wraps (row from modular offset)
    row = int((t - m[t, 0]) % N)
    if 0 <= row < n:
        cand = StencilSet(N, n, row, True)
        if np.array_equal(cand.members_array(), m):
            return cand
    raise InvalidConfig("members are not contiguous select_stencils windows; no device path")


def plan(layout: StencilSet, scheme: int, nl: int, weight_mode: int, steps: int) -> dict:
    """The launch shape liblmep picks (lmep_plan): tile, ksteps, ring, threads."""
    g = c_grid(layout)
    t = nat.LmepTuning()
    st = nat.lib().lmep_plan(C.byref(g), scheme, nl, weight_mode, int(steps), C.byref(t))
    nat.check(st, "lmep_plan")
    return {"tile": t.tile, "ksteps": t.ksteps, "ring": t.ring, "threads": t.threads}
