"""Slab-sharded stepping across GPUs.

One process per GPU.  The grid is cut into contiguous slabs; every rank
harvests what its slab needs without communication (the <= 2n+1 stencil
classes redundantly, or its own nodes' per-node rows) and advances its slab
with the fused step kernels.  The only data exchange is the halo: before a
launch that fuses k steps, each rank sends its first and last
G = k * ext * max(row, n-1-row) nodes to its neighbours (periodic ring or
open chain).  A deep halo (k > 1) trades a little redundant edge compute for
k times fewer exchanges.

The data plane is the library's communicator (``Comm`` = ``lmep_comm`` of
include/lmep.h): NCCL send / receive pairs on the step stream, or peer stores
into CUDA-IPC mailboxes; torch.distributed only carries the bootstrap bytes
(the NCCL id, the IPC handles).  With a ``CommHalo`` exchanger a chunk is

    fork -> halo exchange (side stream) || interior sub-slab (step stream)
         -> join -> the two edge strips

and, on the NCCL transport, the whole chunk is replayed from a CUDA graph
(one graph per ping-pong direction).  Other exchangers share the driver:

  * ``TorchHalo`` -- torch.distributed batch_isend_irecv (gloo on CPU for the
                     host-side tests, NCCL through torch otherwise);
  * ``LocalHalo`` -- P virtual shards inside one process (device copies),
                     used to check sharded == unsharded on a single GPU.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from . import _ops
from .errors import InvalidConfig, NonFinite
from .grid import Grid, as_stencil_set
from .harvest import harvest_compact
from .timestep import (Prepared, SchemeConfig, SemiLinearProblem, _bc_for, _etdrk4_bank,
                       _nl_kind, _scaled, close_initial, derivative_compact)


def partition(N: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous slab [off, off+nloc) of rank; sizes differ by at most one."""
    base, rem = divmod(int(N), int(world))
    off = rank * base + min(rank, rem)
    return off, base + (1 if rank < rem else 0)


def neighbours(rank: int, world: int, periodic: bool) -> tuple[int | None, int | None]:
    if world == 1:
        return (None, None)
    left = (rank - 1) % world if (periodic or rank > 0) else None
    right = (rank + 1) % world if (periodic or rank < world - 1) else None
    return left, right


class Comm:
    """One rank's ``lmep_comm`` (include/lmep.h, "sharded runs")."""

    def __init__(self, rank: int, world: int, periodic: bool, transport: str = "nccl",
                 unique_id: bytes | None = None, max_width: int = 0):
        self.rank, self.world, self.periodic, self.transport = rank, world, bool(periodic), transport
        code = {"nccl": nat.COMM_NCCL, "peer": nat.COMM_PEER}[transport]
        nat.device()
        h = C.c_void_p()
        idb = None
        if code == nat.COMM_NCCL:
            if unique_id is None or len(unique_id) != nat.COMM_ID_BYTES:
                raise InvalidConfig("the NCCL transport needs rank 0's Comm.unique_id()")
            idb = C.create_string_buffer(bytes(unique_id), nat.COMM_ID_BYTES)
        nat.check(nat.lib().lmep_comm_init(C.byref(h), rank, world, int(bool(periodic)), code, idb,
                                           int(max_width)), "lmep_comm_init")
        self.h = h
        l, r = C.c_int(), C.c_int()
        nat.lib().lmep_comm_info(h, None, None, C.byref(l), C.byref(r), None)
        self.left = None if l.value < 0 else l.value
        self.right = None if r.value < 0 else r.value
        self.side_stream = nat.lib().lmep_comm_side_stream(h)
        self._steppers: list = []           # weak references: their graphs go before the communicator

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(nat.COMM_ID_BYTES)
        nat.check(nat.lib().lmep_comm_unique_id(buf), "lmep_comm_unique_id")
        return buf.raw

    def export(self) -> bytes:
        buf = C.create_string_buffer(nat.COMM_BLOB_BYTES)
        nat.check(nat.lib().lmep_comm_export(self.h, buf), "lmep_comm_export")
        return buf.raw

    def connect(self, blobs: list[bytes] | None) -> None:
        raw = None
        if blobs is not None:
            if len(blobs) != self.world or any(len(b) != nat.COMM_BLOB_BYTES for b in blobs):
                raise InvalidConfig("connect() needs one exported blob per rank")
            raw = C.create_string_buffer(b"".join(blobs), self.world * nat.COMM_BLOB_BYTES)
        nat.check(nat.lib().lmep_comm_connect(self.h, raw), "lmep_comm_connect")

    def exchange(self, fields, width: int, gls, grs, stream: int | None = None) -> None:
        """Ghost cells of every field (equal-length device vectors) in one call."""
        k = len(fields)
        nloc = fields[0].numel()
        fp = (C.c_void_p * k)(*[f.data_ptr() for f in fields])
        lp = (C.c_void_p * k)(*[g.data_ptr() for g in gls])
        rp = (C.c_void_p * k)(*[g.data_ptr() for g in grs])
        s = nat.stream_handle() if stream is None else stream
        nat.check(nat.lib().lmep_halo_exchange(self.h, k, fp, nloc, int(width), lp, rp, s),
                  "lmep_halo_exchange")

    # ---- peer transport, piecewise (fused peer stores in the step launches) ----
    def targets(self, field: int = 0):
        """Peer pointers where this rank's left / right edge goes for its next signal."""
        a, b = C.c_void_p(), C.c_void_p()
        nat.check(nat.lib().lmep_comm_targets(self.h, field, C.byref(a), C.byref(b)),
                  "lmep_comm_targets")
        return a.value, b.value

    def ghosts(self, field: int = 0):
        """This rank's own mailbox slots of the latest exchange (left, right ghosts)."""
        a, b = C.c_void_p(), C.c_void_p()
        nat.check(nat.lib().lmep_comm_ghosts(self.h, field, C.byref(a), C.byref(b)),
                  "lmep_comm_ghosts")
        return a.value, b.value

    def push(self, fields, width: int) -> None:
        k = len(fields)
        fp = (C.c_void_p * k)(*[f.data_ptr() for f in fields])
        nat.check(nat.lib().lmep_comm_push(self.h, k, fp, fields[0].numel(), int(width),
                                           nat.stream_handle()), "lmep_comm_push")

    def signal(self) -> None:
        nat.check(nat.lib().lmep_comm_signal(self.h, nat.stream_handle()), "lmep_comm_signal")

    def wait(self) -> None:
        nat.check(nat.lib().lmep_comm_wait(self.h, nat.stream_handle()), "lmep_comm_wait")

    def gather(self, u: torch.Tensor, counts, out: torch.Tensor | None, root: int = 0) -> None:
        cn = (C.c_int64 * self.world)(*[int(c) for c in counts])
        nat.check(nat.lib().lmep_comm_gather(self.h, u.data_ptr(), cn, nat.ptr(out), root,
                                             nat.stream_handle()), "lmep_comm_gather")

    def flag_max(self, flag: torch.Tensor) -> None:
        nat.check(nat.lib().lmep_comm_flag_max(self.h, flag.data_ptr(), flag.numel(),
                                               nat.stream_handle()), "lmep_comm_flag_max")

    def fork(self) -> None:
        nat.check(nat.lib().lmep_comm_fork(self.h, nat.stream_handle()), "lmep_comm_fork")

    def join(self) -> None:
        nat.check(nat.lib().lmep_comm_join(self.h, nat.stream_handle()), "lmep_comm_join")

    def close(self) -> None:
        if self.h is not None:
            # graphs that captured this communicator's NCCL work must be destroyed
            # first (ncclCommDestroy waits for them)
            for ref in self._steppers:
                st = ref()
                if st is not None:
                    st._graphs.clear()
            self._steppers.clear()
            nat.lib().lmep_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Graph:
    """A captured chunk (``lmep_graph``): record with ``with Graph.capture() as g``."""

    def __init__(self):
        self.h = None

    class _Capture:
        def __init__(self, g):
            self.g = g

        def __enter__(self):
            self.s = nat.stream_handle()
            nat.check(nat.lib().lmep_graph_begin(self.s), "lmep_graph_begin")
            return self.g

        def __exit__(self, et, ev, tb):
            h = C.c_void_p()
            st = nat.lib().lmep_graph_end(self.s, C.byref(h))
            if et is None:
                nat.check(st, "lmep_graph_end")
                self.g.h = h
            elif st == 0:
                nat.lib().lmep_graph_destroy(h)
            return False

    @classmethod
    def capture(cls):
        return cls._Capture(cls())

    def launch(self) -> None:
        nat.check(nat.lib().lmep_graph_launch(self.h, nat.stream_handle()), "lmep_graph_launch")

    def __del__(self):
        try:
            if self.h is not None:
                nat.lib().lmep_graph_destroy(self.h)
        except Exception:
            pass


def make_comm(rank: int, world: int, periodic: bool, transport: str = "nccl", group=None,
              max_width: int = 0) -> Comm:
    """Bootstrap a ``Comm`` over a torch.distributed group: the group only
    carries the NCCL id (128 bytes from rank 0) or the ranks' IPC handles."""
    import torch.distributed as dist
    multi = world > 1
    if transport == "nccl":
        box = [Comm.unique_id() if rank == 0 else None]
        if multi:
            dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group else 0,
                                       group=group)
        return Comm(rank, world, periodic, "nccl", unique_id=box[0])
    c = Comm(rank, world, periodic, "peer", max_width=max_width)
    blobs = [c.export()]
    if multi:
        blobs = [None] * world
        dist.all_gather_object(blobs, c.export(), group=group)
    c.connect(blobs)
    return c


class CommHalo:
    """Halo exchange through the library communicator (NCCL or peer stores)."""

    def __init__(self, comm: Comm):
        self.comm = comm
        self.rank, self.world = comm.rank, comm.world
        self.left, self.right = comm.left, comm.right

    def exchange_many(self, fields, width, gls, grs, stream=None) -> None:
        if fields[0].numel() < width:
            raise InvalidConfig(f"slab of {fields[0].numel()} nodes is narrower than the halo {width}")
        self.comm.exchange(fields, width, gls, grs, stream)

    def exchange(self, u, gl, gr) -> None:
        self.exchange_many([u], gl.numel(), [gl], [gr])


class TorchHalo:
    """Halo exchange over torch.distributed point-to-point (one group call).

    Posting order per rank: send right edge -> right, recv left ghosts <- left,
    send left edge -> left, recv right ghosts <- right.  Messages between a
    pair match in posting order, which also makes the 2-rank periodic ring
    (left == right) come out right.  Device slabs on a gloo group are staged
    through the host.
    """

    def __init__(self, rank: int, world: int, periodic: bool, group=None):
        self.rank, self.world, self.group = rank, world, group
        self.left, self.right = neighbours(rank, world, periodic)

    def exchange(self, u: torch.Tensor, gl: torch.Tensor, gr: torch.Tensor) -> None:
        import torch.distributed as dist
        G = gl.numel()
        if u.numel() < G:
            raise InvalidConfig(f"slab of {u.numel()} nodes is narrower than the halo {G}")
        staged = u.is_cuda and dist.get_backend(self.group) == "gloo"
        edge = (lambda t: t.cpu()) if staged else (lambda t: t.contiguous())
        rl = torch.empty(G, dtype=u.dtype) if staged else gl
        rr = torch.empty(G, dtype=u.dtype) if staged else gr
        ops = []
        if self.right is not None:
            ops.append(dist.P2POp(dist.isend, edge(u[u.numel() - G:]), self.right, self.group))
        if self.left is not None:
            ops.append(dist.P2POp(dist.irecv, rl, self.left, self.group))
            ops.append(dist.P2POp(dist.isend, edge(u[:G]), self.left, self.group))
        if self.right is not None:
            ops.append(dist.P2POp(dist.irecv, rr, self.right, self.group))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        if staged:
            if self.left is not None:
                gl.copy_(rl)
            if self.right is not None:
                gr.copy_(rr)


NcclHalo = TorchHalo          # the name earlier callers used


class LocalHalo:
    """P virtual shards of one process: ghosts are copied from the neighbour
    shards' device buffers (registered in ``shards``)."""

    def __init__(self, shards: list, rank: int, periodic: bool):
        self.shards, self.rank = shards, rank
        self.left, self.right = neighbours(rank, len(shards), periodic)
        self.which = "u"

    def _src(self, shard):
        if isinstance(self.which, tuple):
            return getattr(shard, self.which[0])[self.which[1]]
        return getattr(shard, self.which)

    def exchange(self, u: torch.Tensor, gl: torch.Tensor, gr: torch.Tensor) -> None:
        G = gl.numel()
        if self.left is not None:
            src = self._src(self.shards[self.left])
            gl.copy_(src[src.numel() - G:])
        if self.right is not None:
            src = self._src(self.shards[self.right])
            gr.copy_(src[:G])


@dataclass
class SlabPlan:
    off: int
    nloc: int
    width: int          # ghost cells per side
    ksteps: int         # steps per exchange


def _ext(scheme: str, nl: int) -> int:
    cv = 1 if nl == nat.NL_CONVECTIVE else 0
    return {"linear": 1, "etdrk4": 4 + 4 * cv, "etd-multistep": 1 + cv}[scheme]


class ShardedStepper:
    """Advance one slab of a run (the sharded counterpart of timestep.Stepper).

    u and the multistep history ping-pong between two fixed buffers each, so a
    chunk (exchange + fused k-step launch) can be replayed from a CUDA graph.
    ``force_halo`` makes a single periodic rank exchange with itself through
    the communicator (the real data path on one GPU)."""

    def __init__(self, grid: Grid, stencils, problem: SemiLinearProblem, scheme: SchemeConfig,
                 delta_t: float, rank: int, world: int, exchanger, *, exact: bool = True,
                 ksteps: int | None = None, tuning=None, overlap: bool = True,
                 graph: bool | None = None, force_halo: bool = False):
        sset = as_stencil_set(grid, stencils)
        self.sset, self.rank, self.world = sset, rank, world
        self.exact, self.tuning = exact, tuning
        nl = _nl_kind(problem)
        off, nloc = partition(sset.N, world, rank)
        reach = max(sset.row, sset.n - 1 - sset.row)
        ext = _ext(scheme.kind, nl)
        per_node = _is_per_node(grid, problem)
        self.sharded = world > 1 or (force_halo and grid.periodic)
        # periodic per-node linear rows: the shard also harvests its halo
        # nodes' rows (no communication), so k steps fuse per exchange
        pad_ok = per_node and scheme.kind == "linear" and grid.periodic
        if ksteps is None:
            # steps per exchange: 16 for the one-pass schemes; the ETDRK4 kernel keeps
            # one chunk of nodes per thread, so its staged range (tile + k * halo) is
            # bounded and it takes the single-GPU plan's 6 (pointwise N) / 3 (convective)
            cap = 16 if scheme.kind != "etdrk4" else (3 if nl == nat.NL_CONVECTIVE else 6)
            if pad_ok and nloc >= 4096:
                cap = 24                    # the persistent per-node kernels' sweet spot (1536-node spans)
            ksteps = max(1, min(cap, nloc // (4 * ext * max(reach, 1))))
        if per_node and scheme.kind == "linear" and self.sharded and not pad_ok:
            ksteps = 1                      # non-periodic per-node rows: one step per exchange
        if not self.sharded:
            ksteps = 1 << 30                # no halo: the library plans the launches
        if per_node and scheme.kind != "linear" and self.sharded:
            raise InvalidConfig("sharded ETD schemes need shared or class rows")
        width = ksteps * ext * reach if self.sharded else 0
        if self.sharded and width > nloc:
            raise InvalidConfig(f"slab of {nloc} nodes narrower than the halo {width}")
        self.plan = SlabPlan(off, nloc, width, ksteps)
        pad = ksteps * reach if (pad_ok and self.sharded and ksteps > 1) else 0
        self.prep = _prepare_shard(grid, sset, problem, scheme, delta_t, off, nloc, pad)
        self.ex = exchanger
        # interior / edge split and graph replay need the library communicator
        # and kernels whose sub-slabs keep their leading dimensions
        comm_ex = isinstance(exchanger, CommHalo)
        self.overlap = bool(overlap and comm_ex and self.sharded and not per_node and
                            scheme.kind in ("linear", "etdrk4"))
        if graph is None:
            graph = comm_ex and exchanger.comm.transport == "nccl"
        self.graph = bool(graph and comm_ex and self.sharded and
                          exchanger.comm.transport == "nccl")
        # peer transport: the step launches store their edges into the neighbours'
        # mailboxes themselves and read their ghosts straight out of their own
        self.fused = bool(self.overlap and exchanger.comm.transport == "peer")
        self._pushed_w = 0
        self._graphs: dict = {}
        self._seen: set = set()
        if comm_ex:
            import weakref
            exchanger.comm._steppers.append(weakref.ref(self))
        dev = nat.device()
        self.flag = torch.zeros(4, dtype=torch.int32, device=dev)
        G = max(width, 1)
        nh = max(scheme.s - 1, 1) if scheme.kind == "etd-multistep" else 1
        # ghost cells: u's sit right around it -- both ping-pong buffers are extended
        # arrays [G ghosts | nloc | G ghosts], so a slab reads like a whole grid (the
        # persistent per-node kernels bulk-copy straight across the seam); the
        # [s-1][width] multistep history ghosts are separate.  One slab has none.
        self._G = G if self.sharded else 0
        self._ext = None
        if self.sharded:
            self._ext = [torch.zeros(nloc + 2 * G, dtype=torch.float64, device=dev) for _ in range(2)]
            hg = torch.zeros(2 * nh * G, dtype=torch.float64, device=dev)
            self.ql, self.qr = hg[:nh * G], hg[nh * G:]
        else:
            self.ql = self.qr = None
        self.u = None
        self._out = None
        self.hist = None
        self._hout = None
        self.done = 0
        self._warm_done = 0
        # ping-pong scratch for multi-launch calls (u and the etd2 history)
        self.scratch = torch.empty((nh + 1) * nloc, dtype=torch.float64, device=dev)

    # ---------------------------------------------------------------------
    def set_initial(self, u0_global) -> None:
        """Slice the (closed) global initial data for this slab."""
        u = _ops.dev_f64(u0_global)
        u = close_initial(u, self.sset, self.prep.bc)
        self.set_local(u[self.plan.off:self.plan.off + self.plan.nloc])

    def set_local(self, u_local: torch.Tensor) -> None:
        """This slab's initial values (copied: inputs are never written)."""
        if self._ext is not None:
            G, n = self._G, self.plan.nloc
            self.u, self._out = self._ext[0][G:G + n], self._ext[1][G:G + n]
            self.u.copy_(u_local)
        else:
            self.u = u_local.clone().contiguous()
            self._out = torch.empty_like(self.u)
        self._graphs.clear()
        self._seen.clear()
        self._pushed_w = 0

    def _width(self, k, scheme=None):
        ext = _ext(scheme or self.prep.scheme, self.prep.nl)
        return k * ext * max(self.sset.row, self.sset.n - 1 - self.sset.row)

    def _nh(self):
        return max(self.prep.s - 1, 1) if self.prep.scheme == "etd-multistep" else 1

    def _halo(self, k):
        if not self.sharded:
            return None
        w = max(self._width(k), 1)
        nh = self._nh()
        gl, gr = self._ghosts(w)
        return (gl, gr, self.ql[:nh * w], self.qr[:nh * w], w)

    def _ghosts(self, w: int):
        """The w ghost cells on each side of the current u, inside its extended buffer."""
        G, n = self._G, self.plan.nloc
        ext = self._ext[0] if self.u.data_ptr() == self._ext[0][G:].data_ptr() else self._ext[1]
        return ext[G - w:G], ext[G + n:G + n + w]

    def _hist_fields(self):
        p = self.prep
        if p.scheme == "etd-multistep" and p.s > 1 and self.hist is not None:
            return [self.hist[i] for i in range(self.hist.shape[0])]
        return []

    def exchange_phase(self, k: int, stream=None) -> None:
        """Ghost cells of u (and of the multistep history) for a k-step launch."""
        if not self.sharded:
            return
        h = self._halo(k)
        w = h[4]
        hf = self._hist_fields()
        if hasattr(self.ex, "exchange_many"):
            fields = [self.u] + hf
            gls = [h[0]] + [h[2][i * w:(i + 1) * w] for i in range(len(hf))]
            grs = [h[1]] + [h[3][i * w:(i + 1) * w] for i in range(len(hf))]
            self.ex.exchange_many(fields, w, gls, grs, stream)
            return
        local = isinstance(self.ex, LocalHalo)
        if local:
            self.ex.which = "u"
        self.ex.exchange(self.u, h[0], h[1])
        for i, f in enumerate(hf):
            if local:
                self.ex.which = ("hist", i)
            self.ex.exchange(f, h[2][i * w:(i + 1) * w], h[3][i * w:(i + 1) * w])

    def _tuning(self, k):
        if not self.sharded:
            return self.tuning              # single shard: library heuristics
        return {**(self.tuning or {}), "ksteps": k}

    def _launch(self, k: int) -> None:
        """The k-step launch of the whole slab: self.u -> self._out (no swap)."""
        p = self.prep
        kw = dict(bc=p.bc, nl=p.nl, exact=self.exact, tuning=self._tuning(k), flag=self.flag[0:1],
                  off=self.plan.off, nloc=self.plan.nloc, halo=self._halo(k),
                  scratch=self.scratch, out=self._out)
        if p.scheme == "linear":
            _ops.step(nat.SCH_LIN, p.bank, self.u, k, **kw)
        elif p.scheme == "etdrk4":
            _ops.step(nat.SCH_ETDRK4, p.bank, self.u, k, **kw)
        else:
            if self.hist is None:
                raise InvalidConfig("call warm_up() before multistep chunks")
            _ops.step(nat.SCH_ETD2, p.bank, self.u, k, hist=self.hist, delta_t=p.delta_t,
                      etd_order=p.s, hist_out=self._hout, **kw)

    def _swap(self) -> None:
        self.u, self._out = self._out, self.u
        if self.prep.scheme == "etd-multistep" and self.prep.s > 1:
            self.hist, self._hout = self._hout, self.hist

    def _enqueue_chunk(self, k: int, k_next: int) -> None:
        """One chunk in one library call (lmep_comm_chunk): on NCCL, fork -> side
        stream: halo exchange into the ghost cells around u, then the two edge
        strips || step stream: the interior sub-slab -> join; on the peer
        transport no exchange kernel at all -- the interior runs on the side
        stream while the step stream waits for the neighbours, runs the strips
        with their ghosts read in place from this rank's mailbox, and those
        launches store the next chunk's halo straight into the neighbours'
        mailboxes (peer memory)."""
        p, cm = self.prep, self.ex.comm
        g = _ops.c_grid(self.sset, self.plan.off, self.plan.nloc)
        w = p.bank.c_weights()
        b = (p.bc or _ops.BC()).c()
        a = nat.LmepChunkArgs()
        a.grid, a.w, a.bc = C.addressof(g), C.addressof(w), C.addressof(b)
        a.scheme = nat.SCH_LIN if p.scheme == "linear" else nat.SCH_ETDRK4
        a.nl_kind = p.nl
        a.u_in, a.u_out = self.u.data_ptr(), self._out.data_ptr()
        a.ghost_cells = self._G
        a.steps, a.next_steps = int(k), int(k_next)
        a.pushed_cells = self._pushed_w
        a.flags = nat.FLAG_EXACT if self.exact else 0
        a.nonfinite = self.flag.data_ptr()
        nat.check(nat.lib().lmep_comm_chunk(cm.h, C.byref(a), nat.stream_handle()), "lmep_comm_chunk")
        if self.fused:
            self._pushed_w = min(self._width(k_next), self._width(k)) if k_next > 0 else 0

    def _enqueue(self, k: int, k_next: int = 0) -> None:
        if self.overlap:
            self._enqueue_chunk(k, k_next)
        else:
            self.exchange_phase(k)
            self._launch(k)

    def step_chunk(self, k: int, k_next: int = 0) -> None:
        """k <= plan.ksteps steps with one halo exchange (k_next: the size of the
        chunk that follows, so a fused launch can store its halo ahead).  With
        LocalHalo the caller must run exchange_phase on all shards before
        compute_phase."""
        if self.graph and nat.stream_handle() != 0:     # the legacy stream cannot be captured
            # one graph per (k, ping-pong direction): run a chunk shape once
            # eagerly (NCCL connects, kernels get their attributes), capture it
            # the second time it comes up, replay it from then on
            key = (k, self.u.data_ptr(), 0 if self.hist is None else self.hist.data_ptr())
            g = self._graphs.get(key)
            if g is None and key in self._seen:
                with Graph.capture() as g:
                    self._enqueue(k)
                self._graphs[key] = g
            if g is not None:
                g.launch()
            else:
                self._seen.add(key)
                self._enqueue(k)
        else:
            self._enqueue(k, k_next)
        self._swap()
        self.done += k

    def compute_phase(self, k: int) -> None:
        self._launch(k)
        self._swap()
        self.done += k

    # ETD multistep warm-up (timestep.py:375-378): s-1 ETDRK4 steps, each
    # storing N(u) in front of the history; each needs its own halo exchange.
    def warm_up_steps(self) -> int:
        return max(self.prep.s - 1, 0) if self.prep.scheme == "etd-multistep" else 0

    def warm_up_exchange(self) -> None:
        if self.hist is None:
            self.hist = torch.zeros((self._nh(), self.u.numel()), dtype=torch.float64,
                                    device=self.u.device)
            self._hout = torch.empty_like(self.hist)
        if not self.sharded:
            return
        w = self._width(1, "etdrk4")
        dev = self.u.device
        self.wl = torch.zeros(w, dtype=torch.float64, device=dev)
        self.wr = torch.zeros(w, dtype=torch.float64, device=dev)
        if isinstance(self.ex, LocalHalo):
            self.ex.which = "u"
        self.ex.exchange(self.u, self.wl, self.wr)

    def warm_up_compute(self, i: int = 0) -> None:
        """Warm-up step i (0-based) of s-1."""
        p = self.prep
        if i > 0:
            self.hist[1:i + 1] = self.hist[0:i].clone()
        halo = None
        if self.sharded:
            w = self._width(1, "etdrk4")
            halo = (self.wl, self.wr, self.wl, self.wr, w)
        kw = dict(bc=p.bc, nl=p.nl, exact=self.exact, tuning=self._tuning(1), flag=self.flag[0:1],
                  off=self.plan.off, nloc=self.plan.nloc, halo=halo, out=self._out)
        _ops.step(nat.SCH_ETDRK4, p.warm, self.u, 1, nl0_out=self.hist[0], **kw)
        self.u, self._out = self._out, self.u
        self.done += 1
        self._warm_done = i + 1

    def nonfinite(self) -> bool:
        return bool(self.flag.max().item())


def _is_per_node(grid: Grid, problem: SemiLinearProblem) -> bool:
    from .localop import VariableCoefficientSpec
    return isinstance(problem.linear, VariableCoefficientSpec) or \
        (not grid.periodic and grid.uniform_spacing is None)


def _prepare_shard(grid, sset, problem, scheme, delta_t, off, nloc, pad=0) -> Prepared:
    """timestep.prepare restricted to one slab (per-node rows of the slab only)."""
    nl = _nl_kind(problem)
    bc = _bc_for(grid, sset, problem.boundary)
    frozen = (0, grid.size - 1) if problem.boundary.closed and problem.boundary.freeze_rows else ()
    d1 = None
    if nl == nat.NL_CONVECTIVE:
        d1 = _scaled(derivative_compact(grid, sset, 1), float(problem.nonlinear_scale))
    rng = (off, nloc)
    spec = problem.linear
    warm = None
    if scheme.kind == "linear":
        bank = harvest_compact(grid, sset, spec, delta_t, 1, frozen, node_range=rng, pad=pad)
    elif scheme.kind == "etdrk4":
        # (the half-step set from the same exponential, exactly as timestep.prepare does:
        # a separate harvest at dt / 2 agrees to ~1e-16 only)
        full, half = harvest_compact(grid, sset, spec, delta_t, 4, frozen, node_range=rng, half=True)
        bank = _etdrk4_bank(full, half, delta_t, d1)
    else:
        s = scheme.s
        if s > 5:
            raise InvalidConfig("etd-multistep supports s <= 5 (phi rows up to phi_5)")
        ops = harvest_compact(grid, sset, spec, delta_t, s + 1, frozen, node_range=rng)
        parts = {nat.ROW_W + j: ops.row(j) for j in range(s + 1)}
        if s >= 2:
            full, half = harvest_compact(grid, sset, spec, delta_t, 4, frozen, node_range=rng, half=True)
            warm = _etdrk4_bank(full, half, delta_t, d1)
        if d1 is not None:
            parts[nat.ROW_D1] = d1
        bank = _ops.rows_bank_for(sset, parts, max(parts) + 1)
    return Prepared(sset, scheme.kind, nl, bc, bank, warm, float(delta_t), scheme.s)


def run_virtual_shards(grid: Grid, stencils, problem: SemiLinearProblem, scheme: SchemeConfig,
                       delta_t: float, steps: int, P: int, *, exact: bool = True,
                       ksteps: int | None = None) -> torch.Tensor:
    """P slabs advanced in one process with device-copy halos; returns the
    gathered global solution.  Used to check that sharding is exact."""
    shards: list[ShardedStepper] = []
    for r in range(P):
        shards.append(ShardedStepper(grid, stencils, problem, scheme, delta_t, r, P, None,
                                     exact=exact, ksteps=ksteps))
    for r, s in enumerate(shards):
        s.ex = LocalHalo(shards, r, grid.periodic)
        s.set_initial(problem.initial)
    done = 0
    if scheme.kind == "etd-multistep":
        nw = min(shards[0].warm_up_steps(), steps)
        if nw == 0:
            for s in shards:
                s.warm_up_exchange()
        for i in range(nw):
            for s in shards:
                s.warm_up_exchange()
            for s in shards:
                s.warm_up_compute(i)
        done = shards[0].done
    k = shards[0].plan.ksteps
    while done < steps:
        kk = min(k, steps - done)
        for s in shards:
            s.exchange_phase(kk)
        for s in shards:
            s.compute_phase(kk)
        done += kk
    return torch.cat([s.u for s in shards])


def run_sharded(grid: Grid, stencils, problem: SemiLinearProblem, scheme: SchemeConfig,
                delta_t: float, t_final: float, snapshot_stride: float | None = None, *,
                group=None, exact: bool = True, ksteps: int | None = None,
                transport: str = "nccl", overlap: bool = True, graph: bool | None = None,
                comm: Comm | None = None):
    """``timestep.run`` (timestep.py:255-394) over all ranks of a
    torch.distributed group, one GPU per rank: per-rank harvest, slab stepping
    with halo exchange, snapshots gathered on rank 0.

    transport: "nccl" / "peer" = the library communicator (the group only
    carries its bootstrap bytes), "torch" = torch.distributed point-to-point
    (gloo groups stage the halos through the host); comm = an existing
    communicator of the group to reuse (creating one costs a collective).  Returns a
    SimulationResult on rank 0 and None elsewhere; every rank raises NonFinite
    when the run blows up (rank 0's carries the last finite snapshot, as
    timestep.py:345-348)."""
    dev = nat.device()
    cur = torch.cuda.current_stream(dev)
    if cur.cuda_stream == 0:
        # graphs cannot be captured on the legacy default stream: run on a
        # stream of our own, ordered after the caller's work
        own = torch.cuda.Stream(dev)
        own.wait_stream(cur)
        with torch.cuda.stream(own):
            res = run_sharded(grid, stencils, problem, scheme, delta_t, t_final, snapshot_stride,
                              group=group, exact=exact, ksteps=ksteps, transport=transport,
                              overlap=overlap, graph=graph, comm=comm)
        cur.wait_stream(own)
        return res
    import torch.distributed as dist

    from .timestep import SimulationResult, _steps_for

    multi = dist.is_available() and dist.is_initialized()
    rank = dist.get_rank(group) if multi else 0
    world = dist.get_world_size(group) if multi else 1
    if t_final <= 0 or delta_t <= 0:
        raise InvalidConfig("dt and t_final must be positive")
    steps = _steps_for(t_final, delta_t, "final time")
    if snapshot_stride is None:
        snap_every = steps
    else:
        snap_every = _steps_for(snapshot_stride, delta_t, "snapshot stride")
        if snap_every == 0:
            raise InvalidConfig("snapshot stride must be at least one step")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    torch.cuda.synchronize(dev)
    ev[0].record(cur)
    own_comm = comm is None
    if world == 1:
        ex, comm = None, None
    elif comm is not None:
        ex = CommHalo(comm)
    elif transport == "torch":
        ex = TorchHalo(rank, world, grid.periodic, group)
    else:
        # mailbox capacity (peer): the widest halo any chunk can ask for
        sset = as_stencil_set(grid, stencils)
        reach = max(sset.row, sset.n - 1 - sset.row)
        comm = make_comm(rank, world, grid.periodic, transport, group,
                         max_width=max(16, ksteps or 0) * 8 * max(reach, 1))
        ex = CommHalo(comm)
    st = ShardedStepper(grid, stencils, problem, scheme, delta_t, rank, world, ex, exact=exact,
                        ksteps=ksteps, overlap=overlap, graph=graph)
    ev[1].record(cur)
    st.set_initial(problem.initial)
    N = st.sset.N
    counts = [partition(N, world, r)[1] for r in range(world)]
    nsnap = 1 + (-(-steps // snap_every) if snap_every else 0)
    snaps = torch.empty((nsnap, N), dtype=torch.float64, pin_memory=True) if rank == 0 else None
    gbuf = torch.empty(N, dtype=torch.float64, device=dev) if (rank == 0 and world > 1) else None

    def snapshot(i):
        u = gather_slabs(st, group, comm=comm, counts=counts, out=gbuf)
        if rank == 0:
            snaps[i].copy_(u, non_blocking=True)

    def any_nonfinite() -> bool:
        if world == 1:
            return st.nonfinite()
        bad = st.flag.max().reshape(1).to(torch.int32)
        if comm is not None and comm.transport == "nccl":
            comm.flag_max(bad)
            return bool(bad.item())
        box = [None] * world
        dist.all_gather_object(box, int(bad.item()), group=group)
        return any(box)

    times = [0.0]
    snapshot(0)
    step_ns, done = 0, 0
    try:
        while done < steps:
            k = min(snap_every, steps - done)
            ev[2].record(cur)
            advance_all(st, k)
            ev[3].record(cur)
            cur.synchronize()
            step_ns += int(ev[2].elapsed_time(ev[3]) * 1e6)
            done += k
            if any_nonfinite():
                state = snaps[len(times) - 1].numpy().copy() if rank == 0 else None
                raise NonFinite("time integration blew up", state=state, time=times[-1])
            times.append(done * delta_t)
            snapshot(len(times) - 1)
        cur.synchronize()
    finally:
        harvest_ns = int(ev[0].elapsed_time(ev[1]) * 1e6)
        st._graphs.clear()
        if comm is not None and own_comm:
            comm.close()
    if rank != 0:
        return None
    return SimulationResult(times=np.array(times), snapshots=snaps.numpy(), steps=steps,
                            harvest_ns=harvest_ns, step_ns=step_ns)


def advance_all(st: ShardedStepper, steps: int) -> None:
    """`steps` more steps of a rank: (warm-up,) then chunks of plan.ksteps, one
    halo exchange each."""
    todo = steps
    if st.prep.scheme == "etd-multistep":
        if st.hist is None and st.warm_up_steps() == 0:
            st.warm_up_exchange()             # allocates the (unused) history
        while st._warm_done < st.warm_up_steps() and todo > 0:
            st.warm_up_exchange()
            st.warm_up_compute(st._warm_done)
            todo -= 1
    while todo > 0:
        k = min(st.plan.ksteps, todo)
        st.step_chunk(k, min(st.plan.ksteps, todo - k))
        todo -= k


def gather_slabs(st: ShardedStepper, group=None, *, comm: Comm | None = None, counts=None,
                 out: torch.Tensor | None = None) -> torch.Tensor | None:
    """The global state on rank 0 (None elsewhere).  With an NCCL communicator
    the slabs go straight into `out` on the device; otherwise a padded
    all_gather of the group (through the host on gloo groups)."""
    import torch.distributed as dist
    if st.world == 1:
        return st.u
    if comm is not None and comm.transport == "nccl":
        comm.gather(st.u, counts, out if st.rank == 0 else None, 0)
        return out if st.rank == 0 else None
    m = -(-st.sset.N // st.world)
    host = dist.get_backend(group) == "gloo"
    buf = torch.zeros(m, dtype=torch.float64, device="cpu" if host else st.u.device)
    buf[:st.plan.nloc] = st.u
    parts = [torch.empty_like(buf) for _ in range(st.world)]
    dist.all_gather(parts, buf, group=group)
    if st.rank != 0:
        return None
    return torch.cat([parts[r][:partition(st.sset.N, st.world, r)[1]] for r in range(st.world)])
