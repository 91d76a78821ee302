"""Slab-sharded stepping across GPUs.

One process per GPU.  The grid is cut into contiguous slabs; every rank
harvests what its slab needs without communication (the <= 2n+1 stencil
classes redundantly, or its own nodes' per-node rows) and advances its slab
with the fused step kernels.  The only data exchange is the halo: before a
launch that fuses k steps, each rank sends its first and last
G = k * ext * max(row, n-1-row) nodes to its neighbours (periodic ring or
open chain) with NCCL point-to-point over NVLink.  A deep halo (k > 1)
trades a little redundant edge compute for k times fewer exchanges.

The exchange is an object with one method, ``exchange(u_local, ghosts)``,
so the same driver runs with

  * ``NcclHalo``   -- torch.distributed batch_isend_irecv (NCCL on GPUs,
                      gloo on CPU for the host-side tests);
  * ``LocalHalo``  -- P virtual shards inside one process (device copies),
                      used to check sharded == unsharded on a single GPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _native as nat
from . import _ops
from .errors import InvalidConfig
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


class NcclHalo:
    """Halo exchange over torch.distributed point-to-point (one group call).

    Posting order per rank: send right edge -> right, recv left ghosts <- left,
    send left edge -> left, recv right ghosts <- right.  Messages between a
    pair match in posting order, which also makes the 2-rank periodic ring
    (left == right) come out right.
    """

    def __init__(self, rank: int, world: int, periodic: bool, group=None):
        self.rank, self.world, self.group = rank, world, group
        self.left, self.right = neighbours(rank, world, periodic)

    def exchange(self, u: torch.Tensor, gl: torch.Tensor, gr: torch.Tensor) -> None:
        import torch.distributed as dist
        G = gl.numel()
        if u.numel() < G:
            raise InvalidConfig(f"slab of {u.numel()} nodes is narrower than the halo {G}")
        ops = []
        if self.right is not None:
            ops.append(dist.P2POp(dist.isend, u[u.numel() - G:].contiguous(), self.right, self.group))
        if self.left is not None:
            ops.append(dist.P2POp(dist.irecv, gl, self.left, self.group))
            ops.append(dist.P2POp(dist.isend, u[:G].contiguous(), self.left, self.group))
        if self.right is not None:
            ops.append(dist.P2POp(dist.irecv, gr, self.right, self.group))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()


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
    """Advance one slab of a run (the sharded counterpart of timestep.Stepper)."""

    def __init__(self, grid: Grid, stencils, problem: SemiLinearProblem, scheme: SchemeConfig,
                 delta_t: float, rank: int, world: int, exchanger, *, exact: bool = True,
                 ksteps: int | None = None, tuning=None):
        sset = as_stencil_set(grid, stencils)
        self.sset, self.rank, self.world = sset, rank, world
        self.exact, self.tuning = exact, tuning
        nl = _nl_kind(problem)
        off, nloc = partition(sset.N, world, rank)
        reach = max(sset.row, sset.n - 1 - sset.row)
        ext = _ext(scheme.kind, nl)
        per_node = _is_per_node(grid, problem)
        # periodic per-node linear rows: the shard also harvests its halo
        # nodes' rows (no communication), so k steps fuse per exchange
        pad_ok = per_node and scheme.kind == "linear" and grid.periodic
        if ksteps is None:
            ksteps = max(1, min(16, nloc // (4 * ext * max(reach, 1))))
        if per_node and scheme.kind == "linear" and world > 1 and not pad_ok:
            ksteps = 1                      # non-periodic per-node rows: one step per exchange
        if world == 1:
            ksteps = 1 << 30                # no halo: the library plans the launches
        if per_node and scheme.kind != "linear" and world > 1:
            raise InvalidConfig("sharded ETD schemes need shared or class rows")
        width = ksteps * ext * reach if world > 1 else 0
        if world > 1 and width > nloc:
            raise InvalidConfig(f"slab of {nloc} nodes narrower than the halo {width}")
        self.plan = SlabPlan(off, nloc, width, ksteps)
        pad = ksteps * reach if (pad_ok and world > 1 and ksteps > 1) else 0
        self.prep = _prepare_shard(grid, sset, problem, scheme, delta_t, off, nloc, pad)
        self.ex = exchanger
        dev = nat.device()
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        G = max(width, 1)
        nh = max(scheme.s - 1, 1) if scheme.kind == "etd-multistep" else 1
        self.gl = torch.zeros(G, dtype=torch.float64, device=dev)
        self.gr = torch.zeros(G, dtype=torch.float64, device=dev)
        self.ql = torch.zeros(nh * G, dtype=torch.float64, device=dev)   # [s-1][width] ghosts
        self.qr = torch.zeros(nh * G, dtype=torch.float64, device=dev)
        self.u = None
        self.hist = None
        self.done = 0
        # ping-pong scratch for multi-launch calls (u and the etd2 history)
        self.scratch = torch.empty((nh + 1) * nloc, dtype=torch.float64, device=dev)

    # ---------------------------------------------------------------------
    def set_initial(self, u0_global) -> None:
        """Slice the (closed) global initial data for this slab."""
        u = _ops.dev_f64(u0_global)
        u = close_initial(u, self.sset, self.prep.bc)
        self.u = u[self.plan.off:self.plan.off + self.plan.nloc].contiguous()

    def _width(self, k, scheme=None):
        ext = _ext(scheme or self.prep.scheme, self.prep.nl)
        return k * ext * max(self.sset.row, self.sset.n - 1 - self.sset.row)

    def _nh(self):
        return max(self.prep.s - 1, 1) if self.prep.scheme == "etd-multistep" else 1

    def _halo(self, k):
        if self.world == 1:
            return None
        w = max(self._width(k), 1)
        nh = self._nh()
        return (self.gl[:w], self.gr[:w], self.ql[:nh * w], self.qr[:nh * w], w)

    def _exchange(self, k, hist=False):
        if self.world == 1:
            return
        h = self._halo(k)
        w = h[4]
        if isinstance(self.ex, LocalHalo):
            self.ex.which = "hist" if hist else "u"
        if hist:
            for i in range(self.hist.shape[0]):
                if isinstance(self.ex, LocalHalo):
                    self.ex.which = ("hist", i)
                self.ex.exchange(self.hist[i], h[2][i * w:(i + 1) * w], h[3][i * w:(i + 1) * w])
        else:
            self.ex.exchange(self.u, h[0], h[1])

    def step_chunk(self, k: int) -> None:
        """k <= plan.ksteps steps with one halo exchange.  With LocalHalo the
        caller must run exchange_phase on all shards before compute_phase."""
        self.exchange_phase(k)
        self.compute_phase(k)

    def exchange_phase(self, k: int) -> None:
        p = self.prep
        self._exchange(k)
        if p.scheme == "etd-multistep" and self.hist is not None:
            self._exchange(k, hist=True)

    def _tuning(self, k):
        if self.world == 1:
            return self.tuning              # single shard: library heuristics
        return {**(self.tuning or {}), "ksteps": k}

    def compute_phase(self, k: int) -> None:
        p = self.prep
        kw = dict(bc=p.bc, nl=p.nl, exact=self.exact, tuning=self._tuning(k), flag=self.flag,
                  off=self.plan.off, nloc=self.plan.nloc, halo=self._halo(k),
                  scratch=self.scratch)
        if p.scheme == "linear":
            self.u = _ops.step(nat.SCH_LIN, p.bank, self.u, k, **kw)
        elif p.scheme == "etdrk4":
            self.u = _ops.step(nat.SCH_ETDRK4, p.bank, self.u, k, **kw)
        else:
            if self.hist is None:
                raise InvalidConfig("call warm_up() before multistep chunks")
            self.u, q = _ops.step(nat.SCH_ETD2, p.bank, self.u, k, hist=self.hist,
                                  delta_t=p.delta_t, etd_order=p.s, **kw)
            if p.s > 1:
                self.hist = q
        self.done += k

    # ETD multistep warm-up (timestep.py:375-378): s-1 ETDRK4 steps, each
    # storing N(u) in front of the history; each needs its own halo exchange.
    def warm_up_steps(self) -> int:
        return max(self.prep.s - 1, 0) if self.prep.scheme == "etd-multistep" else 0

    def warm_up_exchange(self) -> None:
        if self.hist is None:
            self.hist = torch.zeros((self._nh(), self.u.numel()), dtype=torch.float64,
                                    device=self.u.device)
        if self.world == 1:
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
        if self.world > 1:
            w = self._width(1, "etdrk4")
            halo = (self.wl, self.wr, self.wl, self.wr, w)
        kw = dict(bc=p.bc, nl=p.nl, exact=self.exact, tuning=self._tuning(1), flag=self.flag,
                  off=self.plan.off, nloc=self.plan.nloc, halo=halo)
        self.u = _ops.step(nat.SCH_ETDRK4, p.warm, self.u, 1, nl0_out=self.hist[0], **kw)
        self.done += 1

    def nonfinite(self) -> bool:
        return bool(self.flag.item())


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
        full = harvest_compact(grid, sset, spec, delta_t, 4, frozen, node_range=rng)
        half = harvest_compact(grid, sset, spec, delta_t / 2, 2, frozen, node_range=rng)
        bank = _etdrk4_bank(full, half, delta_t, d1)
    else:
        s = scheme.s
        if s > 5:
            raise InvalidConfig("etd-multistep supports s <= 5 (phi rows up to phi_5)")
        ops = harvest_compact(grid, sset, spec, delta_t, s + 1, frozen, node_range=rng)
        parts = {nat.ROW_W + j: ops.row(j) for j in range(s + 1)}
        if s >= 2:
            full = harvest_compact(grid, sset, spec, delta_t, 4, frozen, node_range=rng)
            half = harvest_compact(grid, sset, spec, delta_t / 2, 2, frozen, node_range=rng)
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
                delta_t: float, t_final: float, *, group=None, exact: bool = True,
                ksteps: int | None = None):
    """``timestep.run`` over all ranks of a torch.distributed group (one GPU per
    rank): per-rank harvest, slab stepping with NCCL halo exchange, and the
    final state gathered on rank 0.  Returns a SimulationResult (snapshots:
    initial and final state) on rank 0 and None elsewhere."""
    import time

    import numpy as np
    import torch.distributed as dist

    from .timestep import SimulationResult, _steps_for

    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if t_final <= 0 or delta_t <= 0:
        raise InvalidConfig("dt and t_final must be positive")
    steps = _steps_for(t_final, delta_t, "final time")
    dev = nat.device()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter_ns()
    st = ShardedStepper(grid, stencils, problem, scheme, delta_t, rank, world,
                        NcclHalo(rank, world, grid.periodic, group), exact=exact, ksteps=ksteps)
    torch.cuda.synchronize(dev)
    harvest_ns = time.perf_counter_ns() - t0
    st.set_initial(problem.initial)
    t0 = time.perf_counter_ns()
    advance_all(st, steps)
    torch.cuda.synchronize(dev)
    step_ns = time.perf_counter_ns() - t0
    u = gather_slabs(st, group)
    if world > 1:
        bad = torch.tensor([int(st.nonfinite())], device=dev)
        dist.all_reduce(bad, group=group)
        nonfinite = bool(bad.item())
    else:
        nonfinite = st.nonfinite()
    if rank != 0:
        return None
    u0 = np.asarray(problem.initial.cpu() if isinstance(problem.initial, torch.Tensor)
                    else problem.initial, dtype=np.float64)
    if nonfinite:
        from .errors import NonFinite
        raise NonFinite("time integration blew up", state=u0, time=0.0)
    return SimulationResult(times=np.array([0.0, steps * delta_t]),
                            snapshots=np.stack([u0, _ops.to_host(u)]), steps=steps,
                            harvest_ns=harvest_ns, step_ns=step_ns)


def advance_all(st: ShardedStepper, steps: int) -> None:
    """All of a rank's steps: (warm-up,) then chunks of plan.ksteps, one halo
    exchange each."""
    done = 0
    if st.prep.scheme == "etd-multistep" and st.hist is None:
        nw = min(st.warm_up_steps(), steps)
        if nw == 0:
            st.warm_up_exchange()             # allocates the (unused) history
        for i in range(nw):
            st.warm_up_exchange()
            st.warm_up_compute(i)
        done = st.done
    while done < steps:
        k = min(st.plan.ksteps, steps - done)
        st.step_chunk(k)
        done += k


def gather_slabs(st: ShardedStepper, group=None) -> torch.Tensor | None:
    """Concatenate the slabs on rank 0 (padded all_gather: slab sizes differ by <= 1)."""
    import torch.distributed as dist
    if st.world == 1:
        return st.u
    m = -(-st.sset.N // st.world)
    buf = torch.zeros(m, dtype=torch.float64, device=st.u.device)
    buf[:st.plan.nloc] = st.u
    parts = [torch.empty_like(buf) for _ in range(st.world)]
    dist.all_gather(parts, buf, group=group)
    if st.rank != 0:
        return None
    return torch.cat([parts[r][:partition(st.sset.N, st.world, r)[1]] for r in range(st.world)])
