"""Sharding: host-side halo exchange over a real 2-rank gloo group (CPU), and
on the GPU, P virtual shards in one process against the unsharded kernels."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_15964_b200.distributed import NcclHalo, neighbours, partition


def test_partition_covers_grid():
    for N in (7, 64, 1000, 1 << 20):
        for world in (1, 2, 3, 4, 8):
            parts = [partition(N, world, r) for r in range(world)]
            assert parts[0][0] == 0
            for (o1, n1), (o2, _) in zip(parts, parts[1:]):
                assert o1 + n1 == o2
            assert sum(n for _, n in parts) == N
            assert max(n for _, n in parts) - min(n for _, n in parts) <= 1


def test_neighbours():
    assert neighbours(0, 1, True) == (None, None)
    assert neighbours(0, 4, True) == (3, 1)
    assert neighbours(0, 4, False) == (None, 1)
    assert neighbours(3, 4, False) == (2, None)
    assert neighbours(1, 2, True) == (0, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, periodic, N, G, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        u_glob = torch.arange(N, dtype=torch.float64) * 1.5 + 0.25
        off, nloc = partition(N, world, rank)
        u = u_glob[off:off + nloc].clone()
        gl = torch.full((G,), -1.0, dtype=torch.float64)
        gr = torch.full((G,), -1.0, dtype=torch.float64)
        NcclHalo(rank, world, periodic).exchange(u, gl, gr)
        left, right = neighbours(rank, world, periodic)
        idx_l = [(off - G + j) % N for j in range(G)]
        idx_r = [(off + nloc + j) % N for j in range(G)]
        ok_l = left is None or torch.equal(gl, u_glob[idx_l])
        ok_r = right is None or torch.equal(gr, u_glob[idx_r])
        out_q.put((rank, bool(ok_l), bool(ok_r), gl.tolist()[:2], gr.tolist()[:2]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,periodic", [(2, True), (2, False), (3, True), (4, False)])
def test_halo_exchange_gloo(world, periodic):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, periodic, 37, 5, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_l, ok_r, a, b in res:
        assert ok_l and ok_r, (rank, a, b)


# ------------------------------------------------------------------ GPU
def _cases():
    import paper_2603_15964_b200 as lx
    from paper_2603_15964_b200 import configs
    out = []
    w = configs.c1(N=1000)
    g = lx.make_periodic_grid(w.N, w.x_min, w.x_max)
    st = lx.select_stencils(g, w.n, lx.StencilPolicy.ONE_SIDED_UPWIND)
    out.append(("c1-linear", g, st, lx.SemiLinearProblem(lx.LinearOperatorSpec(w.terms), None,
                w.u0, lx.Boundary.periodic(), "none"), lx.SchemeConfig("linear"), w.delta_t, 40))
    w = configs.c5(N=3000)
    c, nu = w.coef
    g = lx.make_periodic_grid(w.N, 0.0, 1.0)
    st = lx.select_stencils(g, w.n, lx.StencilPolicy.CENTERED)
    out.append(("c5-pernode", g, st, lx.SemiLinearProblem(
        lx.VariableCoefficientSpec((1, 2), np.stack([-c, nu], 1)), None, w.u0,
        lx.Boundary.periodic(), "none"), lx.SchemeConfig("linear"), w.delta_t, 15))
    out.append(("c5-rowscaled", g, st, lx.SemiLinearProblem(
        lx.VariableCoefficientSpec((1, 2), np.stack([-c, nu], 1), row_scaled=True), None, w.u0,
        lx.Boundary.periodic(), "none"), lx.SchemeConfig("linear"), w.delta_t, 15))
    w = configs.c4(N=4000)
    g = lx.make_uniform_grid(w.N, -1.0, 1.0)
    st = lx.select_stencils(g, w.n, lx.StencilPolicy.CENTERED)
    out.append(("c4-neumann", g, st, lx.SemiLinearProblem(lx.LinearOperatorSpec(w.terms), None,
                w.u0, lx.Boundary.neumann(), "cubic"), lx.SchemeConfig("etdrk4"), w.delta_t, 9))
    w = configs.c3(N=4096)
    g = lx.make_periodic_grid(w.N, w.x_min, w.x_max)
    st = lx.select_stencils(g, w.n, lx.StencilPolicy.CENTERED)
    out.append(("c3-kdv", g, st, lx.SemiLinearProblem(lx.LinearOperatorSpec(w.terms), None,
                w.u0, lx.Boundary.periodic(), "convective", nonlinear_scale=6.0),
                lx.SchemeConfig("etdrk4"), w.delta_t, 7))
    w = configs.c2(N=4096)
    g = lx.make_periodic_grid(w.N, w.x_min, w.x_max)
    st = lx.select_stencils(g, w.n, lx.StencilPolicy.CENTERED)
    out.append(("c2-etd2", g, st, lx.SemiLinearProblem(lx.LinearOperatorSpec(w.terms), None,
                w.u0, lx.Boundary.periodic(), "convective"),
                lx.SchemeConfig("etd-multistep", s=2), w.delta_t, 11))
    for s in (1, 3, 5):
        out.append((f"c2-etd{s}", g, st, lx.SemiLinearProblem(
            lx.LinearOperatorSpec(w.terms), None, w.u0, lx.Boundary.periodic(), "convective"),
            lx.SchemeConfig("etd-multistep", s=s), 0.25 * w.delta_t, 9))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 3, 8])
def test_virtual_shards_bitwise(P):
    from paper_2603_15964_b200 import _ops
    from paper_2603_15964_b200.distributed import run_virtual_shards
    from paper_2603_15964_b200.timestep import Stepper, prepare
    for name, g, st, prob, scheme, dt, steps in _cases():
        ref = Stepper(prepare(g, st, prob, scheme, dt), _ops.dev_f64(prob.initial))
        ref.advance(steps)
        for k in (None, 1):
            u = run_virtual_shards(g, st, prob, scheme, dt, steps, P, ksteps=k)
            assert torch.equal(u, ref.u), (name, P, k, float((u - ref.u).abs().max()))


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 3, 5])
def test_virtual_shards_pernode_slabs_bitwise(P):
    """Per-node linear slabs wide enough for the persistent TMA kernels (ghosts stored
    right around the slab, 24 steps per exchange; odd-sized slabs take the
    register-blocked kernel): bit-identical to the unsharded steps, exact and
    fused arithmetic alike (the per-node kernels compute each node the same way
    whatever the tiling)."""
    import paper_2603_15964_b200 as lx
    from paper_2603_15964_b200 import _ops, configs
    from paper_2603_15964_b200.distributed import ShardedStepper, run_virtual_shards
    from paper_2603_15964_b200.timestep import Stepper, prepare
    w = configs.c5(N=16384 + 2 * P)
    c, nu = w.coef
    g = lx.make_periodic_grid(w.N, 0.0, 1.0)
    st = lx.select_stencils(g, w.n, lx.StencilPolicy.CENTERED)
    prob = lx.SemiLinearProblem(lx.VariableCoefficientSpec((1, 2), np.stack([-c, nu], 1)), None,
                                w.u0, lx.Boundary.periodic(), "none")
    scheme = lx.SchemeConfig("linear")
    # one harvest kernel for every batch size (the default picks the constant-table
    # kernel for batches >= 4096 and the per-item kernel below: rows equal to ~1e-16,
    # not bit for bit), so that only the stepping is compared
    lx._native.set_harvest_method("mvitem")
    try:
        s0 = ShardedStepper(g, st, prob, scheme, w.delta_t, 0, P, None)
        k0 = 24 if s0.plan.nloc >= 4096 else 16
        assert s0.plan.ksteps == k0 and s0.plan.width == k0 * 6
        for exact in (True, False):
            ref = Stepper(prepare(g, st, prob, scheme, w.delta_t), _ops.dev_f64(prob.initial),
                          exact=exact)
            ref.advance(61)
            u = run_virtual_shards(g, st, prob, scheme, w.delta_t, 61, P, exact=exact)
            if exact:
                assert torch.equal(u, ref.u), (P, float((u - ref.u).abs().max()))
            else:
                assert float((u - ref.u).norm() / ref.u.norm()) < 1e-13
    finally:
        lx._native.set_harvest_method("multiply")


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["nccl", "peer"])
def test_comm_self_exchange(transport):
    """A periodic 1-rank ring exchanges with itself through the library
    communicator: the real NCCL group / peer-store path on one GPU."""
    from paper_2603_15964_b200.distributed import Comm
    if transport == "nccl":
        c = Comm(0, 1, True, "nccl", unique_id=Comm.unique_id())
    else:
        c = Comm(0, 1, True, "peer", max_width=64)
        c.connect([c.export()])
    assert (c.left, c.right) == (0, 0)
    dev = torch.device("cuda")
    nloc, W = 1000, 37
    f = [torch.arange(nloc, dtype=torch.float64, device=dev) * (i + 1) + 0.5 for i in range(3)]
    for rep in range(5):                       # several exchanges: both mailbox halves
        gl = [torch.full((W,), -1.0, dtype=torch.float64, device=dev) for _ in f]
        gr = [torch.full((W,), -1.0, dtype=torch.float64, device=dev) for _ in f]
        c.exchange(f, W, gl, gr)
        torch.cuda.synchronize()
        for i in range(3):
            assert torch.equal(gl[i], f[i][nloc - W:]) and torch.equal(gr[i], f[i][:W]), (rep, i)
        f = [x + 1.0 for x in f]
    if transport == "nccl":
        out = torch.empty(nloc, dtype=torch.float64, device=dev)
        c.gather(f[0], [nloc], out, 0)
        flag = torch.tensor([0, 1, 0], dtype=torch.int32, device=dev)
        c.flag_max(flag)
        torch.cuda.synchronize()
        assert torch.equal(out, f[0]) and flag.tolist() == [0, 1, 0]
    # a chain end has no neighbours: nothing moves
    e = Comm(0, 1, False, "peer", max_width=8)
    e.connect(None)
    assert (e.left, e.right) == (None, None)
    e.close()
    c.close()


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["nccl", "peer"])
def test_self_ring_stepper_bitwise(transport):
    """ShardedStepper on a 1-rank periodic ring with forced halos through the
    communicator -- interior / edge split on two streams, chunks replayed from
    CUDA graphs on NCCL -- is bit-identical to the unsharded stepper."""
    from paper_2603_15964_b200 import _ops
    from paper_2603_15964_b200.distributed import Comm, CommHalo, ShardedStepper, advance_all
    from paper_2603_15964_b200.timestep import Stepper, prepare
    if transport == "nccl":
        c = Comm(0, 1, True, "nccl", unique_id=Comm.unique_id())
    else:
        c = Comm(0, 1, True, "peer", max_width=4096)
        c.connect([c.export()])
    try:
        for name, g, st, prob, scheme, dt, steps in _cases():
            if not g.periodic:
                continue
            ref = Stepper(prepare(g, st, prob, scheme, dt), _ops.dev_f64(prob.initial))
            ref.advance(5 * steps + 3)
            for k in (None, 2):
                s = ShardedStepper(g, st, prob, scheme, dt, 0, 1, CommHalo(c), ksteps=k,
                                   force_halo=True)
                assert s.sharded and s.plan.width > 0
                if name in ("c1-linear", "c3-kdv"):
                    # shared rows: interior / edge split; on the peer transport the
                    # edge launches store the next halo into the mailboxes themselves
                    assert s.overlap and s.fused == (transport == "peer")
                s.set_initial(prob.initial)
                own = torch.cuda.Stream()               # graphs need a non-default stream
                own.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(own):
                    advance_all(s, 5 * steps + 3)
                torch.cuda.synchronize()
                assert torch.equal(s.u, ref.u), (name, k, float((s.u - ref.u).abs().max()))
                if transport == "nccl" and k == 2:
                    assert len(s._graphs) == 2, name           # both ping-pong directions replayed
                assert not s.nonfinite()
                s._graphs.clear()
    finally:
        c.close()


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["nccl", "peer"])
def test_chunk_driver_random_shapes_bitwise(transport):
    """lmep_comm_chunk over seeded random shapes (grid size, stencil width, scheme,
    steps per exchange, step counts that leave a shorter last chunk, slabs both
    wider and narrower than three halos): a 1-rank ring through the communicator
    against the unsharded stepper, bit for bit."""
    import paper_2603_15964_b200 as lx
    from paper_2603_15964_b200 import _ops
    from paper_2603_15964_b200.distributed import Comm, CommHalo, ShardedStepper, advance_all
    from paper_2603_15964_b200.timestep import Stepper, prepare
    if transport == "nccl":
        c = Comm(0, 1, True, "nccl", unique_id=Comm.unique_id())
    else:
        c = Comm(0, 1, True, "peer", max_width=2048)
        c.connect([c.export()])
    rng = np.random.default_rng(20260315)
    own = torch.cuda.Stream()
    try:
        for case in range(14):
            n = int(rng.choice([7, 9, 11, 13]))
            kind = ["linear", "cubic", "convective"][case % 3]
            k = int(rng.integers(1, 7))
            reach = (n - 1) // 2
            ext = {"linear": 1, "cubic": 4, "convective": 8}[kind]
            w = k * ext * reach
            # slabs from just over one halo (unsplit) to many halos (interior + strips)
            N = int(w * rng.choice([1.5, 2.9, 3.0, 3.1, 7.3, 40.0])) + int(rng.integers(0, 5)) + 4 * n
            steps = int(rng.integers(1, 4)) * k + int(rng.integers(0, k))
            g = lx.make_periodic_grid(N, 0.0, 2 * math.pi)
            st = lx.select_stencils(g, n, lx.StencilPolicy.CENTERED)
            u0 = np.sin(g.nodes) + 0.2 * np.cos(3 * g.nodes + case)
            h = 2 * math.pi / N
            if kind == "linear":
                prob = lx.SemiLinearProblem(lx.LinearOperatorSpec(((1, -1.0), (2, 0.05))), None, u0,
                                            lx.Boundary.periodic(), "none")
                scheme, dt = lx.SchemeConfig("linear"), 0.4 * h
            else:
                prob = lx.SemiLinearProblem(lx.LinearOperatorSpec(((2, 0.02),)), None, u0,
                                            lx.Boundary.periodic(), kind)
                scheme, dt = lx.SchemeConfig("etdrk4"), 0.3 * h * h / 0.02
            ref = Stepper(prepare(g, st, prob, scheme, dt), _ops.dev_f64(u0))
            ref.advance(steps)
            s = ShardedStepper(g, st, prob, scheme, dt, 0, 1, CommHalo(c), ksteps=k, force_halo=True)
            assert s.overlap and s.plan.width == w
            s.set_initial(u0)
            own.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(own):
                advance_all(s, steps)
            torch.cuda.synchronize()
            assert torch.equal(s.u, ref.u), (case, kind, n, N, k, steps, float((s.u - ref.u).abs().max()))
            assert not s.nonfinite()
            s._graphs.clear()
    finally:
        c.close()


def _rank_main(rank, world, port, transport, q):
    """One rank of the 2-process runs below; both ranks drive cuda:0."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ.setdefault("LMEP_PEER_TIMEOUT_S", "60")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2603_15964_b200 as lx
        from paper_2603_15964_b200.distributed import run_sharded
        from paper_2603_15964_b200.errors import NonFinite
        torch.cuda.set_device(0)
        res = {}
        # periodic runs share one communicator (the ring); the open chain makes its own
        ring = None
        if transport == "peer":
            from paper_2603_15964_b200.distributed import make_comm
            ring = make_comm(rank, world, True, "peer", max_width=16 * 8 * 6)
        for name, g, st, prob, scheme, dt, steps in _cases():
            if name in ("c2-etd1", "c2-etd5", "c5-rowscaled"):
                continue
            T = (3 * steps + 1) * dt
            stride = steps * dt
            a = run_sharded(g, st, prob, scheme, dt, T, stride, transport=transport,
                            comm=ring if g.periodic else None)
            if rank == 0:
                b = lx.run(g, st, prob, scheme, dt, T, stride)
                res[name] = (bool(np.array_equal(a.snapshots, b.snapshots)),
                             bool(np.array_equal(a.times, b.times)), a.steps == b.steps,
                             a.harvest_ns > 0 and a.step_ns > 0)
        # blow-up: every rank raises; rank 0 carries the last finite snapshot, as run()
        name, g, st, prob, scheme, dt, steps = [c for c in _cases() if c[0] == "c2-etd2"][0]
        bad = 400.0 * dt
        try:
            run_sharded(g, st, prob, scheme, bad, 40 * bad, 10 * bad, transport=transport)
            res["blowup"] = "no error"
        except NonFinite as e:
            if rank == 0:
                try:
                    lx.run(g, st, prob, scheme, bad, 40 * bad, 10 * bad)
                    res["blowup"] = "run() did not raise"
                except NonFinite as e2:
                    res["blowup"] = (bool(np.array_equal(e.state, e2.state)), e.time == e2.time)
            else:
                res["blowup"] = (e.state is None,)
        if ring is not None:
            ring.close()
        q.put((rank, res))
    except Exception as e:                                      # noqa: BLE001
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,transport", [(2, "peer"), (2, "torch"), (3, "peer")])
def test_run_sharded_two_processes(world, transport):
    """run_sharded over two or three processes (all on cuda:0; the peer transport
    moves the halos through CUDA-IPC mailboxes, "torch" stages them through a gloo
    group) reproduces run() bit for bit: every snapshot, times, step count, and
    the NonFinite state of a blown-up run.  Three ranks give every rank two
    different neighbours on the ring and a middle rank on the open chain."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, transport, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        out = dict(q.get(timeout=420) for _ in range(world))
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for r in range(world):
        assert "error" not in out[r], out[r]["error"]
    r0 = out[0]
    for name in ("c1-linear", "c5-pernode", "c4-neumann", "c3-kdv", "c2-etd2", "c2-etd3"):
        assert r0[name] == (True, True, True, True), (name, r0[name])
    assert r0["blowup"] == (True, True), r0["blowup"]
    for r in range(1, world):
        assert out[r]["blowup"] == (True,)


@pytest.mark.gpu
def test_run_sharded_single_rank_nccl():
    """The NCCL entry point end to end on a 1-rank group matches run()."""
    import paper_2603_15964_b200 as lx
    from paper_2603_15964_b200 import configs
    from paper_2603_15964_b200.distributed import run_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        w = configs.c5(N=2048, steps=20)
        c, nu = w.coef
        g = lx.make_periodic_grid(w.N, 0.0, 1.0)
        st = lx.select_stencils(g, w.n, lx.StencilPolicy.CENTERED)
        prob = lx.SemiLinearProblem(lx.VariableCoefficientSpec((1, 2), np.stack([-c, nu], 1)),
                                    None, w.u0, lx.Boundary.periodic(), "none")
        T = 20 * w.delta_t
        a = run_sharded(g, st, prob, lx.SchemeConfig("linear"), w.delta_t, T)
        b = lx.run(g, st, prob, lx.SchemeConfig("linear"), w.delta_t, T)
        assert np.array_equal(a.u_final, b.u_final)
    finally:
        dist.destroy_process_group()
