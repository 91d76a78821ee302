"""Streamed linear steps (lmep_lin_stream, csrc/step_stream.cu): the k-step
launches of timestep.run's linear scheme (timestep.py:255-394,
kernels.py:33-43) issued in a skewed space-time order behind a harvest that is
still running.  Every test compares with the level-by-level order
(lmep_step_linear) bit for bit.
"""

import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lx():
    import paper_2603_15964_b200 as m
    m._native.device()
    return m


def _stream_run(lay, W, u, steps, exact, bounds, host=False, tuning=None):
    """Steps through lmep_lin_stream with the rows and the initial values landing
    prefix by prefix: what has not landed yet is NaN when each call is issued, so
    a launch that read past its frontier would poison the result."""
    from paper_2603_15964_b200 import _native as nat, _ops
    L = nat.lib()
    N = lay.N
    Wl = torch.full_like(W, float("nan"))
    ul = torch.full_like(u, float("nan"))
    out, scr = torch.empty_like(u), torch.empty_like(u)
    flag = torch.ones(1, dtype=torch.int32, device="cuda")
    hout = torch.full((N,), float("nan"), dtype=torch.float64).pin_memory() if host else None
    cp = _ops.copy_stream(1)
    g = _ops.c_grid(lay, 0, None)
    w = nat.LmepWeights(nat.W_PERNODE, 1, 0, 0, None, None, Wl.data_ptr(), 0)
    tun = _ops._tuning(tuning)
    h = C.c_void_p()
    cur = torch.cuda.current_stream()
    cp.wait_stream(cur)
    st = L.lmep_lin_stream_begin(C.byref(g), C.byref(w), ul.data_ptr(), out.data_ptr(), scr.data_ptr(),
                                 steps, nat.FLAG_EXACT if exact else 0,
                                 C.byref(tun) if tun is not None else None, flag.data_ptr(),
                                 hout.data_ptr() if host else None, cp.cuda_stream, cur.cuda_stream,
                                 C.byref(h))
    if st == nat.LMEP_INVALID_CONFIG:
        return None
    nat.check(st, "lmep_lin_stream_begin")
    a = 0
    for b in bounds:
        Wl[:, :, a:b] = W[:, :, a:b]
        ul[a:b] = u[a:b]
        nat.check(L.lmep_lin_stream_advance(h, b, cur.cuda_stream), "lmep_lin_stream_advance")
        a = b
    n = C.c_int64()
    nat.check(L.lmep_lin_stream_end(h, C.byref(n)), "lmep_lin_stream_end")
    torch.cuda.synchronize()
    return out, (hout.numpy() if host else None), int(flag.item()), n.value


def _case(N, n, row, seed):
    from paper_2603_15964_b200 import _native as nat, _ops
    from paper_2603_15964_b200.grid import StencilSet
    rng = np.random.default_rng(seed)
    lay = StencilSet(N, n, row, True)
    W = torch.as_tensor(rng.standard_normal((1, n, N)) / n, device="cuda")
    u = torch.as_tensor(rng.standard_normal(N), device="cuda")
    return lay, W, u, _ops.CompactRows(lay, nat.W_PERNODE, pernode=W)


@pytest.mark.parametrize("n,row", [(13, 6), (7, 3), (7, 0)])
@pytest.mark.parametrize("exact", [True, False])
def test_lin_stream_bitwise_poisoned(lx, n, row, exact):
    """Prefixes of every kind -- tile-aligned, odd sizes, a first slice too small
    for any launch, single-shot -- over 1 .. 8 launch levels."""
    from paper_2603_15964_b200 import _native as nat, _ops
    N = 1536 * 61 + 38
    lay, W, u, rows = _case(N, n, row, 11)
    rng = np.random.default_rng(5)
    for steps in (1, 25, 26, 60, 200):
        ref = _ops.step(nat.SCH_LIN, rows, u, steps, exact=exact)
        cuts = [
            [N],
            [100, N],
            [1024 * 7, 1024 * 30, 1024 * 31, 1024 * 70, N],
            sorted(set(int(x) for x in rng.integers(1, N, 9))) + [N],
            list(range(4000, N, 4000)) + [N],
        ]
        for bounds in cuts:
            got = _stream_run(lay, W, u, steps, exact, bounds, host=True)
            if steps == 1:
                assert got is None           # one step per launch: not the blocked plan
                continue
            assert got is not None
            out, hout, flag, launches = got
            assert flag == 0
            assert torch.equal(out, ref), (steps, bounds[:3])
            assert np.array_equal(hout, ref.cpu().numpy()), (steps, bounds[:3])


def test_lin_stream_levels_overlap(lx):
    """With several slices the levels really interleave: more launches than
    levels, the same bits; a non-finite input raises the flag."""
    from paper_2603_15964_b200 import _native as nat, _ops
    N = 1 << 19
    lay, W, u, rows = _case(N, 13, 6, 2)
    ref = _ops.step(nat.SCH_LIN, rows, u, 100, exact=False)
    one = _stream_run(lay, W, u, 100, False, [N])
    many = _stream_run(lay, W, u, 100, False, [N // 8, N // 4, N // 2, 3 * N // 4, N])
    assert one[3] == 4 and many[3] > 4 * 4
    assert torch.equal(one[0], ref) and torch.equal(many[0], ref)
    u2 = u.clone()
    u2[N // 3] = float("inf")
    bad = _stream_run(lay, W, u2, 100, False, [N // 2, N])
    assert bad[2] == 1


def test_lin_stream_declines_other_plans(lx):
    """Grids the persistent per-node plan does not cover (odd N, smaller than one
    span) are declined with LMEP_INVALID_CONFIG: the caller steps afterwards."""
    for N in (1000, 1536 * 9 + 1):
        lay, W, u, _ = _case(N, 13, 6, 1)
        assert _stream_run(lay, W, u, 30, True, [N]) is None


@pytest.mark.parametrize("src", ["numpy", "pinned"])
def test_run_streamed_matches_phases(lx, src):
    """run() from host arrays as one pipeline (stream=True, the default) against
    the phase-by-phase order (stream=False): the same snapshots bit for bit (on
    config 5's fields every harvest slice balances to the same exponents), with
    and without a snapshot stride; harvest_ns / step_ns are reported."""
    from paper_2603_15964_b200 import configs
    N = 1 << 20
    w5 = configs.c5(N=N, steps=1)
    c, nu = w5.coef
    g = lx.make_periodic_grid(N, 0.0, 1.0)
    st = lx.select_stencils(g, w5.n, lx.StencilPolicy.CENTERED)
    coef = np.stack([-c, nu], 1)
    u0 = np.array(w5.u0)
    if src == "pinned":
        hc, hu = torch.from_numpy(coef).pin_memory(), torch.from_numpy(u0).pin_memory()
    else:
        hc, hu = coef, u0
    prob = lx.SemiLinearProblem(lx.VariableCoefficientSpec((1, 2), hc), None, hu,
                                lx.Boundary.periodic(), "none")
    sch = lx.SchemeConfig("linear")
    for exact in (True, False):
        for stride in (None, 40 * w5.delta_t):
            a = lx.run(g, st, prob, sch, w5.delta_t, 90 * w5.delta_t, stride, exact=exact)
            b = lx.run(g, st, prob, sch, w5.delta_t, 90 * w5.delta_t, stride, exact=exact, stream=False)
            assert a.snapshots.shape == b.snapshots.shape
            assert np.array_equal(a.snapshots[0], u0)
            assert np.array_equal(a.snapshots, b.snapshots), (exact, stride)
            assert np.array_equal(a.times, b.times)
            assert a.harvest_ns > 0 and a.step_ns > 0


def test_pipelined_harvest_any_slicing_bitwise(lx, monkeypatch):
    """The constant-table harvest keeps the first slice's prepared tables for the
    later slices (lmep_harvest_reuse_prep), so host coefficients harvested slice
    by slice give the rows of the one-launch harvest bit for bit whatever the
    slice boundaries -- also on fields whose slices would balance differently
    on their own first items (a coefficient jump of 1e4 across the grid)."""
    from paper_2603_15964_b200 import configs, harvest as hv
    N = 1 << 19
    w5 = configs.c5(N=N, steps=1)
    g = lx.make_periodic_grid(N, 0.0, 1.0)
    st = lx.select_stencils(g, w5.n, lx.StencilPolicy.CENTERED)
    x = np.asarray(g.nodes)
    nu = np.where(x < 0.37, 1e-4, 1.0) * (1.0 + 0.3 * np.sin(2 * np.pi * x))
    c = 0.5 + 0.4 * np.cos(2 * np.pi * x)
    dt = 0.4 * w5.h ** 2 / nu.max()
    coef = np.stack([-c, nu], 1)
    ref = hv.harvest_compact(g, st, lx.VariableCoefficientSpec((1, 2), torch.as_tensor(coef, device="cuda")),
                             dt, 1)
    for bounds in ([(0, N)], [(0, 8192), (8192, N)],
                   [(0, 150 * 1024), (150 * 1024, 333 * 1024), (333 * 1024, N)]):
        monkeypatch.setattr(hv, "_pipeline_bounds", lambda n, b=bounds: list(b))
        got = hv.harvest_compact(g, st, lx.VariableCoefficientSpec((1, 2), coef), dt, 1)
        assert torch.equal(got.pernode, ref.pernode), bounds


def test_run_streamed_fallbacks(lx):
    """run(stream=True) where the pipeline does not apply -- a one-step first chunk
    (the library declines the plan) and a grid too small for a pipelined harvest
    (the initial state goes up in one copy) -- gives the phase-by-phase result."""
    from paper_2603_15964_b200 import configs
    sch = lx.SchemeConfig("linear")
    for N, steps, stride in ((1 << 19, 5, 1), (1 << 14, 30, 10)):
        w5 = configs.c5(N=N, steps=1)
        c, nu = w5.coef
        g = lx.make_periodic_grid(N, 0.0, 1.0)
        st = lx.select_stencils(g, w5.n, lx.StencilPolicy.CENTERED)
        prob = lx.SemiLinearProblem(lx.VariableCoefficientSpec((1, 2), np.stack([-c, nu], 1)), None,
                                    np.array(w5.u0), lx.Boundary.periodic(), "none")
        a = lx.run(g, st, prob, sch, w5.delta_t, steps * w5.delta_t, stride * w5.delta_t)
        b = lx.run(g, st, prob, sch, w5.delta_t, steps * w5.delta_t, stride * w5.delta_t, stream=False)
        assert a.snapshots.shape == b.snapshots.shape == (1 + steps // stride, N)
        assert np.array_equal(a.snapshots, b.snapshots), (N, steps)


def test_run_streamed_with_reaction_and_slice_upload(lx):
    """A streamed run whose operator carries a reaction term (no eager prefix: the
    reaction table rides with the slices through the torch copy path) against the
    phase-by-phase order, and lmep_upload_slice on its own: coefficients and
    initial state land behind their events, the snapshot copy comes back."""
    from paper_2603_15964_b200 import configs, _native as nat, _ops
    N = 1 << 19
    w5 = configs.c5(N=N, steps=1)
    c, nu = w5.coef
    g = lx.make_periodic_grid(N, 0.0, 1.0)
    st = lx.select_stencils(g, w5.n, lx.StencilPolicy.CENTERED)
    x = np.asarray(g.nodes)
    spec = lx.VariableCoefficientSpec((1, 2), np.stack([-c, nu], 1), reaction=-0.5 * (1.0 + np.sin(2 * np.pi * x)))
    prob = lx.SemiLinearProblem(spec, None, np.array(w5.u0), lx.Boundary.periodic(), "none")
    sch = lx.SchemeConfig("linear")
    a = lx.run(g, st, prob, sch, w5.delta_t, 60 * w5.delta_t)
    b = lx.run(g, st, prob, sch, w5.delta_t, 60 * w5.delta_t, stream=False)
    assert np.array_equal(a.snapshots[0], np.array(w5.u0))
    assert np.array_equal(a.snapshots, b.snapshots)

    L = nat.lib()
    M, K = 3000, 2
    hc = torch.arange(M * K, dtype=torch.float64).reshape(M, K).pin_memory()
    hu = (torch.arange(M, dtype=torch.float64) * 0.5).pin_memory()
    snap = torch.full((M,), float("nan"), dtype=torch.float64).pin_memory()
    dc = torch.full((M, K), float("nan"), dtype=torch.float64, device="cuda")
    du = torch.full((M,), float("nan"), dtype=torch.float64, device="cuda")
    up, down = _ops.copy_stream(0), _ops.copy_stream(3)
    torch.cuda.synchronize()
    ec, ev = C.c_void_p(), C.c_void_p()
    assert L.lmep_event_create(C.byref(ec)) == nat.LMEP_OK and L.lmep_event_create(C.byref(ev)) == nat.LMEP_OK
    a0, b0 = 1000, 2500
    st_ = L.lmep_upload_slice(dc.data_ptr() + a0 * K * 8, hc.data_ptr() + a0 * K * 8, (b0 - a0) * K * 8,
                              du.data_ptr() + a0 * 8, hu.data_ptr() + a0 * 8, snap.data_ptr() + a0 * 8,
                              (b0 - a0) * 8, up.cuda_stream, down.cuda_stream, ec, ev)
    assert st_ == nat.LMEP_OK
    cur = torch.cuda.current_stream()
    _ops.stream_wait(cur, ev)
    got_c, got_u = dc.clone(), du.clone()          # (behind the event on the current stream)
    torch.cuda.synchronize()
    assert torch.equal(got_c[a0:b0].cpu(), hc[a0:b0]) and torch.equal(got_u[a0:b0].cpu(), hu[a0:b0])
    assert torch.isnan(got_c[:a0]).all() and torch.isnan(got_u[b0:]).all()
    assert torch.equal(snap[a0:b0], hu[a0:b0]) and torch.isnan(snap[:a0]).all() and torch.isnan(snap[b0:]).all()
    assert L.lmep_event_destroy(ec) == nat.LMEP_OK and L.lmep_event_destroy(ev) == nat.LMEP_OK
