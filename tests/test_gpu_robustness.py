"""Library-state and call-convention robustness of the CUDA path (liblmep.so):
misaligned views, zero-step runs, concurrent host threads on separate streams.
"""

import threading

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lx():
    import paper_2603_15964_b200 as m
    m._native.device()
    return m


def test_pernode_steps_on_misaligned_view(lx):
    """A contiguous device view at an odd element offset (8-byte aligned only)
    cannot feed the TMA bulk copies: the step takes the register-blocked kernel
    and gives the same bits as the aligned call (exact mode)."""
    from paper_2603_15964_b200 import _native as nat, _ops
    from paper_2603_15964_b200.grid import StencilSet
    N, n, row = 5000, 13, 6
    rng = np.random.default_rng(3)
    lay = StencilSet(N, n, row, True)
    W = torch.as_tensor(rng.standard_normal((1, n, N)) / n, device="cuda")
    rows = _ops.CompactRows(lay, nat.W_PERNODE, pernode=W)
    buf = torch.as_tensor(rng.standard_normal(N + 1), device="cuda")
    mis = buf[1:]
    assert mis.data_ptr() % 16 == 8
    ali = mis.clone()
    a = _ops.step(nat.SCH_LIN, rows, ali, 21, exact=True)
    b = _ops.step(nat.SCH_LIN, rows, mis, 21, exact=True)
    assert torch.equal(a, b)
    assert torch.equal(buf[1:], ali)          # input untouched


def test_run_zero_steps(lx):
    """t_final below the rounding tolerance of one step (_steps_for): zero steps,
    one snapshot (the pinned initial data) and an integer harvest time, as the
    reference returns (timestep.py:255-394)."""
    from paper_2603_15964_b200 import configs
    w = configs.c2(N=256, steps=1)
    g = lx.make_periodic_grid(w.N, w.x_min, w.x_max)
    st = lx.select_stencils(g, w.n, lx.StencilPolicy.CENTERED)
    prob = lx.SemiLinearProblem(lx.LinearOperatorSpec(w.terms), None, w.u0,
                                lx.Boundary.periodic(), "convective")
    for stride in (None, w.delta_t):
        r = lx.run(g, st, prob, lx.SchemeConfig("etdrk4"), w.delta_t, 1e-10 * w.delta_t,
                   snapshot_stride=stride)
        assert r.steps == 0
        assert r.snapshots.shape == (1, w.N)
        assert np.array_equal(r.u_final, w.u0)
        assert isinstance(r.harvest_ns, int) and r.harvest_ns >= 0


def test_concurrent_threads_on_streams(lx):
    """Two host threads, each on its own stream, harvesting per-node rows
    (constant-table kernel: one constant block per device) and stepping
    (thread-local launch staging) at the same time: every result equals the
    serial one bit for bit."""
    from paper_2603_15964_b200 import configs, _ops
    from paper_2603_15964_b200.timestep import Stepper, prepare
    jobs = []
    for n in (9, 13):
        w = configs.c5(N=1 << 14, steps=1)
        c, nu = w.coef
        g = lx.make_periodic_grid(w.N, 0.0, 1.0)
        st = lx.select_stencils(g, n, lx.StencilPolicy.CENTERED)
        spec = lx.VariableCoefficientSpec((1, 2), _ops.dev_f64(np.stack([-c, nu], 1)))
        prob = lx.SemiLinearProblem(spec, None, w.u0, lx.Boundary.periodic(), "none")
        jobs.append((g, st, prob, w))

    def work(job):
        g, st, prob, w = job
        prep = prepare(g, st, prob, lx.SchemeConfig("linear"), w.delta_t)
        s = Stepper(prep, _ops.dev_f64(w.u0), exact=True)
        s.advance(40)
        return prep.bank.pernode.clone(), s.u.clone()

    ref = [work(j) for j in jobs]
    torch.cuda.synchronize()
    out = [None, None]
    errs = []

    def thread(i):
        try:
            torch.cuda.set_device(0)
            strm = torch.cuda.Stream()
            with torch.cuda.stream(strm):
                for _ in range(4):
                    out[i] = work(jobs[i])
            strm.synchronize()
        except Exception as e:          # surfaced below
            errs.append(e)

    ts = [threading.Thread(target=thread, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for i in range(2):
        assert torch.equal(out[i][0], ref[i][0])
        assert torch.equal(out[i][1], ref[i][1])


def test_harvest_method_switch_is_per_device(lx):
    """lmep_set_harvest_method applies to the current device; retired codes
    (the first-generation kernel) are rejected."""
    from paper_2603_15964_b200 import _native as nat
    assert nat.lib().lmep_set_harvest_method(2) == nat.LMEP_INVALID_CONFIG
    assert nat.lib().lmep_set_harvest_method(3) == nat.LMEP_INVALID_CONFIG
    nat.set_harvest_method("pade")
    nat.set_harvest_method("multiply")
