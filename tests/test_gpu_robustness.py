"""Library-state and call-convention robustness of the CUDA path (liblmep.so):
misaligned views, zero-step runs, concurrent host threads on separate streams.
"""

import os
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


# ------------------------------------------------------------------ glue kernels
@pytest.mark.parametrize("method", ["multiply", "pade"])
@pytest.mark.parametrize("layout", [0, 1])
def test_harvest_half_step_set(lx, orc, method, layout):
    """lmep_harvest_ex half_out: the (w_lin, dt/2 phi_1) rows at delta_t / 2 from
    the same launch (per-item kernel: even number of scaling reps, the iterate
    after half of them) or a second launch (Pade), against the oracle's
    harvest at delta_t / 2 (1e-12), frozen rows included; the full set is
    unchanged."""
    from paper_2603_15964_b200 import _ops
    rng = np.random.default_rng(5)
    n, s, T = 9, 4, 6
    h = 0.01
    tabs, Ls, rows, masks = [], [], [], []
    for t in range(T):
        row = int(rng.integers(0, n))
        x = (np.arange(n) - row) * h * (1 + 0.1 * t)
        terms = ((1, float(rng.uniform(-1, 1))), (2, float(rng.uniform(0.1, 1))))
        Ls.append(orc.local_operator(x, terms))
        rows.append(row)
        masks.append(1 if (t % 2 and row != 0) else 0)
    dt = 0.3 * h * h
    lx._native.set_harvest_method(method)
    try:
        hv = _ops.harvest(n, s, dt, T, L=_ops.dev_f64(np.stack(Ls)), rows=_ops.dev_i32(rows),
                          frozen=torch.as_tensor(np.array(masks, dtype=np.int64), device="cuda"),
                          layout=layout, half=True)
        torch.cuda.synchronize()
    finally:
        lx._native.set_harvest_method("multiply")
    full = hv.rows.cpu().numpy()
    half = hv.half.cpu().numpy()
    if layout == 1:
        full, half = full.transpose(2, 0, 1), half.transpose(2, 0, 1)
    assert int(hv.flag.item()) == 0
    for t in range(T):
        fz = [0] if masks[t] else []
        wl, wp = orc.harvest_phi_weights(Ls[t], dt / 2, 2, rows[t], fz)
        ref = np.vstack([wl, wp[0]])
        den = np.abs(ref).max(axis=1)
        assert (np.abs(half[t] - ref).max(axis=1) / den).max() < 1e-12, (t, method)
        wl, wp = orc.harvest_phi_weights(Ls[t], dt, s, rows[t], fz)
        ref = np.vstack([wl] + list(wp))
        den = np.abs(ref).max(axis=1)
        assert (np.abs(full[t] - ref).max(axis=1) / den).max() < 1e-12, (t, method)


def test_harvest_status_flag(lx):
    """A non-finite operator sets the library's device flag (lmep_harvest_ex
    status_any); raise_on_status reads that flag."""
    from paper_2603_15964_b200 import _ops
    L = np.zeros((3, 7, 7))
    L[1, 2, 3] = np.nan
    hv = _ops.harvest(7, 2, 0.1, 3, L=_ops.dev_f64(L), row_default=3, half=True)
    assert int(hv.flag.item()) == 1
    assert hv.status.cpu().numpy().tolist()[1] != 0
    with pytest.raises(lx.NonFinite):
        _ops.raise_on_status(hv)


def test_combine_kernel_matches_numpy(lx):
    """lmep_combine = harvest.combine's numpy expression (zeros + c * a, list
    order, two roundings per term) bit for bit, on strided row arrays."""
    from paper_2603_15964_b200 import _ops
    rng = np.random.default_rng(9)
    A = rng.standard_normal((5, 3, 11)) * 10.0 ** rng.integers(-20, 3, (5, 3, 1))
    A[0, 0, 0] = -0.0
    coeffs = [1.0, -3.0 / 7e-11, 4.0 / 7e-11 ** 2]
    ref = np.zeros((5, 11))
    for i, c in enumerate(coeffs):
        ref = ref + c * A[:, i]
    d = torch.as_tensor(A, device="cuda")
    out = torch.empty((5, 11), dtype=torch.float64, device="cuda")
    _ops.combine_into(out, [d[:, i] for i in range(3)], coeffs, 5, 11, 11, [33, 33, 33])
    assert np.array_equal(out.cpu().numpy(), ref)


@pytest.mark.parametrize("case", ["shared", "class", "pernode"])
def test_compress_classification(lx, case):
    """Reference-style (N, n) rows are compressed on the device (lmep_rows_classify)
    into shared / class / per-node form, and expand back to the same array."""
    from paper_2603_15964_b200 import _native as nat, _ops
    from paper_2603_15964_b200.grid import StencilSet
    N, n = 257, 7
    rng = np.random.default_rng(2)
    mid = rng.standard_normal(n)
    W = np.tile(mid, (N, 1))
    lay = StencilSet(N, n, 3, case == "shared")
    if case == "class":
        W[:4] = rng.standard_normal((4, n))
        W[N - 3:] = rng.standard_normal((3, n))
    if case == "pernode":
        W[100] += 1.0
    cr = _ops.compress(torch.as_tensor(W, device="cuda"), lay)
    want = {"shared": nat.W_SHARED, "class": nat.W_CLASS, "pernode": nat.W_PERNODE}[case]
    assert cr.mode == want
    if case == "class":
        assert (cr.nleft, cr.nright) == (4, 3)
    assert np.array_equal(cr.dense()[0].cpu().numpy(), W)


def test_reference_style_linspace_grid_takes_class_path(lx):
    """Grid(nodes=np.linspace(...), NON_PERIODIC) -- the reference's way to build
    config 4 -- is recognised as uniform: class rows (not one exponential per
    node) and a run bit-identical to make_uniform_grid's."""
    from paper_2603_15964_b200 import _native as nat, configs
    from paper_2603_15964_b200.harvest import harvest_compact
    w = configs.c4(N=4096, steps=20)
    gref = lx.Grid(nodes=np.linspace(-1.0, 1.0, w.N), x_min=-1.0, x_max=1.0,
                   topology=lx.Topology.NON_PERIODIC)
    gu = lx.make_uniform_grid(w.N, -1.0, 1.0)
    assert gref.uniform_spacing == gu.uniform_spacing
    st = lx.select_stencils(gref, w.n, lx.StencilPolicy.CENTERED)
    rows = harvest_compact(gref, st, lx.LinearOperatorSpec(w.terms), w.delta_t, 1, (0, w.N - 1))
    assert rows.mode == nat.W_CLASS
    prob = lx.SemiLinearProblem(lx.LinearOperatorSpec(w.terms), None, w.u0,
                                lx.Boundary.neumann(), "cubic")
    a = lx.run(gref, st, prob, lx.SchemeConfig("etdrk4"), w.delta_t, 20 * w.delta_t)
    stu = lx.select_stencils(gu, w.n, lx.StencilPolicy.CENTERED)
    b = lx.run(gu, stu, prob, lx.SchemeConfig("etdrk4"), w.delta_t, 20 * w.delta_t)
    assert np.array_equal(a.u_final, b.u_final)


def test_rebinding_caches_read_only_arrays(lx, orc):
    """kernels.run_* called repeatedly with the same read-only (N, n) arrays (the
    reference's run() loop over snapshot chunks) validates the member array
    and uploads / compresses each weight array once; writable arrays are re-read."""
    from paper_2603_15964_b200 import kernels
    N, n, row = 3000, 13, 6
    rng = np.random.default_rng(4)
    W = rng.standard_normal((N, n)) / n
    m = orc.members_for(N, n, row, True)
    W.setflags(write=False)
    m.setflags(write=False)
    u0 = rng.standard_normal(N)
    kernels._ROWS.d.clear()
    kernels._LAYOUTS.d.clear()
    u = u0
    for _ in range(4):
        u = kernels.run_linear(W, m, u, 5)
    assert len(kernels._ROWS.d) == 1 and len(kernels._LAYOUTS.d) == 1
    assert np.array_equal(u, orc.run_linear(W, m, u0, 20))
    W2 = W.copy()                                    # writable: never cached
    kernels.run_linear(W2, m, u0, 1)
    assert len(kernels._ROWS.d) == 1
    W2[0, 0] += 1.0
    assert np.array_equal(kernels.run_linear(W2, m, u0, 3), orc.run_linear(W2, m, u0, 3))


def test_c_program_on_the_c_abi(tmp_path):
    """tests/c_abi/smoke.c: a C program that links liblmep.so and the CUDA runtime only (no
    Python, no torch) runs config 1's path -- Fornberg tables, the harvest of the shared row,
    60 steps -- and matches its own host loop bit for bit."""
    import shutil
    import subprocess
    from paper_2603_15964_b200 import _native
    from tests.conftest import REPO
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    libdir = os.path.dirname(_native.LIB_PATH)
    exe = str(tmp_path / "smoke")
    subprocess.run([nvcc, "-Xcompiler", "-ffp-contract=off", "-I", os.path.join(REPO, "include"),
                    os.path.join(REPO, "tests", "c_abi", "smoke.c"), "-L", libdir, "-llmep",
                    "-Xlinker", "-rpath", "-Xlinker", libdir, "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert "c-abi smoke ok" in out.stdout and "60 steps bit-identical" in out.stdout


@pytest.mark.gpu
def test_status_any_every_alignment():
    """lmep_status_any (16-byte loads over the aligned body, scalar head and tail):
    a single failed item is found wherever it sits, for every offset of the status
    array within a 16-byte line and sizes around the vector width; clean arrays
    leave the flag alone."""
    import torch
    from paper_2603_15964_b200 import _native as nat
    L = nat.lib()
    nat.device()
    base = torch.zeros(5000, dtype=torch.int32, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    for off in range(5):
        for B in (1, 2, 3, 4, 5, 7, 8, 9, 31, 1024, 4093):
            view = base[off:off + B]
            for bad in sorted({0, B // 2, B - 1}):
                flag.zero_()
                assert L.lmep_status_any(view.data_ptr(), B, flag.data_ptr(), nat.stream_handle()) == 0
                assert int(flag.item()) == 0, (off, B)
                view[bad] = nat.LMEP_NONFINITE
                assert L.lmep_status_any(view.data_ptr(), B, flag.data_ptr(), nat.stream_handle()) == 0
                assert int(flag.item()) == 1, (off, B, bad)
                view[bad] = 0
