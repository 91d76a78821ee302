"""Pin the C oracle against golden vectors produced by the live reference
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from tests.conftest import rel_inf, rel_l2


def test_fornberg_bitwise(golden, orc):
    for i in range(int(golden["forn_count"])):
        c = orc.fornberg_weights(float(golden[f"forn{i}_z"]), golden[f"forn{i}_x"],
                                 int(golden[f"forn{i}_m"]))
        assert np.array_equal(c, golden[f"forn{i}_c"]), i


def test_local_operator_bitwise(golden, orc):
    for i in range(int(golden["lop_count"])):
        terms = list(zip(golden[f"lop{i}_k"].tolist(), golden[f"lop{i}_c"].tolist()))
        L = orc.local_operator(golden[f"lop{i}_x"], terms)
        assert np.array_equal(L, golden[f"lop{i}_L"]), i


def test_fornberg_errors(orc):
    from oracle.oracle import OracleError
    with pytest.raises(OracleError):
        orc.fornberg_weights(0.0, [0.0, 1.0, 2.0], 3)       # OrderTooHigh
    with pytest.raises(OracleError):
        orc.fornberg_weights(0.0, [0.0, 1.0, 1.0], 1)       # DuplicateNodes


def test_balance_matches_scipy(golden, orc):
    for i in range(int(golden["bal_count"])):
        B, s = orc.matrix_balance(golden[f"bal{i}_A"])
        assert np.array_equal(s, golden[f"bal{i}_s"]), i
        assert np.array_equal(B, golden[f"bal{i}_B"]), i


def test_expm_matches_reference(golden, orc):
    worst = 0.0
    for i in range(int(golden["ex_count"])):
        E = orc.expm(golden[f"ex{i}_A"])
        ref = golden[f"ex{i}_E"]
        err = rel_inf(E, ref)
        worst = max(worst, err)
        assert err < 1e-12, (i, err)
    print("worst expm rel err", worst)


def test_harvest_block_and_reduced(golden, orc):
    for i in range(int(golden["hv_count"])):
        dt, s, row = golden[f"hv{i}_meta"]
        s, row = int(s), int(row)
        fm = int(golden[f"hv{i}_frozen"])
        frozen = [j for j in range(64) if (fm >> j) & 1]
        ref = golden[f"hv{i}_w"]
        for reduced in (False, True):
            wl, wp = orc.harvest_phi_weights(golden[f"hv{i}_L"], dt, s, row, frozen, reduced=reduced)
            W = np.vstack([wl] + list(wp))
            for r in range(s):
                den = np.abs(ref[r]).max()
                err = np.abs(W[r] - ref[r]).max() / (den if den > 0 else 1.0)
                assert err < 1e-12, (i, reduced, r, err)


def test_c1_run_linear(golden, orc):
    from paper_2603_15964_b200 import configs
    w = configs.c1()
    m = orc.members_for(w.N, w.n, w.row, True)
    W = np.tile(golden["c1_w"], (w.N, 1))
    u = orc.run_linear(W, m, golden["c1_u0"], w.steps)
    # same weights, same ascending unfused arithmetic as numba -> bitwise
    assert np.array_equal(u, golden["c1_u"])


def test_c1_harvest_then_run(golden, orc):
    from paper_2603_15964_b200 import configs
    w = configs.c1()
    L = orc.local_operator((np.arange(w.n) - w.row) * w.h, w.terms)
    wl, _ = orc.harvest_phi_weights(L, w.delta_t, 1, w.row, reduced=True)
    assert rel_inf(wl, golden["c1_w"]) < 1e-12
    m = orc.members_for(w.N, w.n, w.row, True)
    u = orc.run_linear(np.tile(wl, (w.N, 1)), m, golden["c1_u0"], w.steps)
    assert rel_l2(u, golden["c1_u"]) < 1e-10


def _etd4_rows(orc, x, terms, dt, row, frozen=()):
    L = orc.local_operator(x, terms)
    wl, wp = orc.harvest_phi_weights(L, dt, 4, row, frozen)
    hl, hp = orc.harvest_phi_weights(L, dt / 2, 2, row, frozen)
    return [wl, *wp], [hl, *hp]


def test_kdv_etdrk4_bitwise_with_reference_rows(golden, orc):
    N, n = 512, 11
    rows = golden["kdv_rows"]
    full = [np.tile(r, (N, 1)) for r in rows[:4]]
    half = [np.tile(r, (N, 1)) for r in rows[4:6]]
    d1 = np.tile(rows[6], (N, 1))
    dt = float(golden["kdv_dt"])
    w, al, be, ga, wh, p1h = orc.etdrk4_operators(full, half, dt)
    m = orc.members_for(N, n, 5, True)
    u = orc.run_etdrk4(w, al, be, ga, wh, p1h, 6.0 * d1, m, 1, golden["kdv_u0"],
                       int(golden["kdv_steps"]))
    assert np.array_equal(u, golden["kdv_u"])


def test_burgers_etdrk4_and_etd2_end_to_end(golden, orc):
    from paper_2603_15964_b200 import configs
    w2 = configs.c2(N=256, steps=40)
    dt = float(golden["burg4_dt"])
    x = (np.arange(w2.n) - w2.row) * w2.h
    full, half = _etd4_rows(orc, x, w2.terms, dt, w2.row)
    N = w2.N
    T = lambda r: np.tile(r, (N, 1))
    d1 = T(orc.fornberg_weights(0.0, x, 1)[1])
    ops = orc.etdrk4_operators([T(r) for r in full], [T(r) for r in half], dt)
    m = orc.members_for(N, w2.n, w2.row, True)
    u4 = orc.run_etdrk4(*ops, d1, m, 1, golden["burg4_u0"], int(golden["burg4_steps"]))
    assert rel_l2(u4, golden["burg4_u"]) < 1e-12
    L = orc.local_operator(x, w2.terms)
    r0, (r1, r2) = orc.harvest_phi_weights(L, dt, 3, w2.row)
    u2 = orc.run_etd2((T(r0), T(r1), T(r2)), ops, d1, m, 1, golden["burg4_u0"],
                      int(golden["burg4_steps"]), dt)
    assert rel_l2(u2, golden["burg2_u"]) < 1e-12


def test_dirichlet_cubic_end_to_end(golden, orc):
    N, n = 64, 7
    h = 2.0 / (N - 1)
    dt = float(golden["ac_dt"])
    terms = ((0, 1.0), (2, 1e-3))
    rows = orc.target_rows_for(N, n, 3, False)
    m = orc.members_for(N, n, 3, False)
    full = np.zeros((4, N, n))
    half = np.zeros((2, N, n))
    for t in range(N):
        x = (m[t] - t) * h
        fr = [j for j in range(n) if m[t, j] in (0, N - 1)]
        f, hh = _etd4_rows(orc, x, terms, dt, rows[t], fr)
        full[:, t] = f
        half[:, t] = hh
    assert rel_inf(full[0], golden["ac_wfull"]) < 1e-12
    assert rel_inf(full[3], golden["ac_p3"]) < 1e-12
    ops = orc.etdrk4_operators(list(full), list(half), dt)
    u = orc.run_etdrk4(*ops, np.zeros((N, n)), m, 2, golden["ac_u0"], 25,
                       bc=("dirichlet", -1.0, 1.0))
    assert rel_l2(u, golden["ac_u"]) < 1e-10


def test_c4_neumann_adapter_bitwise(golden, orc):
    W = golden["c4_weights"]
    N, n = W.shape[1], W.shape[2]
    m = orc.members_for(N, n, 3, False)
    u0 = golden["c4_u0"].copy()
    dl, dr = golden["c4_dl"], golden["c4_dr"]
    # run() closes the initial data before stepping (timestep.py:310-311)
    acc = 0.0
    for j in range(1, n):
        acc += dl[j] * u0[j]
    u0[0] = -acc / dl[0]
    acc = 0.0
    for j in range(n - 1):
        acc += dr[j] * u0[N - n + j]
    u0[N - 1] = -acc / dr[n - 1]
    u = orc.run_etdrk4(*W, np.zeros((N, n)), m, 2, u0, 40, bc=("neumann", dl, dr))
    assert np.array_equal(u, golden["c4_u"])
    dl2, dr2 = orc.neumann_rows(n, 2.0 / (N - 1))
    assert np.array_equal(dl2, dl) and np.array_equal(dr2, dr)


def test_c5_per_node_harvest_and_run(golden, orc):
    from paper_2603_15964_b200 import configs
    w5 = configs.c5(N=64, steps=20)
    c, nu = w5.coef
    x = (np.arange(w5.n) - w5.row) * w5.h
    tab = orc.fornberg_weights(0.0, x, 2)
    D1 = np.array([orc.fornberg_weights(xi, x, 2)[1] for xi in x])
    D2 = np.array([orc.fornberg_weights(xi, x, 2)[2] for xi in x])
    W = orc.harvest_batch_vc(D1, D2, -c, nu, w5.delta_t, 4, w5.row, reduced=True)
    ref = golden["c5_W"]
    for r in range(4):
        den = np.abs(ref[:, r]).max(axis=1)
        err = (np.abs(W[:, r] - ref[:, r]).max(axis=1) / den).max()
        assert err < 1e-12, (r, err)
    m = orc.members_for(w5.N, w5.n, w5.row, True)
    u = orc.run_linear(np.ascontiguousarray(W[:, 0]), m, w5.u0, w5.steps)
    assert rel_l2(u, golden["c5_u"]) < 1e-12
    del tab


@pytest.mark.parametrize("periodic,mode", [(True, 0), (True, 2), (False, 1), (False, 2),
                                           (False, 3), (True, 3)])
def test_compact_runners_bitwise_with_member_loops(orc, periodic, mode):
    """The index-arithmetic runners (full-size parity runs) against the
    member-array loops that restate kernels.py, on the dense rows the compact
    rows stand for: linear, ETDRK4 (convective + cubic, Neumann closure on
    clamped grids) and ETD2 with its warm-up step, bit for bit."""
    rng = np.random.default_rng(7 + mode)
    N, n, row = 97, 7, 3
    nl, nr = (3, 4) if mode == 1 else (0, 0)
    K = 5
    cls = rng.integers(0, K, N) if mode == 3 else None
    cp = orc.Compact(N, n, row, periodic, mode, nl, nr, cls=cls, nkeys=K)
    shape = {0: (n,), 1: (nl + 1 + nr, n), 2: (N, n), 3: (K, n)}[mode]
    ops = [0.1 * rng.standard_normal(shape) for _ in range(7)]
    dense = [cp.dense(x) for x in ops]
    m = orc.members_for(N, n, row, periodic)
    u0 = 0.1 * rng.standard_normal(N)
    bc = None if periodic else ("neumann", rng.standard_normal(n) + 3, rng.standard_normal(n) + 3)
    assert np.array_equal(cp.run_linear(ops[0], u0, 5, bc), orc.run_linear(dense[0], m, u0, 5, bc))
    for kind in (1, 2):
        a = cp.run_etdrk4(ops[:6], ops[6], kind, u0, 3, bc)
        assert np.array_equal(a, orc.run_etdrk4(*dense[:6], dense[6], m, kind, u0, 3, bc))
        a, ha = cp.run_etd2(ops[:3], ops[:6], ops[6], kind, u0, 4, 0.3, bc, return_hist=True)
        b, hb = orc.run_etd2(dense[:3], dense[:6], dense[6], m, kind, u0, 4, 0.3, bc,
                             return_hist=True)
        assert np.array_equal(a, b) and np.array_equal(ha, hb)


def test_compact_runner_on_golden_kdv(golden, orc):
    """The compact ETDRK4 runner reproduces the reference's KdV run (golden,
    numba loop) bit for bit from the shared rows."""
    N, n = 512, 11
    rows = golden["kdv_rows"]
    dt = float(golden["kdv_dt"])
    ops = orc.etdrk4_rows(rows[:4], rows[4:6], dt)
    cp = orc.Compact(N, n, 5, True, 0)
    u = cp.run_etdrk4(ops, 6.0 * rows[6], 1, golden["kdv_u0"], int(golden["kdv_steps"]))
    assert np.array_equal(u, golden["kdv_u"])
