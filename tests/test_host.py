"""Host-side logic: stencil geometry, member recognition, config validation."""

import numpy as np
import pytest

import paper_2603_15964_b200 as lx
from paper_2603_15964_b200 import _ops
from paper_2603_15964_b200.grid import StencilSet


def _ref_members(N, n, row, periodic):
    # grid.py:136-175 restated with an explicit loop
    out = []
    rows = []
    for t in range(N):
        start = t - row
        if periodic:
            m = [(start + j) % N for j in range(n)]
            r = row
        else:
            start = min(max(start, 0), N - n)
            m = [start + j for j in range(n)]
            r = t - start
        out.append(m)
        rows.append(r)
    return np.array(out), np.array(rows)


@pytest.mark.parametrize("N,n,policy,periodic", [(16, 5, "centered", True), (16, 5, "centered", False),
                                                   (20, 7, "upwind", True), (20, 7, "upwind", False),
                                                   (9, 9, "centered", True)])
def test_stencil_set_matches_reference_windows(N, n, policy, periodic):
    g = lx.make_periodic_grid(N, 0.0, 1.0) if periodic else lx.make_uniform_grid(N, -1.0, 1.0)
    pol = lx.StencilPolicy.CENTERED if policy == "centered" else lx.StencilPolicy.ONE_SIDED_UPWIND
    s = lx.select_stencils(g, n, pol)
    m, r = _ref_members(N, n, s.row, periodic)
    assert np.array_equal(s.members_array(), m)
    assert np.array_equal(s.target_rows(), r)
    for t in (0, N // 2, N - 1):
        st = s[t]
        assert np.array_equal(st.members, m[t]) and st.target_row == r[t]
    assert _ops.validate_members(m, m.shape).__dict__ == s.__dict__


def test_validate_members_rejects_scatter():
    m = np.arange(40).reshape(8, 5) % 8
    with pytest.raises(lx.InvalidConfig):
        _ops.validate_members(m[::-1].copy(), m.shape)


def test_select_stencils_errors():
    g = lx.make_periodic_grid(8, 0.0, 1.0)
    with pytest.raises(lx.StencilTooLarge):
        lx.select_stencils(g, 9, lx.StencilPolicy.CENTERED)
    with pytest.raises(lx.InvalidGrid):
        lx.select_stencils(g, 4, lx.StencilPolicy.CENTERED)


def test_grid_validation():
    with pytest.raises(lx.InvalidGrid):
        lx.Grid(nodes=[0.0, 0.0, 1.0], x_min=0.0, x_max=1.0, topology=lx.Topology.NON_PERIODIC)
    with pytest.raises(lx.InvalidGrid):
        lx.make_periodic_grid(2, 0.0, 1.0)


def test_scheme_and_problem_validation():
    with pytest.raises(lx.InvalidConfig):
        lx.SchemeConfig("rk4")
    with pytest.raises(lx.InvalidConfig):
        lx.SchemeConfig("etd-multistep", s=0)
    with pytest.raises(lx.InvalidConfig):
        lx.SemiLinearProblem(lx.LinearOperatorSpec(((2, 1.0),)), None, np.zeros(5),
                             lx.Boundary.periodic(), "quadratic")
    with pytest.raises(lx.InvalidConfig):
        lx.SemiLinearProblem(lx.LinearOperatorSpec(((2, 1.0),)), None, np.zeros(5),
                             lx.Boundary.dirichlet(1.0, 0.0), "none")


def test_operator_spec():
    s = lx.LinearOperatorSpec(((0, 1.0), (2, 1e-4)))
    assert s.max_order == 2 and s.reaction == 1.0
    with pytest.raises(ValueError):
        lx.LinearOperatorSpec(((1, 1.0), (1, 2.0)))
    with pytest.raises(ValueError):
        lx.LinearOperatorSpec(())


def test_frozen_masks_and_class_plan():
    from paper_2603_15964_b200.harvest import _frozen_masks
    s = StencilSet(32, 7, 3, False)
    t = np.arange(32)
    masks = _frozen_masks(s, t, [0, 31])
    m = s.members_array()
    for i in range(32):
        want = sum(1 << j for j in range(7) if m[i, j] in (0, 31))
        assert int(masks[i]) == want


def test_configs_are_seeded_and_shaped():
    from paper_2603_15964_b200 import configs
    a, b = configs.c1(), configs.c1()
    assert np.array_equal(a.u0, b.u0) and a.N == 1024 and a.n == 7 and a.row == 6
    c5 = configs.c5(N=256)
    c, nu = c5.coef
    assert abs(c.min() + 2) < 1e-12 and abs(c.max() - 2) < 1e-12
    assert nu.min() >= 1e-4 * (1 - 1e-12) and nu.max() <= 1e-1 * (1 + 1e-12)


# ---------------------------------------------------------------- table I/O
@pytest.mark.parametrize("mode", ["shared", "class", "pernode"])
def test_weight_table_binary_roundtrip(tmp_path, mode):
    import torch
    from paper_2603_15964_b200 import _native as nat
    from paper_2603_15964_b200 import _ops
    from paper_2603_15964_b200.grid import StencilSet
    from paper_2603_15964_b200.tableio import load_weight_table, save_weight_table
    rng = np.random.default_rng(3)
    R, n = 3, 7
    if mode == "shared":
        rows = _ops.CompactRows(StencilSet(64, n, 3, True), nat.W_SHARED,
                                torch.from_numpy(rng.standard_normal((R, n))))
    elif mode == "class":
        rows = _ops.CompactRows(StencilSet(64, n, 3, False), nat.W_CLASS,
                                torch.from_numpy(rng.standard_normal((R, n))),
                                torch.from_numpy(rng.standard_normal((7, R, n))), 3, 3)
    else:
        rows = _ops.CompactRows(StencilSet(64, n, 3, True), nat.W_PERNODE,
                                pernode=torch.from_numpy(rng.standard_normal((R, n, 64 + 8))),
                                pernode_pad=4)
    p = tmp_path / "t.lmwt"
    nbytes = save_weight_table(p, rows, 1.25e-3)
    assert nbytes == p.stat().st_size
    back, dt = load_weight_table(p, device="cpu")
    assert dt == 1.25e-3 and back.mode == rows.mode and back.pernode_pad == rows.pernode_pad
    assert (back.layout.N, back.layout.n, back.layout.row, back.layout.periodic) == \
        (rows.layout.N, rows.layout.n, rows.layout.row, rows.layout.periodic)
    for a in ("interior", "classes", "pernode"):
        x, y = getattr(rows, a), getattr(back, a)
        assert (x is None and y is None) or torch.equal(x, y)


def test_weight_table_json_parse(golden):
    """The reference's JSON table (harvest.py:238-265) parses back exactly."""
    import json
    from paper_2603_15964_b200.tableio import parse_weight_table_json
    text = str(golden["wtj"])
    rows, dt = parse_weight_table_json(text, device="cpu")
    ref = json.loads(text)
    assert dt == ref["delta_t"] and rows.layout.periodic and rows.layout.N == ref["N"]
    W = rows.pernode.numpy()
    for i, r in enumerate(ref["nodes"]):
        assert np.array_equal(W[0, :, i], r["w_lin"])
        assert np.array_equal(W[1, :, i], r["w_phi"][0])
    with pytest.raises(Exception):
        bad = json.loads(text)
        bad["nodes"][0]["members"] = [5, 3, 1]
        parse_weight_table_json(json.dumps(bad), device="cpu")


def test_reference_test_oracles_exported():
    """phi_scalar / expm_taylor_oracle (expm.py:45-83) keep the reference's names
    and values: closed forms of phi_j, both branches of phi_scalar."""
    import math
    import paper_2603_15964_b200 as lx
    for z in (0.3, -0.2 + 0.1j, 1.7, -2.5):
        assert abs(lx.phi_scalar(0, z) - np.exp(z)) < 1e-15 * abs(np.exp(z))
        p1 = (np.exp(z) - 1) / z
        assert abs(lx.phi_scalar(1, z) - p1) < 1e-13 * abs(p1)
        p2 = (np.exp(z) - 1 - z) / z ** 2
        assert abs(lx.phi_scalar(2, z) - p2) < 1e-10 * abs(p2)
    assert abs(lx.phi_scalar(3, 0.0) - 1.0 / 6.0) < 1e-16
    with pytest.raises(ValueError):
        lx.phi_scalar(9, 0.1)
    A = np.array([[0.0, 1.0], [-1.0, 0.0]])
    E = lx.expm_taylor_oracle(A)
    R = np.array([[math.cos(1), math.sin(1)], [-math.sin(1), math.cos(1)]])
    assert np.abs(E - R).max() < 1e-15
    with pytest.raises(lx.NoConvergence):
        lx.expm_taylor_oracle(50.0 * A, max_terms=5)


@pytest.mark.parametrize("n,row,nl,P", [(7, 3, 2, 7), (11, 5, 1, 5), (13, 6, 2, 5), (9, 4, 0, 5),
                                        (7, 3, 1, 5)])
def test_plan_etdrk4_one_chunk_per_thread(n, row, nl, P):
    """lmep_plan (host logic only): the register-resident ETDRK4 passes need the whole
    staged range, tile + k * radius, covered by one chunk of P nodes per thread."""
    from paper_2603_15964_b200 import _native as nat
    ext = 8 if nl == nat.NL_CONVECTIVE else 4
    rad = ext * (n - 1)
    for N in (1 << 20, 1 << 24):
        pl = _ops.plan(StencilSet(N, n, row, True), nat.SCH_ETDRK4, nl, nat.W_SHARED, 1000)
        staged = pl["tile"] + pl["ksteps"] * rad
        assert pl["ring"] == 0 and pl["ksteps"] >= 1
        assert staged <= 256 * P and pl["threads"] * P >= staged, pl
        assert pl["threads"] % 32 == 0 and pl["threads"] <= 256


def test_plan_small_grids_and_per_node():
    """Ring mode for grids that fit one CTA's shared memory, the persistent per-node
    kernels' 1536-node spans (tile + k (n-1)) for large per-node linear grids."""
    from paper_2603_15964_b200 import _native as nat
    pl = _ops.plan(StencilSet(1024, 7, 6, True), nat.SCH_LIN, nat.NL_NONE, nat.W_SHARED, 1000)
    assert pl["ring"] == 1 and pl["tile"] == 1024
    pl = _ops.plan(StencilSet(1 << 22, 13, 6, True), nat.SCH_LIN, nat.NL_NONE, nat.W_PERNODE, 200)
    assert pl["ring"] == 0 and pl["ksteps"] == 25 and pl["tile"] + pl["ksteps"] * 12 == 1536
    # a non-periodic grid never takes ring mode
    pl = _ops.plan(StencilSet(1024, 7, 3, False), nat.SCH_LIN, nat.NL_NONE, nat.W_SHARED, 10)
    assert pl["ring"] == 0
