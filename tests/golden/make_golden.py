"""Generate golden vectors from the LIVE reference (localexp) in this container.

Run once here (the reference is not present on the GPU box):

    python tests/golden/make_golden.py

It copies /root/reference/pkg/src/localexp to a temp dir (numba's
cache=True would otherwise write into the read-only reference tree, SURVEY
8(c)), imports it, and stores small inputs + reference outputs in
tests/golden/golden.npz.  Every array is produced by reference code; the
only adapters are (a) the Neumann closure for config 4, built from the
reference's own kernels.banded_matvec and harvest with frozen_nodes, and
(b) the per-node variable-coefficient loop for config 5, built from
local_operator + harvest_phi_weights.
"""

from __future__ import annotations

import math
import os
import shutil
import sys
import tempfile

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)


def import_reference():
    tmp = tempfile.mkdtemp(prefix="localexp_ref_")
    shutil.copytree("/root/reference/pkg/src/localexp", os.path.join(tmp, "localexp"))
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tmp, "nbcache"))
    os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
    sys.path.insert(0, tmp)
    import localexp  # noqa: F401
    return localexp


def main(out=os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")):
    le = import_reference()
    from localexp import kernels, timestep
    from localexp.expm import expm as ref_expm
    from paper_2603_15964_b200 import configs

    import scipy.linalg

    G: dict[str, np.ndarray] = {}
    rng = np.random.default_rng(20260315)

    # ---- 1. Fornberg tables (localop.py:61-96) -------------------------
    cases = []
    for n in (2, 3, 5, 7, 9, 11, 13, 15):
        for row in sorted({0, (n - 1) // 2, n - 1}):
            h = 2.0 * math.pi / 1024
            cases.append(((np.arange(n) - row) * h, 0.0, min(3, n - 1)))
    for n in (4, 7, 13):
        x = np.sort(rng.uniform(-1, 1, n))
        cases.append((x, float(x[n // 2]), min(3, n - 1)))
        cases.append((x, 0.123, min(2, n - 1)))
    m = 20
    cheb = -np.cos(np.arange(m) * np.pi / (m - 1))
    cases.append((cheb[:9] - cheb[0], 0.0, 3))
    for i, (x, z, mo) in enumerate(cases):
        G[f"forn{i}_x"] = np.asarray(x, float)
        G[f"forn{i}_z"] = np.array(z)
        G[f"forn{i}_m"] = np.array(mo)
        G[f"forn{i}_c"] = le.fornberg_weights(z, x, mo)
    G["forn_count"] = np.array(len(cases))

    # ---- 2. local operators (localop.py:111-128) ------------------------
    lo_cases = [
        ((np.arange(7) - 6) * (2 * math.pi / 1024), ((1, -1.0),)),
        ((np.arange(9) - 4) * (2 * math.pi / 65536), ((2, 0.01),)),
        ((np.arange(11) - 5) * (40.0 / 2**20), ((3, -1.0),)),
        ((np.arange(7) - 0) * (2.0 / (2**24 - 1)), ((0, 1.0), (2, 1e-4))),
        ((np.arange(7) - 3) * (2.0 / (2**24 - 1)), ((0, 1.0), (2, 1e-4))),
        ((np.arange(13) - 6) * (1.0 / 2**22), ((1, -1.37), (2, 0.0421))),
        ((np.arange(5) - 2) * 0.1, ((0, -0.5), (1, 0.3), (2, 0.7), (3, -0.2))),
    ]
    for i, (x, terms) in enumerate(lo_cases):
        G[f"lop{i}_x"] = x
        G[f"lop{i}_k"] = np.array([t[0] for t in terms], np.int32)
        G[f"lop{i}_c"] = np.array([t[1] for t in terms], float)
        G[f"lop{i}_L"] = le.local_operator(x, le.LinearOperatorSpec(terms))
    G["lop_count"] = np.array(len(lo_cases))

    # ---- 3. balancing (scipy.linalg.matrix_balance, permute=False) ------
    bal = []
    for d in (3, 6, 10, 16):
        for _ in range(3):
            R = rng.standard_normal((d, d))
            Dg = 2.0 ** rng.integers(-20, 21, d)
            bal.append(R * Dg[:, None] / Dg[None, :])
    for i, A in enumerate(bal):
        B, D = scipy.linalg.matrix_balance(A, permute=False)
        G[f"bal{i}_A"] = A
        G[f"bal{i}_B"] = B
        G[f"bal{i}_s"] = np.diag(D).copy()
    G["bal_count"] = np.array(len(bal))

    # ---- 4. expm (expm.py:24-42 -> scipy) --------------------------------
    ex = []
    for d in (2, 5, 9, 13, 16, 20):
        for target in (1e-3, 0.1, 0.7, 1.8, 4.0, 30.0, 300.0):
            R = rng.standard_normal((d, d)) + 2.0 * np.triu(rng.standard_normal((d, d)), 1)
            ex.append(R * (target / np.abs(R).sum(0).max()))
    for i, A in enumerate(ex):
        G[f"ex{i}_A"] = A
        G[f"ex{i}_E"] = ref_expm(A)
    G["ex_count"] = np.array(len(ex))

    # ---- 5. harvest rows (harvest.py:73-121) -----------------------------
    hv = []
    # (x, terms, dt, s, row, frozen)
    h1 = 2 * math.pi / 1024
    hv.append(((np.arange(7) - 6) * h1, ((1, -1.0),), 3.5 * h1, 1, 6, ()))
    h2 = 2 * math.pi / 65536
    dt2 = 0.5 * h2 * h2 / 0.01
    for s in (2, 3, 4):
        hv.append(((np.arange(9) - 4) * h2, ((2, 0.01),), dt2, s, 4, ()))
    hv.append(((np.arange(9) - 4) * h2, ((2, 0.01),), dt2 / 2, 2, 4, ()))
    h3 = 40.0 / 2**20
    dt3 = 0.05 * h3**3
    hv.append(((np.arange(11) - 5) * h3, ((3, -1.0),), dt3, 4, 5, ()))
    hv.append(((np.arange(11) - 5) * h3, ((3, -1.0),), dt3 / 2, 2, 5, ()))
    h4 = 2.0 / (2**24 - 1)
    dt4 = 0.5 * h4 * h4 / 1e-4
    for row in range(7):
        start_frozen = (0,) if row <= 3 else ()
        hv.append((np.arange(7) * h4 - row * h4, ((0, 1.0), (2, 1e-4)), dt4, 4, row, start_frozen))
        hv.append((np.arange(7) * h4 - row * h4, ((0, 1.0), (2, 1e-4)), dt4 / 2, 2, row, start_frozen))
    hv.append(((np.arange(7) - 3) * h4, ((0, 1.0), (2, 1e-4)), dt4, 4, 3, ()))
    hv.append(((np.arange(7) - 3) * h4, ((0, 1.0), (2, 1e-4)), dt4, 4, 3, (6,)))
    h5 = 1.0 / 2**22
    dt5 = 0.5 * h5 * h5 / 0.1
    for cc, nu in ((-1.9, 0.1), (0.3, 1e-4), (1.2, 3e-3)):
        for s in (1, 4):
            hv.append(((np.arange(13) - 6) * h5, ((1, -cc), (2, nu)), dt5, s, 6, ()))
    # a high-CFL one-sided case (Lagrangian shift) and a large-norm case
    hv.append(((np.arange(7) - 6) * 0.1, ((1, -1.0),), 0.4, 1, 6, ()))
    hv.append(((np.arange(9) - 4) * 0.1, ((2, 1.0),), 0.01, 4, 4, ()))
    for i, (x, terms, dt, s, row, frozen) in enumerate(hv):
        L = le.local_operator(x, le.LinearOperatorSpec(terms))
        ws = le.harvest_phi_weights(L, dt, s, row, frozen_rows=frozen)
        G[f"hv{i}_L"] = L
        G[f"hv{i}_x"] = np.asarray(x, float)
        G[f"hv{i}_k"] = np.array([t[0] for t in terms], np.int32)
        G[f"hv{i}_c"] = np.array([t[1] for t in terms], float)
        G[f"hv{i}_meta"] = np.array([dt, s, row], float)
        fm = 0
        for j in frozen:
            fm |= 1 << j
        G[f"hv{i}_frozen"] = np.array(fm, np.int64)
        G[f"hv{i}_w"] = np.vstack([ws.w_lin] + list(ws.w_phi))
    G["hv_count"] = np.array(len(hv))

    # ---- 6. C1 end to end through run() (timestep.py:255) ----------------
    w1 = configs.c1()
    grid = le.make_periodic_grid(w1.N, w1.x_min, w1.x_max)
    st = le.select_stencils(grid, w1.n, le.StencilPolicy.ONE_SIDED_UPWIND)
    prob = le.SemiLinearProblem(le.LinearOperatorSpec(w1.terms), None, w1.u0,
                                le.Boundary.periodic(), "none")
    res = le.run(grid, st, prob, le.SchemeConfig("linear"), w1.delta_t, w1.steps * w1.delta_t)
    G["c1_u0"] = w1.u0
    G["c1_u"] = res.u_final
    G["c1_w"] = le.assemble_global(grid, st, le.LinearOperatorSpec(w1.terms), w1.delta_t).weights[0]

    # ---- 7. ETDRK4 convective: KdV family (kernels.run_etdrk4, 6*d1w) ----
    w3 = configs.c3(N=512, steps=200)
    grid = le.make_periodic_grid(w3.N, w3.x_min, w3.x_max)
    st = le.select_stencils(grid, w3.n, le.StencilPolicy.CENTERED)
    spec = le.LinearOperatorSpec(w3.terms)
    dt = w3.delta_t
    ops_f = le.assemble_global_phi(grid, st, spec, dt, s=4)
    ops_h = le.assemble_global_phi(grid, st, spec, dt / 2, s=2)
    d1 = le.assemble_derivative(grid, st, 1)
    w, al, be, ga, wh, p1h = timestep.etdrk4_operators(ops_f, ops_h)
    u = kernels.run_etdrk4(w.weights, al.weights, be.weights, ga.weights, wh.weights, p1h.weights,
                           6.0 * d1.weights, w.members, 1, w3.u0, w3.steps, False, 0.0, 0.0)
    G["kdv_u0"] = w3.u0
    G["kdv_u"] = u
    G["kdv_dt"] = np.array(dt)
    G["kdv_steps"] = np.array(w3.steps)
    G["kdv_rows"] = np.vstack([o.weights[0] for o in ops_f] + [o.weights[0] for o in ops_h]
                              + [d1.weights[0]])

    # ---- 8. ETDRK4 convective Burgers through run() ----------------------
    w2 = configs.c2(N=256, steps=40)
    grid = le.make_periodic_grid(w2.N, w2.x_min, w2.x_max)
    st = le.select_stencils(grid, w2.n, le.StencilPolicy.CENTERED)
    prob = le.SemiLinearProblem(le.LinearOperatorSpec(w2.terms), None, w2.u0,
                                le.Boundary.periodic(), "convective")
    # at N=256 the literal mu=0.5 step has convective CFL ~1.2 (ETD2 blows up);
    # use CFL 0.05 for the small-size golden run
    dtb = min(w2.delta_t, 0.05 * (w2.x_max - w2.x_min) / w2.N)
    res = le.run(grid, st, prob, le.SchemeConfig("etdrk4"), dtb, w2.steps * dtb)
    G["burg4_u0"] = w2.u0
    G["burg4_u"] = res.u_final
    G["burg4_dt"] = np.array(dtb)
    G["burg4_steps"] = np.array(w2.steps)

    # ---- 9. ETD2 (etd-multistep s=2) Burgers through run() ---------------
    res = le.run(grid, st, prob, le.SchemeConfig("etd-multistep", s=2), dtb, w2.steps * dtb)
    G["burg2_u"] = res.u_final
    # ---- 9b. etd-multistep of orders 1, 3, 4, 5 (backward-difference form)
    for s in (1, 3, 4, 5):
        res = le.run(grid, st, prob, le.SchemeConfig("etd-multistep", s=s), dtb, w2.steps * dtb)
        G[f"burg_s{s}_u"] = res.u_final

    # ---- 10. cubic ETDRK4 with Dirichlet pins on a non-periodic grid -----
    N = 64
    xg = np.linspace(-1.0, 1.0, N)
    gridd = le.Grid(nodes=xg, x_min=-1.0, x_max=1.0, topology=le.Topology.NON_PERIODIC)
    std = le.select_stencils(gridd, 7, le.StencilPolicy.CENTERED)
    u0 = 0.53 * xg + 0.47 * np.sin(-1.5 * np.pi * xg)
    u0[0], u0[-1] = -1.0, 1.0
    probd = le.SemiLinearProblem(le.LinearOperatorSpec(((0, 1.0), (2, 1e-3))), None, u0,
                                 le.Boundary.dirichlet(-1.0, 1.0), "cubic")
    hd = 2.0 / (N - 1)
    dtd = 0.5 * hd * hd / 1e-3
    res = le.run(gridd, std, probd, le.SchemeConfig("etdrk4"), dtd, 25 * dtd)
    G["ac_u0"] = u0
    G["ac_u"] = res.u_final
    G["ac_dt"] = np.array(dtd)
    ops_f = le.assemble_global_phi(gridd, std, le.LinearOperatorSpec(((0, 1.0), (2, 1e-3))), dtd,
                                   s=4, frozen_nodes=(0, N - 1))
    G["ac_wfull"] = ops_f[0].weights
    G["ac_p3"] = ops_f[3].weights

    # ---- 11. C4 family: Neumann closure adapter -----------
    w4 = configs.c4(N=256, steps=40)
    grid4 = le.Grid(nodes=w4.nodes, x_min=-1.0, x_max=1.0, topology=le.Topology.NON_PERIODIC)
    st4 = le.select_stencils(grid4, w4.n, le.StencilPolicy.CENTERED)
    spec4 = le.LinearOperatorSpec(w4.terms)
    dt4 = w4.delta_t
    of = le.assemble_global_phi(grid4, st4, spec4, dt4, s=4, frozen_nodes=(0, w4.N - 1))
    oh = le.assemble_global_phi(grid4, st4, spec4, dt4 / 2, s=2, frozen_nodes=(0, w4.N - 1))
    w, al, be, ga, wh, p1h = timestep.etdrk4_operators(of, oh)
    h4s = w4.h
    dl = le.fornberg_weights(0.0, np.arange(w4.n) * h4s, 1)[1]
    dr = le.fornberg_weights(0.0, (np.arange(w4.n) - (w4.n - 1)) * h4s, 1)[1]
    G["c4_dl"], G["c4_dr"] = dl, dr
    G["c4_u0"] = w4.u0
    G["c4_u"] = _etdrk4_neumann(kernels, w, al, be, ga, wh, p1h, w4.u0, w4.steps, dl, dr)
    G["c4_weights"] = np.stack([w.weights, al.weights, be.weights, ga.weights, wh.weights,
                                p1h.weights])

    # ---- 12. C5 family: per-node variable coefficient --------------------
    w5 = configs.c5(N=64, steps=20)
    c, nu = w5.coef
    grid5 = le.make_periodic_grid(w5.N, 0.0, 1.0)
    st5 = le.select_stencils(grid5, w5.n, le.StencilPolicy.CENTERED)
    rows = []
    for i, s_ in enumerate(st5):
        coords = s_.offsets * grid5.spacing
        L = le.local_operator(coords, le.LinearOperatorSpec(((1, -c[i]), (2, nu[i]))))
        ws = le.harvest_phi_weights(L, w5.delta_t, 4, s_.target_row)
        rows.append(np.vstack([ws.w_lin] + list(ws.w_phi)))
    W5 = np.array(rows)                      # (N, 4, n)
    members = np.array([s_.members for s_ in st5])
    G["c5_W"] = W5
    G["c5_u0"] = w5.u0
    G["c5_u"] = kernels.run_linear(np.ascontiguousarray(W5[:, 0, :]), members, w5.u0, w5.steps,
                                   False, 0.0, 0.0)

    # ---- 13. Chebyshev grid (the paper's Allen-Cahn setup, problems.py:150-167):
    #          per-node harvest with frozen ends + pinned Dirichlet ETDRK4 run
    from localexp import problems as le_problems
    spec = le_problems.allen_cahn_benchmark(N=64, n=21)
    gridc = le.make_chebyshev_grid(spec.N, spec.x_min, spec.x_max)
    stc = le.select_stencils(gridc, spec.n, spec.policy)
    u0c = spec.initial(gridc.nodes)
    probc = le.SemiLinearProblem(spec.linear, None, u0c, spec.boundary, "cubic")
    resc = le.run(gridc, stc, probc, le.SchemeConfig("etdrk4"), spec.delta_t, 30 * spec.delta_t)
    G["cheb_u0"] = u0c
    G["cheb_u"] = resc.u_final
    ofc = le.assemble_global_phi(gridc, stc, spec.linear, spec.delta_t, s=4,
                                 frozen_nodes=(0, spec.N - 1))
    G["cheb_w"] = np.stack([o.weights for o in ofc])
    # 60-digit values of the same rows (mpmath expm of the (n+3) augmentation,
    # mathematically identical to the reference's block form): the truth the
    # reference and the device harvest are both measured against, because the
    # boundary-adjacent Chebyshev operators (||dt L||_1 ~ 1e9) are too
    # ill-conditioned for any fp64 formulation to agree to 1e-12.
    G["cheb_exact"] = _cheb_exact(le, gridc, stc, spec, (0, spec.N - 1))

    # ---- 14. weight_table_json (harvest.py:238-265) ---------------------------
    gw = le.make_periodic_grid(6, 0.0, 1.0)
    sw = le.select_stencils(gw, 3, le.StencilPolicy.CENTERED)
    from localexp import harvest as le_harvest
    rows = le_harvest._harvest_rows(gw, sw, le.LinearOperatorSpec(((2, 0.3), (1, -0.7))), 0.01, 2)
    G["wtj"] = np.array(le.weight_table_json(sw, rows))

    # ---- 15. analysis (analysis.py:42-193): stability scan, footprint, quadrature
    from localexp import analysis as le_an
    ga = le.make_periodic_grid(256, 0.0, 2 * math.pi)
    sa = le.select_stencils(ga, 7, le.StencilPolicy.ONE_SIDED_UPWIND)
    ha = ga.spacing
    dts = [c * ha for c in (0.5, 1.5, 3.5, 5.0, 6.5, 8.0, 9.5)]
    sb = le_an.scan_stability(ga, sa, le.LinearOperatorSpec(((1, -1.0),)), dts, steps=300)
    G["scan_dt"] = np.array(sb.dt_grid)
    G["scan_stable"] = np.array(sb.stable[0])
    G["scan_dt_star"] = np.array(sb.dt_star[0])
    row = le.assemble_global(ga, sa, le.LinearOperatorSpec(((1, -1.0),)), 3.5 * ha).weights[0]
    fp = le_an.spectral_footprint(row, np.arange(7) - 6, ha, 33, shift=3.5 * ha)
    G["fp_row"], G["fp_G"], G["fp_disp"] = row, fp.amplification, fp.dispersion
    G["cc_w"] = le_an.clenshaw_curtis_weights(17)
    G["cc_w_odd"] = le_an.clenshaw_curtis_weights(18)
    gc = le.make_chebyshev_grid(17, -1.0, 1.0)
    uq = np.sin(3 * gc.nodes) + 0.2
    cq = le_an.conserved_quantities(uq, gc)
    G["cq"] = np.array([cq["mass_l1"], cq["energy_l2"]])
    G["cq_u"] = uq

    np.savez_compressed(out, **G)
    print(f"wrote {out}: {len(G)} arrays, {os.path.getsize(out)} bytes")


def _cheb_exact(le, grid, stencils, spec, frozen_nodes, digits=50):
    import mpmath
    mpmath.mp.dps = digits
    N, n, s = grid.size, stencils[0].n, 4
    out = np.zeros((s, N, n))
    for t, st in enumerate(stencils):
        coords = grid.nodes[st.members] - grid.nodes[t]
        L = le.local_operator(coords, spec.linear)
        fz = [j for j, m in enumerate(st.members.tolist()) if m in frozen_nodes]
        r = st.target_row
        D = n + s - 1
        A = mpmath.zeros(D, D)
        dt = mpmath.mpf(float(spec.delta_t))
        for i in range(n):
            if i in fz:
                continue
            for j in range(n):
                A[j, i] = dt * mpmath.mpf(float(L[i, j]))
        A[r, n] = dt
        for q in range(s - 2):
            A[n + q, n + q + 1] = dt
        E = mpmath.expm(A)
        out[0, t] = [float(E[j, r]) for j in range(n)]
        for q in range(1, s):
            out[q, t] = [0.0 if j in fz else float(E[j, n + q - 1]) for j in range(n)]
    return out


def _etdrk4_neumann(kernels, w, al, be, ga, wh, p1h, u0, steps, dl, dr):
    """kernels.run_etdrk4 (kernels.py:62-132) with the reference's pin lines
    replaced by the zero-gradient closure; every banded product is the
    reference's own kernels.banded_matvec."""
    bm = kernels.banded_matvec
    m = w.members
    N = u0.size
    n = dl.size

    def close(v):
        acc = 0.0
        for j in range(1, n):
            acc += dl[j] * v[j]
        v[0] = -acc / dl[0]
        acc = 0.0
        for j in range(n - 1):
            acc += dr[j] * v[N - n + j]
        v[N - 1] = -acc / dr[n - 1]

    u = u0.copy()
    close(u)
    t1, t2, tmp, whu = (np.empty(N) for _ in range(4))
    for _ in range(steps):
        n0 = -u * u * u
        bm(wh.weights, m, u, whu)
        bm(p1h.weights, m, n0, t1)
        a = whu + t1
        close(a)
        n1 = -a * a * a
        bm(p1h.weights, m, n1, t1)
        b = whu + t1
        close(b)
        n2 = -b * b * b
        bm(wh.weights, m, a, t1)
        t2 = 2.0 * n2 - n0
        bm(p1h.weights, m, t2, tmp)
        cc = t1 + tmp
        close(cc)
        n3 = -cc * cc * cc
        bm(w.weights, m, u, t1)
        bm(al.weights, m, n0, t2)
        t1 = t1 + t2
        tmp = n1 + n2
        bm(be.weights, m, tmp, t2)
        t1 = t1 + t2
        bm(ga.weights, m, n3, t2)
        u = t1 + t2
        close(u)
        t2 = np.empty(N)
        tmp = np.empty(N)
    return u


if __name__ == "__main__":
    main()
