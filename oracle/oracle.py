"""ctypes front-end for the C oracle (oracle/lmep_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs, never by the product
package.  Every function mirrors a reference function (file:line cited in
the C source) and takes/returns numpy arrays in the reference's layouts:
(N, n) weight rows and (N, n) int64 member indices.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liblmep_oracle.so")
_lib = None

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


class Geom(C.Structure):
    """orc_geom: the select_stencils window rule (grid.py:136-175) plus the
    compact row mode (0 shared [n], 1 classes [nleft+1+nright][n], 2 per-node [N][n])."""
    _fields_ = [("N", C.c_int64), ("n", C.c_int32), ("row", C.c_int32), ("periodic", C.c_int32),
                ("mode", C.c_int32), ("nleft", C.c_int32), ("nright", C.c_int32),
                ("cls", C.c_void_p)]


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"oracle {what} failed with status {code}")
        self.code = code


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_SO):
        build()
    L = C.CDLL(_SO)
    L.orc_fornberg.argtypes = [C.c_double, _dp, C.c_int, C.c_int, _dp]
    L.orc_local_operator.argtypes = [_dp, C.c_int, _i32p, _dp, C.c_int, _dp]
    L.orc_matrix_balance.argtypes = [_dp, C.c_int, _dp]
    L.orc_expm_raw.argtypes = [_dp, C.c_int, _dp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.orc_expm.argtypes = [_dp, C.c_int, _dp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.orc_build_augmented.argtypes = [_dp, C.c_int, C.c_int, _dp]
    for f in (L.orc_harvest_phi, L.orc_harvest_phi_reduced):
        f.argtypes = [_dp, C.c_int, C.c_double, C.c_int, C.c_int, C.c_uint64, _dp,
                      C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.orc_harvest_batch_vc.argtypes = [_dp, _dp, C.c_int, _dp, _dp, C.c_int64, C.c_double,
                                       C.c_int, C.c_int, C.c_int, _dp, C.c_int]
    L.orc_banded_matvec.argtypes = [_dp, _ip, _dp, _dp, C.c_int64, C.c_int]
    L.orc_banded_matvec.restype = None
    L.orc_run_linear.argtypes = [_dp, _ip, _dp, C.c_int64, C.c_int, C.c_int64, C.c_int,
                                 C.c_double, C.c_double, C.c_void_p, C.c_void_p, _dp]
    L.orc_run_linear.restype = None
    L.orc_run_etdrk4.argtypes = [_dp] * 7 + [_ip, C.c_int, _dp, C.c_int64, C.c_int, C.c_int64,
                                            C.c_int, C.c_double, C.c_double, C.c_void_p,
                                            C.c_void_p, _dp]
    L.orc_run_etdrk4.restype = None
    L.orc_run_etd2.argtypes = [_dp] * 10 + [_ip, C.c_int, _dp, C.c_int64, C.c_int, C.c_int64,
                                             C.c_double, C.c_int, C.c_double, C.c_double,
                                             C.c_void_p, C.c_void_p, _dp, C.c_void_p]
    L.orc_run_etd2.restype = None
    G = C.POINTER(Geom)
    L.orc_run_linear_c.argtypes = [G, _dp, _dp, C.c_int64, C.c_int, C.c_double, C.c_double,
                                   C.c_void_p, C.c_void_p, _dp]
    L.orc_run_linear_c.restype = None
    L.orc_run_etdrk4_c.argtypes = [G] + [_dp] * 7 + [C.c_int, _dp, C.c_int64, C.c_int, C.c_double,
                                                    C.c_double, C.c_void_p, C.c_void_p, _dp,
                                                    C.c_void_p]
    L.orc_run_etdrk4_c.restype = None
    L.orc_run_etd2_c.argtypes = [G] + [_dp] * 10 + [C.c_int, _dp, C.c_int64, C.c_double, C.c_int,
                                                     C.c_double, C.c_double, C.c_void_p,
                                                     C.c_void_p, _dp, C.c_void_p]
    L.orc_run_etd2_c.restype = None
    L.orc_num_threads.restype = C.c_int
    L.orc_set_threads.argtypes = [C.c_int]
    L.orc_set_threads.restype = None
    _lib = L
    return L


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _check(code, what):
    if code != 0:
        raise OracleError(code, what)


def set_threads(t: int) -> None:
    lib().orc_set_threads(int(t))


def num_threads() -> int:
    return int(lib().orc_num_threads())


# --- localop.py ---------------------------------------------------------
def fornberg_weights(z, nodes, max_order):
    x = _f64(nodes)
    out = np.zeros((max_order + 1) * x.size)
    _check(lib().orc_fornberg(float(z), x, x.size, int(max_order), out), "fornberg")
    return out.reshape(max_order + 1, x.size)


def local_operator(nodes, terms):
    x = _f64(nodes)
    k = np.ascontiguousarray([int(t[0]) for t in terms], dtype=np.int32)
    c = _f64([float(t[1]) for t in terms])
    L = np.zeros(x.size * x.size)
    _check(lib().orc_local_operator(x, x.size, k, c, len(terms), L), "local_operator")
    return L.reshape(x.size, x.size)


# --- expm.py / scipy ----------------------------------------------------
def matrix_balance(A):
    B = _f64(A).copy()
    d = B.shape[0]
    scale = np.zeros(d)
    _check(lib().orc_matrix_balance(B.reshape(-1), d, scale), "matrix_balance")
    return B, scale


def expm_raw(A):
    A = _f64(A)
    d = A.shape[0]
    E = np.zeros(d * d)
    m, s = C.c_int(), C.c_int()
    _check(lib().orc_expm_raw(A.reshape(-1), d, E, C.byref(m), C.byref(s)), "expm_raw")
    return E.reshape(d, d), m.value, s.value


def expm(A, return_ms=False):
    A = _f64(A)
    d = A.shape[0]
    E = np.zeros(d * d)
    m, s = C.c_int(), C.c_int()
    _check(lib().orc_expm(A.reshape(-1), d, E, C.byref(m), C.byref(s)), "expm")
    E = E.reshape(d, d)
    return (E, m.value, s.value) if return_ms else E


# --- harvest.py ---------------------------------------------------------
def _mask(frozen_rows):
    m = 0
    for j in frozen_rows:
        m |= 1 << int(j)
    return m


def harvest_phi_weights(L, delta_t, s, target_row, frozen_rows=(), reduced=False):
    """Returns (w_lin, (w_phi_1, ...)) like PhiWeightSet (harvest.py:97-121)."""
    L = _f64(L)
    n = L.shape[0]
    w = np.zeros(s * n)
    f = lib().orc_harvest_phi_reduced if reduced else lib().orc_harvest_phi
    _check(f(L.reshape(-1), n, float(delta_t), int(s), int(target_row), _mask(frozen_rows), w,
             None, None), "harvest_phi")
    w = w.reshape(s, n)
    return w[0].copy(), tuple(w[j].copy() for j in range(1, s))


def harvest_propagator(L, delta_t, target_row):
    return harvest_phi_weights(L, delta_t, 1, target_row)[0]


def harvest_batch_vc(D1, D2, c1, c2, delta_t, s, row, reduced=True, threads=0):
    """Per-node L_i = c1_i*D1 + c2_i*D2 harvest (config-5 oracle).  -> (count, s, n)."""
    D1 = _f64(D1)
    D2 = _f64(D2)
    n = D1.shape[0]
    c1 = _f64(c1)
    c2 = _f64(c2)
    w = np.zeros(c1.size * s * n)
    _check(lib().orc_harvest_batch_vc(D1.reshape(-1), D2.reshape(-1), n, c1, c2, c1.size,
                                      float(delta_t), int(s), int(row), int(bool(reduced)), w,
                                      int(threads)), "harvest_batch_vc")
    return w.reshape(c1.size, s, n)


# --- stencil members (grid.py:136-175) ------------------------------------
def members_for(N, n, row, periodic):
    t = np.arange(N, dtype=np.int64)[:, None]
    j = np.arange(n, dtype=np.int64)[None, :]
    if periodic:
        return np.ascontiguousarray((t - row + j) % N)
    start = np.clip(t - row, 0, N - n)
    return np.ascontiguousarray(start + j)


def target_rows_for(N, n, row, periodic):
    if periodic:
        return np.full(N, row, dtype=np.int64)
    t = np.arange(N, dtype=np.int64)
    return t - np.clip(t - row, 0, N - n)


# --- kernels.py -----------------------------------------------------------
def _bc_args(bc):
    """bc: None | ('dirichlet', lo, hi) | ('neumann', dl, dr)."""
    if bc is None:
        return 0, 0.0, 0.0, None, None, ()
    if bc[0] == "dirichlet":
        return 1, float(bc[1]), float(bc[2]), None, None, ()
    dl, dr = _f64(bc[1]), _f64(bc[2])
    return 2, 0.0, 0.0, dl.ctypes.data, dr.ctypes.data, (dl, dr)


def banded_matvec(weights, members, u):
    w = _f64(weights)
    m = np.ascontiguousarray(members, dtype=np.int64)
    out = np.zeros(w.shape[0])
    lib().orc_banded_matvec(w, m, _f64(u), out, w.shape[0], w.shape[1])
    return out


def run_linear(weights, members, u0, steps, bc=None):
    w = _f64(weights)
    m = np.ascontiguousarray(members, dtype=np.int64)
    u0 = _f64(u0)
    out = np.zeros_like(u0)
    kind, lo, hi, dl, dr, keep = _bc_args(bc)
    lib().orc_run_linear(w, m, u0, u0.size, w.shape[1], int(steps), kind, lo, hi, dl, dr, out)
    return out


def run_etdrk4(w_full, w_alpha, w_beta, w_gamma, w_half, w_p1h, d1w, members, kind, u0, steps,
               bc=None):
    ws = [_f64(x) for x in (w_full, w_alpha, w_beta, w_gamma, w_half, w_p1h, d1w)]
    m = np.ascontiguousarray(members, dtype=np.int64)
    u0 = _f64(u0)
    out = np.zeros_like(u0)
    b, lo, hi, dl, dr, keep = _bc_args(bc)
    lib().orc_run_etdrk4(*ws, m, int(kind), u0, u0.size, ws[0].shape[1], int(steps), b, lo, hi,
                         dl, dr, out)
    return out


def run_etd2(ops, etd4_ops, d1w, members, kind, u0, steps, delta_t, bc=None, return_hist=False):
    """ops = (exp, dt*phi1, dt^2*phi2) raw rows; etd4_ops = (w, alpha, beta, gamma, wh, p1h)."""
    ws = [_f64(x) for x in list(ops[:3]) + list(etd4_ops) + [d1w]]
    m = np.ascontiguousarray(members, dtype=np.int64)
    u0 = _f64(u0)
    out = np.zeros_like(u0)
    hist = np.zeros_like(u0)
    b, lo, hi, dl, dr, keep = _bc_args(bc)
    lib().orc_run_etd2(*ws, m, int(kind), u0, u0.size, ws[0].shape[1], int(steps),
                       float(delta_t), b, lo, hi, dl, dr, out, hist.ctypes.data)
    return (out, hist) if return_hist else out


def etdrk4_operators(ops_full, ops_half, delta_t):
    """timestep.py:141-156 + harvest.py:225-235 (combine accumulates from zeros
    in list order).  ops_* are weight arrays (N, n)."""
    w, p1, p2, p3 = (_f64(x) for x in ops_full[:4])
    dt = float(delta_t)

    def combine(arrs, coeffs):
        acc = np.zeros_like(arrs[0])
        for a, c in zip(arrs, coeffs):
            acc = acc + c * a
        return acc

    alpha = combine([p1, p2, p3], [1.0, -3.0 / dt, 4.0 / dt**2])
    beta = combine([p2, p3], [2.0 / dt, -4.0 / dt**2])
    gamma = combine([p3, p2], [4.0 / dt**2, -1.0 / dt])
    return w, alpha, beta, gamma, _f64(ops_half[0]), _f64(ops_half[1])


def neumann_rows(n, h):
    """One-sided first-derivative rows for the zero-gradient closure
    (SURVEY Appendix B.2), built with the oracle's Fornberg restatement."""
    dl = fornberg_weights(0.0, np.arange(n) * h, 1)[1]
    dr = fornberg_weights(0.0, (np.arange(n) - (n - 1)) * h, 1)[1]
    return dl, dr


# --- compact rows (index arithmetic; full-size parity runs) ----------------
class Compact:
    """Operator rows in compact form on the select_stencils windows of
    (N, n, row, periodic): mode 0 shared [n], 1 classes [nleft+1+nright][n],
    2 per-node [N][n] (the reference's weights layout), 3 keyed rows [K][n]
    with node i using key cls[i] (the reference's exact-match harvest cache,
    harvest.py:135-159)."""

    def __init__(self, N, n, row, periodic, mode, nleft=0, nright=0, cls=None, nkeys=0):
        self._cls = None if cls is None else np.ascontiguousarray(cls, dtype=np.int32)
        self.nkeys = int(nkeys)
        self.geom = Geom(int(N), int(n), int(row), int(bool(periodic)), int(mode), int(nleft),
                         int(nright), None if self._cls is None else self._cls.ctypes.data)

    def rows(self, r):
        """Validate one operator's rows for this geometry."""
        r = _f64(r)
        g = self.geom
        want = {0: (g.n,), 1: (g.nleft + 1 + g.nright, g.n), 2: (g.N, g.n),
                3: (self.nkeys, g.n)}[g.mode]
        if r.shape != want and not (g.mode == 0 and r.shape == (1, g.n)):
            raise ValueError(f"rows of shape {r.shape}, expected {want}")
        return np.ascontiguousarray(r.reshape(-1))

    def dense(self, r):
        """The (N, n) array these compact rows stand for."""
        g = self.geom
        r = _f64(r)
        if g.mode == 0:
            return np.tile(r.reshape(1, g.n), (g.N, 1))
        if g.mode == 2:
            return r.reshape(g.N, g.n).copy()
        if g.mode == 3:
            return r.reshape(self.nkeys, g.n)[self._cls]
        out = np.tile(r[g.nleft].reshape(1, g.n), (g.N, 1))
        out[:g.nleft] = r[:g.nleft]
        if g.nright:
            out[g.N - g.nright:] = r[g.nleft + 1:]
        return out

    def run_linear(self, w, u0, steps, bc=None):
        u0 = _f64(u0)
        out = np.zeros_like(u0)
        kind, lo, hi, dl, dr, keep = _bc_args(bc)
        lib().orc_run_linear_c(C.byref(self.geom), self.rows(w), u0, int(steps), kind, lo, hi,
                               dl, dr, out)
        return out

    def _zeros(self):
        g = self.geom
        return np.zeros({0: g.n, 1: (g.nleft + 1 + g.nright) * g.n, 2: g.N * g.n,
                         3: self.nkeys * g.n}[g.mode])

    def run_etdrk4(self, ops, d1w, kind, u0, steps, bc=None, return_nl0=False):
        """ops = (w, alpha, beta, gamma, w_half, p1_half) compact rows."""
        rs = [self.rows(x) for x in ops] + [self._zeros() if d1w is None else self.rows(d1w)]
        u0 = _f64(u0)
        out = np.zeros_like(u0)
        nl0 = np.zeros_like(u0)
        b, lo, hi, dl, dr, keep = _bc_args(bc)
        lib().orc_run_etdrk4_c(C.byref(self.geom), *rs, int(kind), u0, int(steps), b, lo, hi,
                               dl, dr, out, nl0.ctypes.data)
        return (out, nl0) if return_nl0 else out

    def run_etd2(self, ops, warm, d1w, kind, u0, steps, delta_t, bc=None, return_hist=False):
        """ops = (exp, dt*phi1, dt^2*phi2) raw rows; warm = the ETDRK4 rows."""
        rs = [self.rows(x) for x in list(ops[:3]) + list(warm)]
        rs.append(self._zeros() if d1w is None else self.rows(d1w))
        u0 = _f64(u0)
        out = np.zeros_like(u0)
        hist = np.zeros_like(u0)
        b, lo, hi, dl, dr, keep = _bc_args(bc)
        lib().orc_run_etd2_c(C.byref(self.geom), *rs, int(kind), u0, int(steps), float(delta_t),
                             b, lo, hi, dl, dr, out, hist.ctypes.data)
        return (out, hist) if return_hist else out


def combine_rows(arrs, coeffs):
    """harvest.combine (harvest.py:225-235): from zeros, in list order, numpy's
    two roundings per term."""
    acc = np.zeros_like(_f64(arrs[0]))
    for a, c in zip(arrs, coeffs):
        acc = acc + float(c) * _f64(a)
    return acc


def etdrk4_rows(full, half, delta_t):
    """timestep.py:141-156 on any row arrays: (w, alpha, beta, gamma, w_half, p1_half)."""
    dt = float(delta_t)
    w, p1, p2, p3 = (_f64(x) for x in full[:4])
    return (w, combine_rows([p1, p2, p3], [1.0, -3.0 / dt, 4.0 / dt**2]),
            combine_rows([p2, p3], [2.0 / dt, -4.0 / dt**2]),
            combine_rows([p3, p2], [4.0 / dt**2, -1.0 / dt]), _f64(half[0]), _f64(half[1]))


def close(u, bc):
    """The boundary closure of the initial data (timestep.py:310-311 pin;
    Appendix B.2 zero-gradient closure), as apply_bc does it."""
    u = _f64(u).copy()
    if bc is None:
        return u
    if bc[0] == "dirichlet":
        u[0], u[-1] = bc[1], bc[2]
        return u
    dl, dr = _f64(bc[1]), _f64(bc[2])
    n, N = dl.size, u.size
    acc = 0.0
    for j in range(1, n):
        acc += dl[j] * u[j]
    u[0] = -acc / dl[0]
    acc = 0.0
    for j in range(n - 1):
        acc += dr[j] * u[N - n + j]
    u[N - 1] = -acc / dr[n - 1]
    return u
