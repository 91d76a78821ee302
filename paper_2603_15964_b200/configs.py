"""The five BASELINE.json workloads as concrete seeded synthetic inputs.

Restates SURVEY.md section 8(d): grids, stencil policies, operator specs,
schemes, stabilised time steps (Appendix B.1) and the seeded initial data
(``np.random.default_rng(seed)``, draws in the listed order, seeds 1-5).
No public dataset is involved; these are synthetic stand-ins with the
configs' shapes, sizes and value distributions.  ``N`` can be overridden to
build the same workload family at test sizes.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    N: int
    n: int
    x_min: float
    x_max: float
    periodic: bool
    policy: str              # "centered" | "upwind"
    terms: tuple             # LinearOperatorSpec terms (constant-coefficient configs)
    nonlinear: str           # "none" | "convective" | "cubic"
    nl_scale: float          # N(u) = -nl_scale * u * D1 u  (KdV: 6)
    scheme: str              # "linear" | "etdrk4" | "etd2"
    delta_t: float
    steps: int
    boundary: str            # "periodic" | "neumann"
    u0: np.ndarray = field(repr=False)
    coef: tuple | None = field(default=None, repr=False)   # C5: (c(x), nu(x)) per node

    @property
    def h(self) -> float:
        if self.periodic:
            return (self.x_max - self.x_min) / self.N
        return (self.x_max - self.x_min) / (self.N - 1)

    @property
    def nodes(self) -> np.ndarray:
        if self.periodic:
            return self.x_min + self.h * np.arange(self.N)
        return np.linspace(self.x_min, self.x_max, self.N)

    @property
    def row(self) -> int:
        return self.n - 1 if self.policy == "upwind" else (self.n - 1) // 2


def _periodic_nodes(N, a, b):
    return a + ((b - a) / N) * np.arange(N)


def c1(N: int = 1024, steps: int = 1000) -> Workload:
    """Linear advection, upwind n=7, CFL 3.5."""
    rng = np.random.default_rng(1)
    k = np.arange(1, 9)
    a = rng.standard_normal(8) / k
    theta = rng.uniform(0.0, 2.0 * math.pi, 8)
    x = _periodic_nodes(N, 0.0, 2.0 * math.pi)
    u0 = np.zeros(N)
    for i in range(8):
        u0 += a[i] * np.sin(k[i] * x + theta[i])
    h = 2.0 * math.pi / N
    return Workload("c1-advection", N, 7, 0.0, 2.0 * math.pi, True, "upwind", ((1, -1.0),),
                    "none", 0.0, "linear", 3.5 * h, steps, "periodic", u0)


def c2(N: int = 65536, steps: int = 5000) -> Workload:
    """Viscous Burgers, centred n=9, ETD2, mu = nu dt/h^2 = 0.5 (C2)."""
    rng = np.random.default_rng(2)
    k = np.arange(1, 17)
    theta = rng.uniform(0.0, 2.0 * math.pi, 16)
    x = _periodic_nodes(N, 0.0, 2.0 * math.pi)
    u0 = np.sin(x)
    for i in range(16):
        u0 += (0.1 / k[i]) * np.sin(k[i] * x + theta[i])
    nu = 0.01
    h = 2.0 * math.pi / N
    return Workload("c2-burgers", N, 9, 0.0, 2.0 * math.pi, True, "centered", ((2, nu),),
                    "convective", 1.0, "etd2", 0.5 * h * h / nu, steps, "periodic", u0)


def c3(N: int = 1 << 20, steps: int = 2000) -> Workload:
    """KdV two-soliton, centred n=11, ETDRK4, dt = 0.05 h^3 (C3)."""
    rng = np.random.default_rng(3)
    cs = rng.uniform(0.5, 4.0, 2)
    xs = rng.uniform(-15.0, 15.0, 2)
    x = _periodic_nodes(N, -20.0, 20.0)
    u0 = np.zeros(N)
    for ci, xi in zip(cs, xs):
        u0 += (ci / 2.0) / np.cosh(math.sqrt(ci) / 2.0 * (x - xi)) ** 2
    h = 40.0 / N
    return Workload("c3-kdv", N, 11, -20.0, 20.0, True, "centered", ((3, -1.0),),
                    "convective", 6.0, "etdrk4", 0.05 * h ** 3, steps, "periodic", u0)


def c4(N: int = 1 << 24, steps: int = 1000) -> Workload:
    """Allen-Cahn, uniform non-periodic, centred n=7 with clamped boundary
    classes, Neumann (frozen-row harvest + zero-gradient closure), ETDRK4,
    mu = eps^2 dt/h^2 = 0.5 (C4)."""
    rng = np.random.default_rng(4)
    u0 = 0.1 * rng.uniform(-1.0, 1.0, N)
    eps2 = 1e-4
    h = 2.0 / (N - 1)
    return Workload("c4-allen-cahn", N, 7, -1.0, 1.0, False, "centered", ((0, 1.0), (2, eps2)),
                    "cubic", 1.0, "etdrk4", 0.5 * h * h / eps2, steps, "neumann", u0)


def _smooth_field(rng, x):
    k = np.arange(1, 9)
    a = rng.standard_normal(8)
    b = rng.standard_normal(8)
    f = np.zeros_like(x)
    for i in range(8):
        f += (a[i] * np.cos(2 * math.pi * k[i] * x) + b[i] * np.sin(2 * math.pi * k[i] * x)) / k[i]
    return f


def c5(N: int = 1 << 22, steps: int = 200) -> Workload:
    """Variable-coefficient advection-diffusion, one exponential per node,
    frozen-at-target L_i = -c_i D1 + nu_i D2 (Appendix B.3), linear, mu_max = 0.5 (C5)."""
    rng = np.random.default_rng(5)
    x = _periodic_nodes(N, 0.0, 1.0)
    f = _smooth_field(rng, x)
    c = 2.0 * (2.0 * (f - f.min()) / (f.max() - f.min()) - 1.0)
    g = _smooth_field(rng, x)
    nu = 10.0 ** (-4.0 + 3.0 * (g - g.min()) / (g.max() - g.min()))
    u = _smooth_field(rng, x)
    u0 = u / np.abs(u).max()
    h = 1.0 / N
    return Workload("c5-varcoef", N, 13, 0.0, 1.0, True, "centered", (), "none", 0.0, "linear",
                    0.5 * h * h / 0.1, steps, "periodic", u0, coef=(c, nu))


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}


def make(name: str, **kw) -> Workload:
    return CONFIGS[name](**kw)
