"""Small, fast invocations of each hot kernel for timing sweeps and ncu.

  python tools/prof_cases.py harvest|c3|c4|c5step|c1|c2 [--reps R] [--tile T --k K] [--fma]
Prints one JSON line with the per-launch time measured by CUDA events.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_15964_b200 as lx  # noqa: E402
from paper_2603_15964_b200 import configs, _ops  # noqa: E402
from paper_2603_15964_b200.timestep import Stepper, prepare  # noqa: E402


def setup(name, N=None):
    w = configs.make(name) if N is None else configs.make(name, N=N)
    g = lx.make_periodic_grid(w.N, w.x_min, w.x_max) if w.periodic else \
        lx.make_uniform_grid(w.N, w.x_min, w.x_max)
    pol = lx.StencilPolicy.ONE_SIDED_UPWIND if w.policy == "upwind" else lx.StencilPolicy.CENTERED
    st = lx.select_stencils(g, w.n, pol)
    if name == "c5":
        c, nu = w.coef
        spec = lx.VariableCoefficientSpec((1, 2), np.stack([-c, nu], 1))
    else:
        spec = lx.LinearOperatorSpec(w.terms)
    bc = lx.Boundary.neumann() if w.boundary == "neumann" else lx.Boundary.periodic()
    prob = lx.SemiLinearProblem(spec, None, w.u0, bc, w.nonlinear, nonlinear_scale=w.nl_scale or 1.0)
    scheme = {"linear": lx.SchemeConfig("linear"), "etdrk4": lx.SchemeConfig("etdrk4"),
              "etd2": lx.SchemeConfig("etd-multistep", s=2)}[w.scheme]
    return w, g, st, prob, scheme


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--tile", type=int, default=0)
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--fma", action="store_true")
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--method", default="multiply")
    ap.add_argument("--N", type=int, default=None)
    ap.add_argument("--s", type=int, default=1, help="harvest: phi rows (1 = w_lin only)")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if a.case == "harvest":
        from paper_2603_15964_b200 import _native
        _native.set_harvest_method(a.method)
        w, g, st, prob, scheme = setup("c5", N=a.N or (1 << 20))
        c, nu = w.coef                      # resident coefficients: time the device path only
        spec = lx.VariableCoefficientSpec((1, 2), _ops.dev_f64(np.stack([-c, nu], 1)))
        prob = lx.SemiLinearProblem(spec, None, w.u0, lx.Boundary.periodic(), "none")
        from paper_2603_15964_b200.grid import as_stencil_set
        from paper_2603_15964_b200.harvest import harvest_compact
        sset = as_stencil_set(g, st)

        def once():
            return harvest_compact(g, sset, spec, w.delta_t, a.s)
        for _ in range(2):
            once()
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(a.reps):
            once()
        ev1.record()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1) / a.reps
        print(json.dumps({"case": "harvest", "method": a.method, "N": w.N, "s": a.s, "ms": ms,
                          "harvests_per_s": w.N / ms * 1e3}))
        return
    name = {"c3": "c3", "c4": "c4", "c5step": "c5", "c1": "c1", "c2": "c2"}[a.case]
    w, g, st, prob, scheme = setup(name, N=a.N)
    prep = prepare(g, st, prob, scheme, w.delta_t)
    tun = {"tile": a.tile, "ksteps": a.k, "threads": a.threads} if (a.tile or a.k or a.threads) else None
    s = Stepper(prep, _ops.dev_f64(w.u0), exact=not a.fma, tuning=tun)
    s.advance(3)
    torch.cuda.synchronize()
    ev0.record()
    s.advance(a.reps)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / a.reps
    print(json.dumps({"case": a.case, "N": w.N, "us_per_step": ms * 1e3,
                      "updates_per_s": w.N / ms * 1e3, "tile": a.tile, "k": a.k, "fma": a.fma, "threads": a.threads,
                      "finite": bool(torch.isfinite(s.u).all())}))


if __name__ == "__main__":
    main()
