"""run() from host arrays at config 5: the streamed pipeline (stream=True)
against the phase-by-phase order, wall time per pass, over slice plans.
Diagnostic only.

  python tools/e2e_stream.py [--exact] [--reps K]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import bench
    from paper_2603_15964_b200 import _ops
    import paper_2603_15964_b200 as lx
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 7
    b = bench.C5(0, 1, exact="--exact" in sys.argv)
    b.e2e_pass()
    spec = lx.VariableCoefficientSpec((1, 2), b.coef_pin)
    prob = lx.SemiLinearProblem(spec, None, b.u0_pin, lx.Boundary.periodic(), "none")

    def once(stream):
        return lx.run(b.grid, b.sset, prob, b.scheme, b.w.delta_t, b.w.steps * b.w.delta_t,
                      exact=b.exact, stream=stream)

    def timed(stream):
        for _ in range(2):
            once(stream)
        ms = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = once(stream)
            torch.cuda.synchronize()
            ms.append((time.perf_counter() - t0) * 1e3)
        return float(np.median(ms)), float(np.min(ms)), r

    m, lo, ref = timed(False)
    print(f"phases:   median {m:.3f} ms  min {lo:.3f}  harvest_ns {ref.harvest_ns} step_ns {ref.step_ns}")
    plans = [(1, 4, 7, 7), (1, 3, 6, 6, 4), (1, 3, 5, 5, 5), (1, 3, 4, 5, 5, 3), (1, 2, 3, 4, 5, 5),
             (1, 3, 4, 4, 4, 4), (1, 2, 4, 5, 5, 3), (1, 3, 4, 5, 4, 3, 1.5), (1, 2, 3, 4, 4, 4, 3),
             (1, 3, 5, 6, 4, 2), (0.5, 1.5, 3, 4, 5, 5, 2), (1, 3, 4, 5, 6, 2.5)]
    if "--last-min" in sys.argv:
        _ops.LinearStream.LAST_MIN = float(sys.argv[sys.argv.index("--last-min") + 1])
    for wv in plans:
        _ops.LinearStream.WAVES = wv
        m, lo, r = timed(True)
        same = np.array_equal(r.snapshots, ref.snapshots)
        print(f"stream {wv}: median {m:.3f} ms  min {lo:.3f}  harvest_ns {r.harvest_ns} "
              f"step_ns {r.step_ns}  bitwise {same}")


if __name__ == "__main__":
    main()
