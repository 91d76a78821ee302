"""Host-side timeline of one streamed run() at config 5: when (wall clock, from
the call) the host reaches each stage of the pipeline.  Diagnostic only."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import bench
    from paper_2603_15964_b200 import _ops, harvest, timestep
    import paper_2603_15964_b200 as lx
    b = bench.C5(0, 1)
    b.e2e_pass()
    spec = lx.VariableCoefficientSpec((1, 2), b.coef_pin)
    prob = lx.SemiLinearProblem(spec, None, b.u0_pin, lx.Boundary.periodic(), "none")
    log = []
    t0 = [0.0]

    def wrap(obj, name, tag=None):
        f = getattr(obj, name)

        def g(*a, **k):
            log.append((time.perf_counter() - t0[0], "> " + (tag or name)))
            r = f(*a, **k)
            log.append((time.perf_counter() - t0[0], "< " + (tag or name)))
            return r
        setattr(obj, name, g)

    keep = []
    init0 = _ops.LinearStream.__init__

    def init1(self, *a, **k):
        keep.append(self)
        init0(self, *a, **k)
    _ops.LinearStream.__init__ = init1
    wrap(_ops.LinearStream, "__init__", "LinearStream()")
    wrap(_ops.LinearStream, "begin")
    wrap(_ops.LinearStream, "ready")
    wrap(_ops.LinearStream, "close")
    wrap(_ops, "harvest")
    wrap(harvest, "_tables_for")
    wrap(harvest, "_plan")
    wrap(harvest, "_checked_nodes")
    wrap(harvest, "_harvest_pipelined")
    wrap(timestep, "prepare")
    wrap(_ops, "check_deferred")

    def once():
        return lx.run(b.grid, b.sset, prob, b.scheme, b.w.delta_t, b.w.steps * b.w.delta_t,
                      exact=False)
    for _ in range(3):
        once()
    torch.cuda.synchronize()
    log.clear()
    t0[0] = time.perf_counter()
    once()
    end = time.perf_counter() - t0[0]
    for t, what in log:
        print(f"{t * 1e3:8.3f} ms  {what}")
    print(f"{end * 1e3:8.3f} ms  run() returned")
    ls = keep[-1]
    print("slices", ls.bounds)
    e0 = ls.marks[0][0]
    prev = e0
    for (eh, es), (a, bnd) in zip(ls.marks, ls.bounds):
        print(f"slice [{a},{bnd}): harvest done at +{e0.elapsed_time(eh):.3f} ms (since prev steps end "
              f"{prev.elapsed_time(eh):.3f}), steps {eh.elapsed_time(es):.3f} ms")
        prev = es


if __name__ == "__main__":
    main()
