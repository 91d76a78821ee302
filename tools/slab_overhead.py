"""One config-4-sized slab (2^21 nodes, ETDRK4 cubic) stepped as a rank of a sharded run: a periodic
1-rank ring exchanging with itself through the library communicator (NCCL with graph replay, peer
mailboxes with fused stores), against the unsharded stepper on the same grid.  Diagnostic."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_15964_b200 as lx
from paper_2603_15964_b200 import _ops, _native as nat
from paper_2603_15964_b200.distributed import Comm, CommHalo, ShardedStepper, advance_all
from paper_2603_15964_b200.timestep import Stepper, prepare
N = 1 << 21                                   # one eighth of config 4, periodic so that one rank can ring with itself
g = lx.make_periodic_grid(N, -1.0, 1.0)
st = lx.select_stencils(g, 7, lx.StencilPolicy.CENTERED)
rng = np.random.default_rng(4)
u0 = 0.1 * rng.uniform(-1, 1, N)
prob = lx.SemiLinearProblem(lx.LinearOperatorSpec(((0, 1.0), (2, 1e-4))), None, u0, lx.Boundary.periodic(), "cubic")
h = 2.0 / N
dt = 0.5 * h * h / 1e-4
scheme = lx.SchemeConfig("etdrk4")
for exact in (False, True):
    ref = Stepper(prepare(g, st, prob, scheme, dt), _ops.dev_f64(u0), exact=exact)
    ref.advance(24); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ref.advance(240); e1.record(); torch.cuda.synchronize()
    base = e0.elapsed_time(e1) * 1e3 / 240
    out = {"exact": exact, "unsharded_us_per_step": round(base, 2)}
    for transport in ("nccl", "nccl-eager", "peer"):
        if transport.startswith("nccl"):
            c = Comm(0, 1, True, "nccl", unique_id=Comm.unique_id())
        else:
            c = Comm(0, 1, True, "peer", max_width=4096); c.connect([c.export()])
        s = ShardedStepper(g, st, prob, scheme, dt, 0, 1, CommHalo(c), exact=exact, force_halo=True,
                           graph=(transport == "nccl"))
        s.set_initial(u0)
        own = torch.cuda.Stream(); own.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(own):
            advance_all(s, 24); torch.cuda.synchronize()
            e0.record(own); advance_all(s, 240); e1.record(own)
        torch.cuda.synchronize()
        out[transport + "_us_per_step"] = round(e0.elapsed_time(e1) * 1e3 / 240, 2)
        out[transport + "_graphs"] = len(s._graphs)
        assert torch.equal(s.u, ref.u) or not exact
        s._graphs.clear(); c.close()
    print(json.dumps(out))
