import sys, json, torch
sys.path.insert(0, '.')
from paper_2603_15964_b200 import _native as nat, _ops, configs
import paper_2603_15964_b200 as lx
from paper_2603_15964_b200.timestep import Stepper, prepare
from tools.prof_cases import setup
w, g, st, prob, scheme = setup("c5")
prep = prepare(g, st, prob, scheme, w.delta_t)
for var in ("window", "registers", "window", "registers"):
    nat.set_pernode_kernel(var)
    for exact in (False, True):
        s = Stepper(prep, _ops.dev_f64(w.u0), exact=exact)
        s.advance(16)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(); s.advance(200); e1.record(); torch.cuda.synchronize()
        print(json.dumps({"kernel": var, "exact": exact, "us_per_step": e0.elapsed_time(e1)*1e3/200}))
