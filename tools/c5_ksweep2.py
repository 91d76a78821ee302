"""Registers kernel, FMA: steps per launch sweep (plan spreads S steps evenly)."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_15964_b200 import _native as nat, _ops
from paper_2603_15964_b200.timestep import Stepper, prepare
from tools.prof_cases import setup
w, g, st, prob, scheme = setup("c5")
prep = prepare(g, st, prob, scheme, w.delta_t)
for exact in (False, True):
    for k in (22, 25, 28, 30, 34, 40, 50, 67):
        s = Stepper(prep, _ops.dev_f64(w.u0), exact=exact, tuning={"ksteps": k})
        s.advance(24)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(); s.advance(200); e1.record(); torch.cuda.synchronize()
        print(json.dumps({"exact": exact, "k": k, "us_per_step": round(e0.elapsed_time(e1) * 1e3 / 200, 3)}))
