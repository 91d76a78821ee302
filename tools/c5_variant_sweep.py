"""C5 per-node steps: kernel variant x steps-per-launch sweep (FMA and exact).
  python tools/c5_variant_sweep.py [variants...]   (registers, registers2, window)"""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_15964_b200 import _native as nat, _ops
from paper_2603_15964_b200.timestep import Stepper, prepare
from tools.prof_cases import setup
w, g, st, prob, scheme = setup("c5")
prep = prepare(g, st, prob, scheme, w.delta_t)
ref = {}
for var in (sys.argv[1:] or ["registers", "registers2"]):
    nat.set_pernode_kernel(var)
    for exact in (False, True):
        for k in (10, 12, 14, 16, 18, 20, 22, 25, 29, 34):
            s = Stepper(prep, _ops.dev_f64(w.u0), exact=exact, tuning={"ksteps": k})
            s.advance(24)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record(); s.advance(200); e1.record(); torch.cuda.synchronize()
            key = exact
            same = None
            if exact:
                if key in ref: same = bool(torch.equal(ref[key], s.u))
                else: ref[key] = s.u.clone()
            print(json.dumps({"variant": var, "exact": exact, "k": k,
                              "us_per_step": round(e0.elapsed_time(e1) * 1e3 / 200, 3),
                              "bitwise_same_as_first": same}), flush=True)
