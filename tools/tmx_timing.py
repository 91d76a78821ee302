"""Per-tile phase timestamps of lin_pernode_tmx_kernel (build liblmep with -DLMEP_TMX_TIMING:
  make -C paper_2603_15964_b200/csrc NVFLAGS="... -DLMEP_TMX_TIMING"), r2: wait 86, fill 1100,
issue 170, 25 steps 16300, store 950, gap 330 clk per tile."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2603_15964_b200 import _native as nat, _ops
from paper_2603_15964_b200.timestep import Stepper, prepare
from tools.prof_cases import setup
w, g, st, prob, scheme = setup("c5")
prep = prepare(g, st, prob, scheme, w.delta_t)
s = Stepper(prep, _ops.dev_f64(w.u0), exact=False)
s.advance(50); torch.cuda.synchronize()
s.advance(25); torch.cuda.synchronize()
buf = (C.c_longlong * 512)()
print("rc", nat.lib().lmep_debug_tmx_timing(buf))
a = np.array(buf[:]).reshape(2, 256)
for b in range(2):
    t = a[b, :180].reshape(30, 6)
    t = t[t[:, 0] > 0]
    print("block", b, "tiles", len(t))
    d = np.diff(t, axis=1)
    print("cols: wait, fill, issue, steps, store ; and gap to next tile")
    for i in range(len(t)):
        gap = t[i + 1, 0] - t[i, 5] if i + 1 < len(t) else 0
        print(i, d[i].tolist(), gap)
    print("mean", d.mean(0).round(0).tolist(), "total/tile", (t[-1, 5] - t[0, 0]) / len(t))
