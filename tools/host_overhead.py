"""Host-side overhead of one C5 device pass (ShardedStepper construction +
stepping): wall clock with syncs, the harvest kernel alone, and a cProfile
of the construction.  python tools/host_overhead.py"""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

torch.cuda.set_device(0)
b = bench.C5()
for _ in range(3):
    b.device_pass()
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter()
    b.device_pass()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    h, s = b.phase_ms()
    print(f"host enqueue {1e3*(t1-t0):.3f} ms, wall {1e3*(t2-t0):.3f} ms, events harvest {h:.3f} steps {s:.3f}")
pr = cProfile.Profile()
pr.enable()
b.device_pass()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
