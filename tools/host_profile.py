"""Host-side (Python) cost of one config-5 device pass: cProfile of
bench.C5.device_pass after warm-up, top functions by cumulative time.
Diagnostic only."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import bench
    b = bench.C5(0, 1)
    for _ in range(3):
        b.device_pass()
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(5):
        b.device_pass()
        torch.cuda.synchronize()          # each pass starts on an idle device, as in bench.py
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(45)
    pstats.Stats(pr).sort_stats("tottime").print_stats(15)


if __name__ == "__main__":
    main()
