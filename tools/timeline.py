"""Device timeline of one config-5 device pass (bench.C5.device_pass) from the
torch profiler: every kernel / copy with its start offset and duration, so the
gaps between the harvest and the steps show up.  Diagnostic only.

  python tools/timeline.py [--exact] [--e2e]   (--e2e: the run() pass from host arrays)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile
    import bench
    b = bench.C5(0, 1, exact="--exact" in sys.argv)
    fn = b.e2e_pass if "--e2e" in sys.argv else b.device_pass
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        fn()
        torch.cuda.synchronize()
    path = "/tmp/c5_trace.json"
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"]
          if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e]
    ev.sort(key=lambda e: e["ts"])
    t0 = ev[0]["ts"]
    prev_end = t0
    for e in ev:
        gap = e["ts"] - prev_end
        print(f"{e['ts'] - t0:9.1f} us  +gap {gap:7.1f}  dur {e['dur']:8.1f}  s{e.get('args', {}).get('stream', '?')}  {e['name'][:80]}")
        prev_end = max(prev_end, e["ts"] + e["dur"])
    print(f"span {prev_end - t0:.1f} us, busy {sum(e['dur'] for e in ev):.1f} us")


if __name__ == "__main__":
    main()
