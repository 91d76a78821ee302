"""Device timeline of one streamed run() at config 5 WITHOUT a profiler: every
event the pipeline records (uploads landed, harvests done, result landed) is made a
timing event and read back against the start of the call, next to the host time at
which it was queued; then the step interval of every slice.  Diagnostic only.

  python tools/e2e_events.py
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
import paper_2603_15964_b200 as lx
from paper_2603_15964_b200 import _ops
b = bench.C5(0, 1)
for _ in range(4): b.e2e_pass()
torch.cuda.synchronize()
evs=[]
orig = torch.cuda.Stream.record_event
def rec(self, event=None):
    if event is None:
        event = torch.cuda.Event(enable_timing=True)
    r = orig(self, event)
    evs.append((self.cuda_stream, time.perf_counter(), event))
    return r
torch.cuda.Stream.record_event = rec
keep=[]
init0=_ops.LinearStream.__init__
def init1(self,*a,**k):
    keep.append(self); init0(self,*a,**k)
_ops.LinearStream.__init__=init1
for rep in range(3):
    evs.clear(); keep.clear()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e0.record()
    t0=time.perf_counter()
    b.e2e_pass()
    t1=time.perf_counter()
    torch.cuda.synchronize()
    t2=time.perf_counter()
print(f"host returned {1e3*(t1-t0):.3f} ms, synced {1e3*(t2-t0):.3f}")
streams={}
for sid, th, ev in evs:
    try:
        streams.setdefault(sid,len(streams))
        print(f"stream{streams[sid]} host {1e3*(th-t0):7.3f} ms  gpu {e0.elapsed_time(ev):7.3f} ms")
    except Exception as ex:
        print("stream", sid, "host", 1e3*(th-t0), "untimed", ex)
ls=keep[-1]
for (eh, es),(a,bb) in zip(ls.marks, ls.bounds):
    print(f"slice [{a},{bb}) steps queued-after-harvest at gpu {e0.elapsed_time(eh):.3f} .. steps end {e0.elapsed_time(es):.3f}")
