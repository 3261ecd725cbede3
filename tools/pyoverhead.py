"""Host cost of the Python binding per call (what bench's events include before the launch)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes
import torch
import paper_1609_04471_b200 as sr
t1 = torch.zeros(1, dtype=torch.int32, device="cuda")
t2 = torch.zeros(2_000_000, dtype=torch.int32, device="cuda")
torch.cuda.synchronize()
def T(name, f, R=2000):
    for _ in range(50): f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(R): f()
    t = (time.perf_counter() - t0) / R * 1e6
    torch.cuda.synchronize()
    print(f"{name:40s} {t:7.2f} us/call")
T("sr.sort_keys(n=1)", lambda: sr.sort_keys(t1))
T("torch.cuda.current_stream()", lambda: torch.cuda.current_stream(t1.device).cuda_stream)
T("t.data_ptr()", lambda: t1.data_ptr())
lib = sr.lib()
T("lib.sr_sort_keys direct (n=1)", lambda: lib.sr_sort_keys(ctypes.c_void_p(t1.data_ptr()), 1, 0, None))
ev = torch.cuda.Event(enable_timing=True)
T("event.record()", lambda: ev.record())
T("sr.sort_keys(n=2M sorted)", lambda: sr.sort_keys(t2), R=200)
T("lib.sr_sort_keys direct (n=2M sorted)", lambda: lib.sr_sort_keys(ctypes.c_void_p(t2.data_ptr()), t2.numel(), 0, None), R=200)
