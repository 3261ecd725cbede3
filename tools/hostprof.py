"""Host-side cost of one resident-path call: SR_HOSTPROF step times + event/host totals."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1609_04471_b200 as sr
from workloads import gen
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
src = torch.from_numpy(gen.make("random", n, np.int32, config=1)).cuda()
w = torch.empty_like(src)
for i in range(8):
    w.copy_(src); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); t0 = time.perf_counter(); sr.sort_keys(w); t1 = time.perf_counter(); b.record(); torch.cuda.synchronize()
    print(f"call {i}: event {a.elapsed_time(b)*1e3:.1f} us, host {(t1-t0)*1e6:.1f} us", file=sys.stderr, flush=True)
