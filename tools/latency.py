"""Per-call latency breakdown: device event time vs host time, and profile-mode kernel sum."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1609_04471_b200 as sr
from workloads import gen
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
for order in ["random", "reversed", "nearly", "few_unique", "sorted"]:
    src = torch.from_numpy(gen.make(order, n, np.int32, config=1)).cuda()
    w = torch.empty_like(src)
    flush = torch.empty(128 << 20, dtype=torch.int32, device="cuda")
    ev = []
    host = []
    for i in range(23):
        w.copy_(src); flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(); t0 = time.perf_counter(); sr.sort_keys(w); t1 = time.perf_counter(); b.record()
        torch.cuda.synchronize()
        if i >= 3: ev.append(a.elapsed_time(b) * 1e3); host.append((t1 - t0) * 1e6)
    sr.set_option(sr.OPT_PROFILE, 1)
    w.copy_(src); torch.cuda.synchronize(); sr.sort_keys(w); prof = sr.last_profile()
    sr.set_option(sr.OPT_PROFILE, 0)
    ks = sum(p[1] for p in prof) * 1e3
    print(f"{order:11s} event {np.median(ev):7.1f} us  host-in-call {np.median(host):7.1f} us  kernels(profiled) {ks:7.1f} us  "
          f"plan={sr.last_plan()['route_name']} launches={sr.last_plan()['launches']}")
    print("    ", ", ".join(f"{p[0]}={p[1]*1e3:.1f}" for p in prof))
