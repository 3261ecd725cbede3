import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1609_04471_b200 as sr
from workloads import gen
n = int(sys.argv[1]); order = sys.argv[2]; dt = np.dtype(sys.argv[3])
k = gen.make(order, n, dt, config=3)
src = torch.from_numpy(k).cuda(); v0 = torch.arange(n, dtype=torch.int32, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ref = None
for cap in [0, 2048, 1024, 512, 256, 128, 64]:
    sr.set_option(sr.OPT_TUNE + 3, cap)
    ts = []
    for r in range(6):
        w = src.clone(); v = v0.clone(); flush.zero_(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); sr.sort_pairs(w, v); b.record(); torch.cuda.synchronize()
        if r >= 2: ts.append(a.elapsed_time(b))
    if ref is None: ref = (w.clone(), v.clone())
    ok = torch.equal(ref[0], w) and torch.equal(ref[1], v)
    print(f"pairs {order} n={n} {dt} cap={cap}: mean {np.mean(ts):.3f} ms levels={sr.last_plan()['levels']} same={ok}")
