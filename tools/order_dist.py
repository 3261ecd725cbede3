"""Per-sort device times of one C2 order, timed as bench.py does (input
restored, 512 MiB L2 flush, then events around the sort with no host sync in
between): prints the distribution.  usage: python tools/order_dist.py ORDER [N] [REPS]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1609_04471_b200 as sr
from workloads import gen
order = sys.argv[1]
prev = os.environ.get("PREV")  # another order sorted (untimed) before every timed sort, as in bench.py's step
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2_000_000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 60
src = torch.from_numpy(gen.make(order, n, np.int32, config=1)).cuda()
work = torch.empty_like(src)
psrc = torch.from_numpy(gen.make(prev, n, np.int32, config=1)).cuda() if prev else None
pwork = torch.empty_like(src)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
for i in range(reps):
    if psrc is not None:
        pwork.copy_(psrc)
        flush.fill_(i)
        sr.sort_keys(pwork)
        keep = pwork.clone()
    work.copy_(src)
    flush.fill_(i)
    ev[i][0].record(st)
    sr.sort_keys(work)
    ev[i][1].record(st)
torch.cuda.synchronize()
t = np.array([a.elapsed_time(b) * 1e3 for a, b in ev[5:]])
print(f"{order}: mean {t.mean():.1f} us  min {t.min():.1f}  p50 {np.median(t):.1f}  p90 {np.percentile(t, 90):.1f}  max {t.max():.1f}")
print(" ".join(f"{x:.0f}" for x in t))
