"""Run a few sorts of one workload/order (for ncu captures): warmup sorts, then ONE profiled sort."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1609_04471_b200 as sr
from workloads import gen

ap = argparse.ArgumentParser()
ap.add_argument("--order", default="random")
ap.add_argument("--n", type=int, default=2_000_000)
ap.add_argument("--dtype", default="int32")
ap.add_argument("--pairs", action="store_true")
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--route", type=int, default=0)
ap.add_argument("--flush", action="store_true", help="write 512 MiB before every sort (as bench.py)")
ap.add_argument("--prewarm", type=int, default=0, help="after the flush, sort this many random keys first")
a = ap.parse_args()
dt = np.dtype(a.dtype)
k = gen.make(a.order, a.n, dt, config=1)
src = torch.from_numpy(k).cuda()
work = torch.empty_like(src)
v = torch.arange(a.n, dtype=torch.int32, device="cuda")
vw = torch.empty_like(v)
sr.set_option(sr.OPT_FORCE_ROUTE, a.route)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda") if a.flush else None
pre = torch.from_numpy(gen.make("random", max(a.prewarm, 1), dt, config=2)).cuda()
pre_w = torch.empty_like(pre)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for i in range(a.warmup + 1):
    work.copy_(src)
    vw.copy_(v)
    if flush is not None:
        flush.fill_(i)
    if a.prewarm:
        pre_w.copy_(pre)
        sr.sort_keys(pre_w)
    torch.cuda.synchronize()
    ev[0].record()
    if a.pairs:
        sr.sort_pairs(work, vw)
    else:
        sr.sort_keys(work)
    ev[1].record()
    torch.cuda.synchronize()
print(sr.last_plan())
print(f"last sort: {ev[0].elapsed_time(ev[1]) * 1e3:.1f} us (events)")
