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
a = ap.parse_args()
dt = np.dtype(a.dtype)
k = gen.make(a.order, a.n, dt, config=1)
src = torch.from_numpy(k).cuda()
work = torch.empty_like(src)
v = torch.arange(a.n, dtype=torch.int32, device="cuda")
vw = torch.empty_like(v)
sr.set_option(sr.OPT_FORCE_ROUTE, a.route)
for i in range(a.warmup + 1):
    work.copy_(src)
    vw.copy_(v)
    torch.cuda.synchronize()
    if a.pairs:
        sr.sort_pairs(work, vw)
    else:
        sr.sort_keys(work)
    torch.cuda.synchronize()
print(sr.last_plan())
