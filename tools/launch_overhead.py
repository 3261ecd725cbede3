import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1609_04471_b200 as sr
from workloads import gen
x = torch.zeros(1, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(1000): x.add_(1)
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"torch launch: {(t1-t0)*1e3:.1f} us/launch enqueue, {(t2-t0)*1e3:.1f} us/launch incl drain")
for order in ["sorted", "random"]:
    src = torch.from_numpy(gen.make(order, 2_000_000, np.int32, config=1)).cuda()
    w = torch.empty_like(src)
    for i in range(6):
        w.copy_(src); torch.cuda.synchronize()
        sr.sort_keys(w); torch.cuda.synchronize()
