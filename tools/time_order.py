"""Time sort_keys on one generated order (device events, L2 flushed, output checked vs a reference sort).
usage: python tools/time_order.py N ORDER DTYPE PARAM [opt=value ...]   (opt: sr.OPT_* numeric key)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1609_04471_b200 as sr
n, order, dt, param = int(sys.argv[1]), sys.argv[2], sys.argv[3], int(sys.argv[4])
for kv in sys.argv[5:]:
    k, v = kv.split("=")
    sr.set_option(int(k), int(v))
src = torch.empty(n, dtype=getattr(torch, dt), device="cuda")
sr.generate(src, order, seed=77, param=param)
ref = torch.sort(src).values
work = torch.empty_like(src)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ts = []
for r in range(12):
    work.copy_(src); flush.zero_(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); sr.sort_keys(work); b.record(); torch.cuda.synchronize()
    if r >= 2: ts.append(a.elapsed_time(b))
ok = torch.equal(work, ref)
ts = np.array(ts)
print(f"n={n} {order}({param}) {dt} {sys.argv[5:]}: mean {ts.mean()*1e3:.1f} us min {ts.min()*1e3:.1f} -> "
      f"{n / ts.mean() / 1e3:.0f} Mkeys/s route={sr.last_plan()['route_name']} ok={ok}", flush=True)
