"""Time sorts of one workload under several SR_OPT_TUNE settings (device events, L2 flushed, output checked).

usage: python tools/ab_tune.py N ORDER DTYPE REPS "i=v,i=v" ["i=v" ...]   (empty string = defaults)
Prints per setting: mean / min ms, Mkeys/s, route, levels, and the per-kernel profile of the last rep."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1609_04471_b200 as sr

n, order, dt, reps = int(sys.argv[1]), sys.argv[2], np.dtype(sys.argv[3]), int(sys.argv[4])
settings = sys.argv[5:] or [""]
code = {"random": 0, "reversed": 1, "nearly": 2, "few_unique": 3}.get(order, 0)
src = torch.empty(n, dtype=torch.int32 if dt == np.int32 else torch.int64, device="cuda")
sr.generate(src, order, seed=12345, param=int(os.environ.get("GEN_PARAM", "0")))
work = torch.empty_like(src)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ref = None
DEF = {0: 0, 1: 512, 2: 256, 3: 0, 4: 0, 5: 2, 6: 0, 7: 0}
for st in settings:
    kv = dict(DEF)
    for p in filter(None, st.split(",")):
        i, v = p.split("=")
        kv[int(i)] = int(v)
    for i, v in kv.items():
        sr.set_option(sr.OPT_TUNE + i, v)
    ts = []
    for r in range(reps + 2):
        work.copy_(src)
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        sr.sort_keys(work)
        b.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(a.elapsed_time(b))
    if ref is None:
        ref = work.clone()
        ok = bool((ref[1:] >= ref[:-1]).all().item())
    else:
        ok = bool(torch.equal(ref, work))
    p = sr.last_plan()
    sr.set_option(sr.OPT_PROFILE, 1)
    work.copy_(src); flush.zero_(); torch.cuda.synchronize()
    sr.sort_keys(work); torch.cuda.synchronize()
    prof = sr.last_profile()
    sr.set_option(sr.OPT_PROFILE, 0)
    ts = np.array(ts)
    print(f"[{st or 'default'}] n={n} {order} {dt.name}: mean {ts.mean():.3f} ms min {ts.min():.3f} -> "
          f"{n / ts.mean() / 1e3:.1f} Mkeys/s route={p['route_name']} levels={p['levels']} ok={ok}", flush=True)
    agg = {}
    for name, ms, by in prof:
        a_ = agg.setdefault(name, [0, 0.0, 0])
        a_[0] += 1; a_[1] += ms; a_[2] += by
    print("   " + "  ".join(f"{k}:{v[1]:.3f}ms/{v[0]}" for k, v in sorted(agg.items(), key=lambda x: -x[1][1])), flush=True)
for i, v in DEF.items():
    sr.set_option(sr.OPT_TUNE + i, v)
