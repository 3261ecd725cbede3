"""One small sort on every route (for compute-sanitizer memcheck / racecheck /
synccheck runs): resident one-launch partition (keys int32 /
int64), multi-kernel partition, merge (forced), outlier, reversed, sorted,
stable pairs, float keys, record keys, presortedness measures.  Each output is
checked against the oracle; exits non-zero on a mismatch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1609_04471_b200 as sr  # noqa: E402
from workloads import gen  # noqa: E402

N = int(os.environ.get("SR_SAN_N", 1 << 18))
bad = 0


def check(name, got, exp):
    global bad
    ok = np.array_equal(got, exp)
    bad += 0 if ok else 1
    print(f"{name:40s} route={sr.last_plan()['route_name']:9s} {'ok' if ok else 'MISMATCH'}", flush=True)


def keys(name, k, route=0, resident=1):
    sr.set_option(sr.OPT_FORCE_ROUTE, route)
    sr.set_option(sr.OPT_RESIDENT, resident)
    d = torch.from_numpy(k.copy()).cuda()
    sr.sort_keys(d)
    torch.cuda.synchronize()
    check(name, d.cpu().numpy(), oracle.sort_keys(k))
    sr.set_option(sr.OPT_FORCE_ROUTE, 0)
    sr.set_option(sr.OPT_RESIDENT, 1)


for dt in (np.int32, np.int64):
    for order in ("random", "nearly", "few_unique", "reversed", "sorted", "organ_pipe"):
        keys(f"resident {np.dtype(dt).name} {order}", gen.make(order, N, dt, config=1))
    keys(f"multi-kernel partition {np.dtype(dt).name}", gen.make("random", N, dt, config=1), resident=0)
    keys(f"forced merge {np.dtype(dt).name}", gen.make("runs1024", N, dt, config=2), route=sr.ROUTE_MERGE, resident=0)
    keys(f"forced partition {np.dtype(dt).name}", gen.make("runs1024", N, dt, config=2), route=sr.ROUTE_PARTITION,
         resident=0)
keys("outlier (multi-kernel)", gen.make("swaps_1e4", 4 * N, np.int32, config=2), resident=0)
keys("tile route (n <= 8192)", gen.make("random", 5000, np.int32, config=1))
k = gen.make("few100", N, np.int32, config=3)
v = gen.index_payload(N)
for resident in (1, 0):
    dk, dv = torch.from_numpy(k.copy()).cuda(), torch.from_numpy(v.view(np.int32).copy()).cuda()
    sr.sort_pairs(dk, dv)
    torch.cuda.synchronize()
    ek, ev = oracle.sort_pairs(k, v)
    check("pairs few100", np.concatenate([dk.cpu().numpy(), dv.cpu().numpy().view(np.int32)]),
          np.concatenate([ek, ev.view(np.int32)]))
kf = gen.make_float("fbits", N, np.float32, config=40)
df = torch.from_numpy(kf.copy()).cuda()
sr.sort_keys(df)
torch.cuda.synchronize()
check("float32 bits", df.cpu().numpy().view(np.uint32), oracle.sort_keys(kf).view(np.uint32))
rec = gen.make_list("lprefix", N // 16, 8, config=60)
dr = torch.from_numpy(rec.copy()).cuda()
sr.sort_records(dr)
torch.cuda.synchronize()
check("records lprefix x8", dr.cpu().numpy(), oracle.sort_records(rec))
km = gen.make("nearly", N // 4, np.int32, config=71)
m = sr.presortedness(torch.from_numpy(km).cuda())
got = [m[f] for f in ("runs", "inversions", "mono", "max_dis", "misplaced")]
exp = oracle.measures(km)
check("presortedness measures", np.array(got), np.array([exp[f] for f in ("runs", "inversions", "mono", "max_dis",
                                                                          "misplaced")]))
print("sanitize cases:", "ok" if bad == 0 else f"{bad} mismatches")
sys.exit(1 if bad else 0)
