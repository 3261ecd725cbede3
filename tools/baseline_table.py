"""Print BASELINE.md §4's results rows from a directory of bench.py lines
(usage: python tools/baseline_table.py profiles/r2s5_bench)."""
import glob, json, os, sys

d = sys.argv[1]
NAME = {"c1": "C1", "c2": "C2", "c3": "C3", "c4": "C4", "c5a": "C5a", "c5b": "C5b", "c5c": "C5c"}


def lines():
    for f in sorted(glob.glob(os.path.join(d, "bench_*.json"))):
        try:
            j = json.loads(open(f).read().strip().splitlines()[-1])
        except Exception:
            continue
        yield j
        if j.get("c5a"):
            yield j["c5a"] | {"verified": j["c5a"].get("verified"), "cpu_baseline": j["c5a"].get("cpu_baseline")}


for j in lines():
    cfg = j.get("config", {})
    w = cfg.get("workload")
    if w not in NAME:
        continue
    label = NAME[w] + (" (L2 flushed)" if w == "c2" and cfg.get("l2", "").startswith("flushed") else "")
    n = cfg["n"]
    per = j["detail"]["per_order_ms_mean"]
    routes = j["detail"]["routes"]
    hb = j.get("whole_step_hbm", {})
    rf = j.get("roofline") or {}
    ver = j.get("verified") or {}
    cpu = j.get("cpu_baseline") or {}
    par = f"{ver.get('checked', 0) - ver.get('failed', 0)}/{ver.get('checked', 0)} ok" if ver else ""
    orc = f"{n / cpu['value']:.0f}" if cpu.get("value") else ""
    dt = cfg.get("dtype", "") + (" pairs" if cfg.get("pairs") else "")
    for o, ms in per.items():
        print(f"| {label} | {o} | {n:,} | {dt} | {ms * 1e3:.1f} | {n / (ms * 1e3):,.0f} | {routes.get(o, '')} | | | | | {orc} | {par} |")
    print(f"| {label} | **step ({len(per)} orders)** | | | {j['ms_per_step'] * 1e3:.1f} | {j['value']:,.0f} | | "
          f"{hb.get('bytes_planned_per_step', 0) / 1e6:,.0f} MB | {hb.get('frac_of_peak', '')} | {hb.get('ideal_pass_frac', '')} | "
          f"{(rf.get('traffic') or 0) / 1e6:,.0f} MB ({rf.get('kernel', '')}, {rf.get('traffic_source', {}).get('source', '') if rf.get('traffic_source') else ''}) | | {par} |")
