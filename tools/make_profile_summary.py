"""Summarise ncu outputs into profiles/: the launch list (share of the step per
kernel, from --metrics gpu__time_duration.sum) and the --set full capture
(per-kernel time, DRAM traffic, occupancy, issue, top stall reasons)."""
import csv, collections, json, subprocess, sys

tag, launches, rep = sys.argv[1], sys.argv[2], sys.argv[3]
workload = sys.argv[4] if len(sys.argv) > 4 else None  # bench --workload the captures belong to
out = {"tag": tag, "workload": workload, "launch_list": {}, "full": {}}
rows = list(csv.reader(open(launches)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]; ix = {k: i for i, k in enumerate(h)}
per = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
for r in rows[hi + 1:]:
    name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "").split("<")[0]
    m, v = r[ix["Metric Name"]], float(r[ix["Metric Value"]].replace(",", ""))
    per[name][m] += v
    if m == "gpu__time_duration.sum": cnt[name] += 1
tot = sum(d["gpu__time_duration.sum"] for k, d in per.items() if k.startswith("sr::"))
for k, d in sorted(per.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
    out["launch_list"][k] = {"launches": cnt[k], "total_us": round(d["gpu__time_duration.sum"] / 1e3, 2),
                             "share_of_sr_kernels": round(d["gpu__time_duration.sum"] / tot, 4) if k.startswith("sr::") else None,
                             "dram_read_MB": round(d.get("dram__bytes_read.sum", 0) / 1e6, 3),
                             "dram_write_MB": round(d.get("dram__bytes_write.sum", 0) / 1e6, 3)}
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines())); H = rr[0]; U = rr[1]; IX = {k: i for i, k in enumerate(H)}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
         "ns": 1e-3, "us": 1, "ms": 1e3}
def f(r, k):
    try:
        v = float(r[IX[k]].replace(",", ""))
        return v * SCALE.get(U[IX[k]], 1)
    except Exception: return None
for r in rr[2:]:
    name = r[IX["Kernel Name"]].split("(")[0].replace("void ", "")
    st = []
    for k, i in IX.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            v = f(r, k)
            if v: st.append((v, k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
    ts = sum(v for v, _ in st) or 1
    d = {"duration_us": f(r, "gpu__time_duration.sum"), "grid": r[IX["launch__grid_size"]],
         "block": r[IX["launch__block_size"]], "regs": f(r, "launch__registers_per_thread"),
         "dram_bytes_read": f(r, "dram__bytes_read.sum"), "dram_bytes_write": f(r, "dram__bytes_write.sum"),
         "dram_throughput_pct": f(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
         "sm_throughput_pct": f(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
         "warps_active_pct": f(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
         "issue_active_pct": f(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
         "inst_executed": f(r, "smsp__inst_executed.sum"),
         "top_stalls": {k: round(v / ts, 3) for v, k in sorted(st, reverse=True)[:5]}}
    out["full"].setdefault(name, d)
json.dump(out, open(f"profiles/{tag}_ncu_summary.json", "w"), indent=1)
with open(f"profiles/{tag}_ncu_summary.md", "w") as fo:
    fo.write(f"# ncu summary {tag}\n\n## Launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n\n")
    fo.write("| kernel | launches | total us | share of sr kernels | DRAM read MB | DRAM write MB |\n|---|---|---|---|---|---|\n")
    for k, d in out["launch_list"].items():
        fo.write(f"| {k} | {d['launches']} | {d['total_us']} | {d['share_of_sr_kernels']} | {d['dram_read_MB']} | {d['dram_write_MB']} |\n")
    fo.write("\n## --set full captures\n\n| kernel | us | grid x block | regs | DRAM r/w MB | DRAM % | SM % | warps active % | issue active % | top stalls |\n|---|---|---|---|---|---|---|---|---|---|\n")
    for k, d in out["full"].items():
        fo.write(f"| {k} | {d['duration_us']} | {d['grid']} x {d['block']} | {d['regs']} | "
                 f"{(d['dram_bytes_read'] or 0)/1e6:.2f}/{(d['dram_bytes_write'] or 0)/1e6:.2f} | {d['dram_throughput_pct']} | "
                 f"{d['sm_throughput_pct']} | {d['warps_active_pct']} | {d['issue_active_pct']} | "
                 + ", ".join(f"{a}={b}" for a, b in d["top_stalls"].items()) + " |\n")
print(open(f"profiles/{tag}_ncu_summary.md").read())
