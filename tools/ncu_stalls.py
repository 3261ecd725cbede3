"""Per-kernel stall breakdown + key metrics from an ncu report (raw page)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]; data = rows[2:]
idx = {k: i for i, k in enumerate(h)}
def f(r, k):
    try: return float(r[idx[k]].replace(",", ""))
    except Exception: return None
for r in data:
    name = r[idx["Kernel Name"]][:60]
    print(f"--- {name}  {f(r,'gpu__time_duration.sum')} us  grid={r[idx['launch__grid_size']]} regs={r[idx['launch__registers_per_thread']]} "
          f"inst={f(r,'smsp__inst_executed.sum'):.0f} dram_r={f(r,'dram__bytes_read.sum')} dram_w={f(r,'dram__bytes_write.sum')}")
    st = []
    for k, i in idx.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            v = f(r, k)
            if v: st.append((v, k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
    tot = sum(v for v, _ in st) or 1
    print("   stalls:", ", ".join(f"{k}={v/tot*100:.0f}%" for v, k in sorted(st, reverse=True)[:7]))
