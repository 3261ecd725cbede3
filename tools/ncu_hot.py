"""Summarise an ncu report's SASS source page: hottest instructions by stall samples, opcode mix.

usage: ncu_hot.py REPORT KERNEL_REGEX [TOP]   (of several matching launches, the one with most instructions)"""
import csv, subprocess, sys, collections
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif r and r[0] == "Address":
        cur["h"] = r
    elif cur is not None and "h" in cur and len(r) == len(cur["h"]):
        cur["rows"].append(r)
def num(x):
    try: return float((x or "0").replace(",", ""))
    except ValueError: return 0.0
best = max(blocks, key=lambda b: sum(num(r[b["h"].index("Instructions Executed")]) for r in b["rows"]))
h, data = best["h"], best["rows"]
ix = {k: i for i, k in enumerate(h)}
ie, ist = ix["Instructions Executed"], ix["Warp Stall Sampling (All Samples)"]
tot_i = sum(num(r[ie]) for r in data); tot_s = sum(num(r[ist]) for r in data) or 1
print(best["name"][:100])
print(f"total warp-instr {tot_i:.0f}  stall samples {tot_s:.0f}")
ops = collections.Counter()
for r in data:
    t = r[1].split()
    if not t: continue
    op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
    ops[op.split(".")[0]] += num(r[ie])
print("by opcode:", ", ".join(f"{k}={v/tot_i*100:.1f}%" for k, v in ops.most_common(16)))
stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot_by = {c: sum(num(r[ix[c]]) for r in data) for c in stall_cols}
print("stalls:", ", ".join(f"{c[6:]}={v/tot_s*100:.1f}%" for c, v in sorted(tot_by.items(), key=lambda kv: -kv[1])[:8]))
print("-- top by stall samples")
for r in sorted(data, key=lambda r: -num(r[ist]))[:top]:
    print(f"{r[0][-5:]} stall={num(r[ist])/tot_s*100:5.1f}% inst={num(r[ie])/tot_i*100:4.1f}%  {r[1][:80]}")
