"""Summarise an ncu report's SASS source page: hottest instructions by executed count and stall samples."""
import csv, subprocess, sys, collections
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]; data = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0] != "Address"]
ix = {k: i for i, k in enumerate(h)}
ie, ist = ix["Instructions Executed"], ix["Warp Stall Sampling (All Samples)"]
tot_i = sum(float((r[ie] or "0").replace(",","")) for r in data); tot_s = sum(float((r[ist] or "0").replace(",","")) for r in data)
print(f"total warp-instr {tot_i:.0f}  stall samples {tot_s:.0f}")
ops = collections.Counter()
for r in data:
    op = r[1].split()[0] if r[1].split() else "?"
    if op.startswith("@"): op = r[1].split()[1]
    ops[op.split(".")[0]] += float((r[ie] or "0").replace(",",""))
print("by opcode:", ", ".join(f"{k}={v/tot_i*100:.1f}%" for k, v in ops.most_common(14)))
print("-- top by stall samples")
for r in sorted(data, key=lambda r: -float((r[ist] or "0").replace(",","")))[:top]:
    print(f"{r[0][-5:]} stall={float((r[ist] or "0").replace(",",""))/tot_s*100:5.1f}% inst={float((r[ie] or "0").replace(",",""))/tot_i*100:4.1f}%  {r[1][:80]}")
