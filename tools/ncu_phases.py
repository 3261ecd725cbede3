"""Group an ncu source page (cuda,sass) by source file / line range: executed
warp-instructions and stall samples per region.  usage: ncu_phases.py rep kernel file:name:start-end ..."""
import collections, csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
ranges = []
for spec in sys.argv[3:]:
    f, name, lr = spec.split(":")
    a, b = lr.split("-")
    ranges.append((f, name, int(a), int(b)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg, aggs = collections.Counter(), collections.Counter()
fname = hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr and len(r) == len(hdr):
        try:
            st = float(r[4].replace(",", "") or 0); ie = float(r[7].replace(",", "") or 0); ln = int(r[0])
        except ValueError:
            continue
        key = fname
        for f, name, a, b in ranges:
            if f == fname and a <= ln <= b: key = name
        agg[key] += ie; aggs[key] += st
tot = sum(agg.values()) or 1; tots = sum(aggs.values()) or 1
print(f"warp-inst={tot:.0f} samples={tots:.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    print("%-24s inst %5.1f%%  stall %5.1f%%" % (k, 100 * v / tot, 100 * aggs[k] / tots))
