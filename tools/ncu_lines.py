"""Per-CUDA-source-line stall samples / executed instructions for one kernel of an ncu report."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
by_inst = len(sys.argv) > 4 and sys.argv[4] == 'inst'
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
res = []; fname = None; hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr and len(r) == len(hdr) and r[0] not in ("",):
        try:
            st = float(r[4].replace(",", "") or 0); ie = float(r[7].replace(",", "") or 0)
        except ValueError:
            continue
        res.append((st, ie, fname, r[0], r[1].strip()))
tot_s = sum(x[0] for x in res) or 1; tot_i = sum(x[1] for x in res) or 1
print(f"samples={tot_s:.0f} warp-inst={tot_i:.0f}")
for st, ie, f, ln, src in sorted(res, reverse=True, key=(lambda x: x[1]) if by_inst else None)[:top]:
    print(f"{st/tot_s*100:5.1f}% stall {ie/tot_i*100:5.1f}% inst  {f}:{ln}  {src[:90]}")
