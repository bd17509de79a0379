"""Per-CUDA-line stall samples / executed instructions from an ncu report."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname = "?"
res = []
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or r[2] != "-":
        continue
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ii = hdr.index("Instructions Executed")
    s = int(r[si]) if r[si].isdigit() else 0
    n = int(r[ii]) if r[ii].isdigit() else 0
    res.append((s, n, fname, r[0], r[1].strip()[:90]))
tot = sum(x[0] for x in res) or 1
toti = sum(x[1] for x in res) or 1
print(f"samples {tot}  warp-instructions {toti:.3e}")
for s, n, f, ln, src in sorted(res, key=lambda x: -x[0])[:top]:
    print(f"{100*s/tot:5.1f}% stall {100*n/toti:5.1f}% instr {n:>11} {f}:{ln:<5} {src}")
