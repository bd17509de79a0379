"""Top stalled SASS instructions of a kernel with preceding context and stall reasons (dev tool)."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 6
ctx = int(sys.argv[4]) if len(sys.argv) > 4 else 8
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr]
si = h.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[hdr + 1:] if len(r) > si and r[si].isdigit()]
tot = sum(int(r[si] or 0) for r in body)
seen = set()
for k in sorted(range(len(body)), key=lambda k: -int(body[k][si] or 0)):
    if body[k][1] in seen:
        continue
    seen.add(body[k][1])
    if len(seen) > top:
        break
    r = body[k]
    print(f"{int(r[si]) / tot * 100:5.1f}%  {r[1][:80]}")
    for j in range(max(0, k - ctx), k):
        print("        ", body[j][1][:80])
    det = [(h[i], r[i]) for i in range(len(h)) if h[i].startswith("stall_") and "Not Issued" not in h[i]
           and r[i] not in ("0", "", "0.0")]
    print("     ", sorted(det, key=lambda x: -float(x[1]))[:5])
