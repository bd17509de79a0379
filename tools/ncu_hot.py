"""Summarise an ncu source page (SASS) by stall samples: top instructions."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr]
si = h.index("Warp Stall Sampling (All Samples)")
ii = h.index("Instructions Executed")
body = [r for r in rows[hdr + 1:] if len(r) > si and r[si].isdigit()]
tot = sum(int(r[si]) for r in body)
print(f"total samples {tot}, instructions {len(body)}")
stall_cols = [i for i, n in enumerate(h) if n.startswith("stall_") or "Stall" in n and i not in (si,)]
for r in sorted(body, key=lambda r: -int(r[si]))[:top]:
    print(f"{int(r[si]) / tot * 100:5.1f}%  exec={r[ii]:>10}  {r[1].strip()[:90]}")
