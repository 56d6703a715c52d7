"""Per-source-line warp-stall samples from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if r and r[0] == "Line No")
wi = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
lines = [r for r in rows if r and r[0].isdigit() and r[2] == "-" and len(r) > wi]
tot = sum(float(r[wi] or 0) for r in lines)
tin = sum(float(r[ie] or 0) for r in lines)
print(f"samples {tot:.0f}  warp-instructions {tin:.3g}")
for r in sorted(lines, key=lambda r: -float(r[wi] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{100 * float(r[wi] or 0) / tot:5.1f}% inst {100 * float(r[ie] or 0) / tin:5.1f}%  L{r[0]:>4}  {r[1].strip()[:100]}")
