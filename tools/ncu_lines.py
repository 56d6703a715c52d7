"""Per-CUDA-line hot spots of one kernel in an ncu report (warp-stall samples, shared wavefronts).
usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [TOP]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kern,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, out = None, []
for r in rows:
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 3 and r[0] != "" and r[2] == "-":
        out.append(r)
col = {}
for i, h in enumerate(hdr):
    col.setdefault(h, i)


def f(r, k):
    try:
        return float(r[col[k]])
    except (KeyError, ValueError):
        return 0.0


S = "Warp Stall Sampling (All Samples)"
tot = sum(f(r, S) for r in out)
print(f"total samples {tot:.0f}")
for r in sorted(out, key=lambda r: -f(r, S))[:top]:
    print(f"{r[0]:>5} {f(r, S):6.0f} inst {f(r, 'Instructions Executed'):9.0f} wf {f(r, 'L1 Wavefronts Shared'):8.0f}/"
          f"{f(r, 'L1 Wavefronts Shared Ideal'):8.0f} lsb {f(r, 'stall_long_sb'):4.0f} ssb {f(r, 'stall_short_sb'):4.0f} "
          f"bar {f(r, 'stall_barrier'):4.0f} wait {f(r, 'stall_wait'):4.0f} | {r[1].strip()[:80]}")
