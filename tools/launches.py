"""Summarise an ncu --metrics gpu__time_duration.sum launch list (second half = measured solve)."""
import collections
import csv
import io
import re
import sys

txt = open(sys.argv[1]).read()
rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
rows = rows[int(len(rows) * frac):]
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows:
    nm = re.sub(r"\(.*", "", r["Kernel Name"]).replace("fbmp_gpu::", "").replace("<unnamed>::", "")
    nm = nm.replace("fast::", "")
    tot[nm] += float(r["Metric Value"]) / 1e3
    cnt[nm] += 1
T = sum(tot.values())
print(f"total {T:.1f} us over {len(rows)} launches")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:25]:
    print(f"{k[:56]:56s} {v:10.1f} us {cnt[k]:5d} x  avg {v / cnt[k]:8.2f} us  {100 * v / T:5.1f}%")
