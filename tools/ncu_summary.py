"""Summarise an `ncu --set full` report of the CG kernels into profiles/ (per-launch DRAM
traffic, duration, achieved bandwidth, occupancy, stall mix) and profiles/ncu_traffic.json
(the per-launch DRAM bytes bench.py reports as roofline.traffic)."""
import csv
import io
import json
import subprocess
import sys

rep, out_txt = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
col = {h: i for i, h in enumerate(hdr)}


def cls(name):
    if "k_q" in name:
        return "K_Q"
    if "k_dterm" in name:
        return "K_D"
    if "k_llp" in name or "k_apply" in name:
        return "K_L"
    if "k_update" in name or "k_du" in name:  # K_DU runs in the K_U slot of the fused path
        return "K_U"
    return name.split("(")[0][-40:]


lines, traffic = [], {}
for r in rows[2:]:
    k = cls(r[col["Kernel Name"]])
    t_us = float(r[col["gpu__time_duration.sum"]])
    rd = float(r[col["dram__bytes_read.sum"]])
    wr = float(r[col["dram__bytes_write.sum"]])
    ur = units[col["dram__bytes_read.sum"]]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[ur]
    rd, wr = rd * scale, wr * scale
    stalls = {h[len("smsp__pcsamp_warps_issue_stalled_"):]: float(r[i] or 0)
              for h, i in col.items() if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")
              and r[i] not in ("", "n/a")}
    tot = sum(stalls.values()) or 1.0
    top = sorted(stalls.items(), key=lambda kv: -kv[1])[:4]
    traffic[k] = rd + wr
    lines.append(f"{k}: {r[col['Kernel Name']][:70]}\n"
                 f"  duration {t_us:.1f} us | DRAM read {rd / 1e6:.1f} MB write {wr / 1e6:.1f} MB -> "
                 f"{(rd + wr) / t_us / 1e3:.0f} GB/s | warps active "
                 f"{r[col['sm__warps_active.avg.pct_of_peak_sustained_active']]}% | issue active "
                 f"{r[col['smsp__issue_active.avg.pct_of_peak_sustained_active']]}% | regs "
                 f"{r[col['launch__registers_per_thread']]}\n"
                 f"  stalls: " + ", ".join(f"{a} {100 * b / tot:.0f}%" for a, b in top))
open(out_txt, "w").write("\n".join(lines) + "\n")
traffic["config"] = sys.argv[4] if len(sys.argv) > 4 else "C2"  # the configuration the capture ran
json.dump(traffic, open(sys.argv[3] if len(sys.argv) > 3 else "profiles/ncu_traffic.json", "w"), indent=1)
print("\n".join(lines))
