"""One-paragraph-per-kernel summary of `ncu --set full` reports (for profiles/):
duration, DRAM bytes and bandwidth, FP64 pipe use (thread DFMA/DADD/DMUL per cycle against the
64/clk/SM peak), issue / warp occupancy, registers, local-memory frame and the top stall reasons.

    python tools/ncu_brief.py REPORT.ncu-rep [REPORT2 ...] > profiles/rNN_ncu_xxx.txt
"""
import csv
import io
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TSCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}


def summarize(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}

    def f(r, k, default=0.0):
        i = col.get(k)
        if i is None or r[i] in ("", "n/a"):
            return default
        return float(r[i].replace(",", ""))

    out = []
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        t_us = f(r, "gpu__time_duration.sum") * TSCALE.get(units[col["gpu__time_duration.sum"]], 1.0)
        rd = f(r, "dram__bytes_read.sum") * SCALE.get(units[col["dram__bytes_read.sum"]], 1)
        wr = f(r, "dram__bytes_write.sum") * SCALE.get(units[col["dram__bytes_write.sum"]], 1)
        cyc = f(r, "sm__cycles_elapsed.avg")
        fp64 = sum(f(r, f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed")
                   for op in ("dfma", "dadd", "dmul"))
        fp64_peak = 64.0 * 148
        stalls = {h[len("smsp__pcsamp_warps_issue_stalled_"):]: float(r[i] or 0)
                  for h, i in col.items() if h.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not h.endswith("not_issued") and r[i] not in ("", "n/a")}
        tot = sum(stalls.values()) or 1.0
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:4]
        out.append(
            f"{name[:110]}\n"
            f"  duration {t_us:.1f} us ({cyc:.0f} cycles) | DRAM read {rd / 1e6:.1f} MB write {wr / 1e6:.1f} MB -> "
            f"{(rd + wr) / max(t_us, 1e-9) / 1e3:.0f} GB/s\n"
            f"  FP64 ops/cycle {fp64:.0f} of {fp64_peak:.0f} ({100 * fp64 / fp64_peak:.0f} %) | issue active "
            f"{f(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.0f} % | warps active "
            f"{f(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.0f} % | warp instr "
            f"{f(r, 'smsp__inst_executed.sum') / 1e6:.1f} M | regs {int(f(r, 'launch__registers_per_thread'))} | "
            f"grid {int(f(r, 'launch__grid_size'))} x {int(f(r, 'launch__block_size'))}\n"
            f"  stalls: " + ", ".join(f"{a} {100 * b / tot:.0f}%" for a, b in top))
    return out


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print(f"# {rep}")
        print("\n".join(summarize(rep)))
        print()
