"""Brief of one kernel in an ncu report: time, issue, pipes, stalls, per-op counts.

    python tools/ncu_brief.py <report.ncu-rep> [units_per_launch]
"""
import collections
import csv
import io
import re
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[2]


def sass(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    return hdr, rows[2:]


def main():
    rep = sys.argv[1]
    units = float(sys.argv[2]) if len(sys.argv) > 2 else None
    hdr, vals = raw(rep)
    get = lambda k: vals[hdr.index(k)] if k in hdr else "n/a"  # noqa: E731
    for k in ("gpu__time_duration.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
              "smsp__warps_eligible.avg.per_cycle_active", "smsp__inst_executed.sum",
              "dram__bytes_read.sum", "dram__bytes_write.sum"):
        print(f"{k:70s} {get(k)}")
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                st.append((float(vals[i].replace(",", "")), h[33:]))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    print("stalls:", ", ".join(f"{h} {100 * v / tot:.1f}%" for v, h in sorted(st, reverse=True)[:8]))
    sh, rows = sass(rep)
    iS, iE = sh.index("Source"), sh.index("Instructions Executed")
    ops = collections.Counter()
    tot_i = 0.0
    for r in rows:
        try:
            e = float(r[iE].replace(",", ""))
        except (ValueError, IndexError):
            continue
        src = r[iS].strip()
        op = re.sub(r"^@!?U?P\w+\s+", "", src).split()[0] if src else "?"
        ops[op] += e
        tot_i += e
    scale = (32.0 / units) if units else 1.0
    print(f"warp instructions executed {tot_i:.4g}" + (f" = {tot_i * scale:.2f} thread-instr per unit" if units else ""))
    for op, c in ops.most_common(30):
        print(f"  {op:24s} {c * scale:8.2f}")


if __name__ == "__main__":
    main()
