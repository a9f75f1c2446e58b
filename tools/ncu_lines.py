"""Dynamic instruction counts per CUDA source line: ncu SASS page (executed counts per
instruction) joined with nvdisasm -g line markers of the same kernel.

    python tools/ncu_lines.py <report.ncu-rep> <cubin> <mangled-kernel-substring> [units] [top]
"""
import collections
import csv
import io
import re
import subprocess
import sys


def main():
    rep, cubin, pat = sys.argv[1:4]
    units = float(sys.argv[4]) if len(sys.argv) > 4 else None
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
    dis = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout.splitlines()
    line_of = {}
    keep, cur = False, None
    for ln in dis:
        if re.match(r"\s*\.text\.", ln):
            keep = pat in ln
            continue
        if not keep:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            line_of[int(m.group(1), 16)] = cur
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    iA, iS, iE = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
    base = int(rows[2][iA], 16)
    per_line = collections.Counter()
    per_line_fp64 = collections.Counter()
    ops = collections.defaultdict(collections.Counter)
    tot = 0.0
    for r in rows[2:]:
        try:
            e = float(r[iE].replace(",", ""))
            off = int(r[iA], 16) - base
        except (ValueError, IndexError):
            continue
        src = re.sub(r"^@!?U?P\w+\s+", "", r[iS].strip())
        op = src.split()[0] if src else "?"
        key = line_of.get(off)
        per_line[key] += e
        if op.startswith(("DFMA", "DMUL", "DADD")):
            per_line_fp64[key] += e
        ops[key][op.split(".")[0]] += e
        tot += e
    scale = 32.0 / units if units else 1.0
    print(f"total warp instructions {tot:.4g}" + (f" = {tot * scale:.2f} per unit" if units else ""))
    for key, e in per_line.most_common(top):
        o = " ".join(f"{k}:{v * scale:.2f}" for k, v in ops[key].most_common(6))
        print(f"{str(key):28s} {e * scale:8.2f}  fp64 {per_line_fp64[key] * scale:6.2f}   {o}")


if __name__ == "__main__":
    main()
