"""SASS census of a kernel's hot loops (instructions per sample).

    python tools/sass_loop.py <cubin-or-so> <mangled-name-regex> [samples_per_iter]

Finds every backward branch (a loop) in the kernel, prints the loop body size
and its per-opcode counts; with samples_per_iter, instructions per sample.
"""
import re
import subprocess
import sys
from collections import Counter


def kernel_sass(binary, pat):
    out = subprocess.run(["cuobjdump", "-sass", binary], capture_output=True, text=True).stdout
    lines, keep = [], False
    for ln in out.splitlines():
        if "Function : " in ln:
            keep = re.search(pat, ln) is not None
            if keep:
                name = ln.split("Function : ")[1].strip()
            continue
        if keep:
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
            if m:
                lines.append((int(m.group(1), 16), m.group(2).strip()))
        if keep and "EXIT" in ln and False:
            pass
    return lines


def loops(ins):
    res = []
    for addr, txt in ins:
        m = re.search(r"BRA\S*\s+(?:!?U?P\d,\s*)?(0x[0-9a-f]+)", txt)
        if m:
            tgt = int(m.group(1), 16)
            if tgt < addr:
                body = [t for a, t in ins if tgt <= a <= addr]
                res.append((tgt, addr, body))
    return res


def opcode(t):
    op = t.split()[0]
    if op.startswith("@"):
        op = t.split()[1]
    return op


if __name__ == "__main__":
    binary, pat = sys.argv[1], sys.argv[2]
    per = int(sys.argv[3]) if len(sys.argv) > 3 else None
    ins = kernel_sass(binary, pat)
    for tgt, end, body in sorted(loops(ins), key=lambda x: -len(x[2]))[:3]:
        c = Counter(opcode(t) for t in body)
        print(f"loop {tgt:#x}..{end:#x}: {len(body)} instructions" + (f" = {len(body)/per:.2f} per sample" if per else ""))
        for op, n in c.most_common():
            print(f"  {n:5d} {op}")
