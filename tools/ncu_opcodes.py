"""Executed warp instructions per SASS opcode of one kernel in an ncu report (source page).

    python tools/ncu_opcodes.py <report.ncu-rep> <kernel-regex> [top]
"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter

NCU = "/usr/local/cuda/bin/ncu"


def main(path, kregex, top=30):
    out = subprocess.run([NCU, "-i", path, "--page", "source", "--csv", "--print-source", "sass",
                          "--kernel-name", f"regex:{kregex}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    si = h.index("Source")
    ei = h.index("Instructions Executed")
    wi = h.index("Warp Stall Sampling (All Samples)")
    ex, st = Counter(), Counter()
    for r in rows[2:]:
        src = re.sub(r"^@!?U?P\w+\s+", "", r[si].strip())
        op = src.split(" ")[0] if src else "?"
        ex[op] += float(r[ei] or 0)
        st[op] += float(r[wi] or 0)
    tot, tots = sum(ex.values()) or 1, sum(st.values()) or 1
    print(f"warp instructions {tot:.0f}, stall samples {tots:.0f}")
    for op, n in ex.most_common(int(top)):
        print(f"{op:28s} {n:14.0f} {100 * n / tot:6.2f}%   stalls {100 * st[op] / tots:6.2f}%")


if __name__ == "__main__":
    main(*sys.argv[1:])
