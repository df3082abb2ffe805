"""Hottest SASS lines (warp-stall samples) of one kernel in an ncu report.

    python tools/ncu_hot.py <report.ncu-rep> <kernel-regex> [top]
"""
import csv
import io
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"


def main(path, kregex, top=40):
    out = subprocess.run([NCU, "-i", path, "--page", "source", "--csv", "--print-source", "sass",
                          "--kernel-name", f"regex:{kregex}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    data = rows[2:]
    si = h.index("Warp Stall Sampling (All Samples)")
    ei = h.index("Instructions Executed")
    tot = sum(float(r[si] or 0) for r in data) or 1
    toti = sum(float(r[ei] or 0) for r in data) or 1
    print(f"samples {tot:.0f}, warp instructions {toti:.0f}")
    idx = sorted(range(len(data)), key=lambda i: -float(data[i][si] or 0))[:top]
    for i in sorted(idx):
        r = data[i]
        print(f"{i:5d} {r[0]:>6} {100 * float(r[si] or 0) / tot:5.1f}% ex={float(r[ei] or 0) / toti * 100:5.2f}%  {r[1][:80]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
