"""Print per-kernel warp-stall breakdown (pc-sampling counts) from an ncu report.

    python tools/ncu_stalls.py <report.ncu-rep>
"""
import csv
import io
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"


def main(path):
    out = subprocess.run([NCU, "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    for row in rows[2:]:
        d = dict(zip(h, row))
        pre = "smsp__pcsamp_warps_issue_stalled_"
        st = {}
        for k, v in d.items():
            if k.startswith(pre) and not k.endswith("_not_issued") and v not in ("", "n/a"):
                st[k[len(pre):]] = float(v.replace(",", ""))
        tot = sum(st.values()) or 1.0
        top = sorted(st.items(), key=lambda x: -x[1])[:10]
        print(d["Kernel Name"][:70], d.get("gpu__time_duration.sum"), "us")
        print("   " + ", ".join(f"{k}={100 * v / tot:.1f}%" for k, v in top))


if __name__ == "__main__":
    main(sys.argv[1])
