"""Top SASS instructions by warp-stall samples from an ncu report (source page):
    python scripts/ncu_hot.py report.ncu-rep [N]
"""
import csv
import subprocess
import sys


def main():
    rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    data = rows[2:]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(int(r[si]) for r in data if r[si].isdigit())
    print(f"total samples {tot}")
    for idx, r in sorted(enumerate(data), key=lambda x: -int(x[1][si]) if x[1][si].isdigit() else 0)[:top]:
        s = int(r[si])
        reasons = sorted(((int(r[i]), hdr[i][6:]) for i in stall_cols if r[i].isdigit() and int(r[i]) > 0), reverse=True)[:3]
        print(f"{idx:5d} {100 * s / tot:5.1f}%  {r[1].strip()[:60]:60s} {reasons}")


if __name__ == "__main__":
    main()
