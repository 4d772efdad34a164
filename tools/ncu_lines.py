"""Per-source-line warp-stall samples of an ncu report (cuda+sass source view).

usage: python tools/ncu_lines.py REP [N]  -> the N source lines with the most stall samples
"""
import csv
import io
import subprocess
import sys


def main(rep, n=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    lines = []
    for r in rows:
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0]:
            lines.append(r)
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    iI = hdr.index("Instructions Executed")
    tot = sum(float(r[iS] or 0) for r in lines) or 1.0
    print(f"samples {tot:.0f}")
    for r in sorted(lines, key=lambda r: -float(r[iS] or 0))[:n]:
        print(f"{100 * float(r[iS] or 0) / tot:5.1f}%  L{r[0]:>4}  inst {float(r[iI] or 0):12.0f}  {r[1].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
