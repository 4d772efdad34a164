"""Top stall sites of an ncu report (SASS view with source line correlation).

usage: python tools/ncu_stalls.py REP [N]   -> prints the N hottest SASS instructions
"""
import csv
import io
import subprocess
import sys


def main(rep, n=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    data = []
    for r in rows:
        if "Address" in r and "Source" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(r)
    if not hdr:
        print("no source page")
        return
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    iSrc, iA = hdr.index("Source"), hdr.index("Address")
    tot = sum(float(r[iS] or 0) for r in data) or 1.0
    print(f"samples {tot:.0f}")
    for r in sorted(data, key=lambda r: -float(r[iS] or 0))[:n]:
        print(f"{100 * float(r[iS] or 0) / tot:5.1f}%  {r[iA]}  {r[iSrc][:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
