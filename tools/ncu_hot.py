"""Top stalled SASS lines of an ncu report (source page), optionally excluding grid-sync spins.

usage: python tools/ncu_hot.py report.ncu-rep [N] [--no-spin]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 40
    nospin = "--no-spin" in sys.argv
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    data = rows[2:]
    si = h.index("Warp Stall Sampling (All Samples)")
    src = h.index("Source")
    ex = h.index("Instructions Executed")
    spin = lambda r: nospin and ("CCTL" in r[src] or "STRONG.GPU" in r[src] or
                                 r[src].strip().startswith("BRA") or "NANOSLEEP" in r[src])
    data = [r for r in data if not spin(r)]
    tot = sum(float(r[si] or 0) for r in data)
    print("samples", tot)
    for r in sorted(data, key=lambda r: -float(r[si] or 0))[:n]:
        print(f"{float(r[si]) / tot * 100:5.1f}% ex={r[ex]:>9} {r[src][:95]}")


if __name__ == "__main__":
    main()
