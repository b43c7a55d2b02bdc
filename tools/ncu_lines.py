"""Aggregate ncu warp-stall samples by CUDA source line (cuda,sass view).

usage: python tools/ncu_lines.py report.ncu-rep [N]
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    agg = collections.Counter()
    text = {}
    fname = ""
    h = None
    for row in csv.reader(io.StringIO(out)):
        if len(row) == 2 and row[0] == "File Path":
            fname = row[1].split("/")[-1]
            continue
        if row and row[0] == "Line No":
            h = row
            si = h.index("Warp Stall Sampling (All Samples)")
            continue
        if h is None or len(row) <= si or not row[0].isdigit():
            continue
        key = (fname, int(row[0]))
        text[key] = row[1]
        try:
            agg[key] += float(row[si] or 0)
        except ValueError:
            pass
    tot = sum(agg.values()) or 1.0
    for key, v in agg.most_common(n):
        print(f"{100 * v / tot:5.1f}% {key[0]}:{key[1]}: {text[key].strip()[:100]}")


if __name__ == "__main__":
    main()
