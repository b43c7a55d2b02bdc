"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel: count, total, share.

usage: python tools/launch_summary.py gpurun_out/launches.csv [out.md]
"""
import collections
import csv
import re
import sys


def kernel_name(s):
    s = s.replace("<unnamed>::", "").replace("void ", "")
    s = s.split("(")[0]
    return re.sub(r"<.*>", "", s).strip()


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ui = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value",
                                            "Metric Unit"))
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[hdr + 1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = kernel_name(r[ki])
        tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        cnt[name] += 1
    total = sum(tot.values())
    lines = [f"launches: {sum(cnt.values())}, summed device time {total:.2f} ms "
             "(ncu, cold-cache, serialised)", "",
             "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in tot.most_common():
        lines.append(f"| {k} | {cnt[k]} | {v:.3f} | {100 * v / total:.1f} % |")
    out = "\n".join(lines)
    print(out)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(out + "\n")


if __name__ == "__main__":
    main()
