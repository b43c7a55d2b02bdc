"""Convert an ncu CSV (gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum over
the dgemm_kernel launches of `bench.py --steps 1 --warmup 0`) into profiles/r02/dgemm_traffic.json:
the DRAM bytes per heavy launch of the dominant kernel (bench.py roofline.traffic).
usage: python tools/dgemm_traffic.py gpurun_out/dgemm_traffic_r02.csv"""
import csv
import json
import os
import sys

rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
hdr, rows = rows[0], rows[1:]
ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
per = {}
for r in rows:
    d = per.setdefault(int(r[ii]), {})
    d[r[mi]] = float(r[vi].replace(",", ""))
launches = [per[k] for k in sorted(per)]
# ops captured = number of form_W launches (the only dgemm launch longer than 15 ms at c4)
steps = max(1, sum(1 for d in launches if d.get("gpu__time_duration.sum", 0) > 15e6))
# the bench's heavy set is the launches with >= 1e8 algorithmic flops or bytes (46 per c4 step):
# here the 46 longest per step
TOP = int(sys.argv[2]) if len(sys.argv) > 2 else 46
heavy = sorted(launches, key=lambda d: -d.get("gpu__time_duration.sum", 0))[: TOP * steps]
byts = [d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in heavy]
out = {
    "source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
              "-k regex:dgemm (dgemm_tma_kernel + dgemm_kernel) over `bench.py --steps 1 --warmup 0 "
              f"--no-cpu-baseline` on c4 ({steps} apply+round ops captured)",
    "csv": os.path.basename(sys.argv[1]),
    "launches_per_step": len(launches) / steps,
    "heavy_launches_per_step": len(heavy) / steps,
    "heavy_rule": f"the {TOP} longest dgemm launches per step (bench.py's heavy set)",
    "dram_bytes_per_launch": sum(byts) / max(len(byts), 1),
    "total_heavy_dram_bytes_per_step": sum(byts) / steps,
    "avg_heavy_launch_ms": sum(d["gpu__time_duration.sum"] for d in heavy) / max(len(heavy), 1) / 1e6,
}
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
json.dump(out, open(os.path.join(root, "profiles", "r02", "dgemm_traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
