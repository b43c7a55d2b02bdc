# Round-2 stage g (final): TMA-fed GEMM + dataflow Jacobi: full GPU suite, bench lines, ncu launch list,
# full captures of the top kernels, DRAM traffic of the dgemm launches.
mkdir -p gpurun_out
timeout 300 python tools/ubench/gemm_feed.py 5 > gpurun_out/gemm_feed_r2g.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pt_r2g.log 2>&1; echo "rc=$?" >> gpurun_out/pt_r2g.log
python bench.py --steps 5 --warmup 3 --breakdown > gpurun_out/bench_c4_r2g.json 2> gpurun_out/bench_c4_r2g.err
for c in c3 c5 c6; do timeout 400 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --breakdown > gpurun_out/bench_${c}_r2g.json 2> gpurun_out/bench_${c}_r2g.err; done
C="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_c4_r2g.csv $C > gpurun_out/ncu_list.log 2>&1
python3 - <<'PY'
import csv, json
rows = [r for r in csv.reader(open("gpurun_out/launches_c4_r2g.csv")) if len(r) > 10]
hdr = rows[0]; rows = rows[1:]
ki, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("ID")
d = [(int(r[ii]), r[ki], float(r[vi].replace(",", ""))) for r in rows if r[vi].replace(",", "").replace(".", "").isdigit()]
def pick(sub, nth=0):
    xs = [x for x in d if sub in x[1]]
    order = sorted(range(len(xs)), key=lambda i: -xs[i][2])
    return order[nth] if len(order) > nth else 0
# the longest dgemm_tma_kernel launch is form_W; the second longest kind (gram_W) follows it
tma = [x for x in d if "dgemm_tma_kernel" in x[1]]
fw = pick("dgemm_tma_kernel")
gw = next((i for i in sorted(range(len(tma)), key=lambda i: -tma[i][2]) if "<1, 1>" in tma[i][1]), 0)
json.dump({"tma_skip": fw, "gram_skip": gw, "jacobi_skip": pick("jacobi_flow_k")}, open("gpurun_out/ncu_pick.json", "w"))
PY
DS=$(python3 -c "import json; print(json.load(open('gpurun_out/ncu_pick.json'))['tma_skip'])")
JS=$(python3 -c "import json; print(json.load(open('gpurun_out/ncu_pick.json'))['jacobi_skip'])")
GS=$(python3 -c "import json; print(json.load(open('gpurun_out/ncu_pick.json'))['gram_skip'])")
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dgemm_tma_kernel -s $DS -c 1 -o gpurun_out/prof_r2g_formW $C > gpurun_out/ncu_formW.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jacobi_flow_k -s $JS -c 1 -o gpurun_out/prof_r2g_jacobi $C > gpurun_out/ncu_jacobi.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dgemm_tma_kernel -s $GS -c 1 -o gpurun_out/prof_r2g_gramW $C > gpurun_out/ncu_gramW.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:dgemm --csv --log-file gpurun_out/dgemm_traffic_r2g.csv $C > gpurun_out/ncu_traffic.log 2>&1
tail -3 gpurun_out/pt_r2g.log
