# Round-2 stage b: full GPU suite, bench lines, ncu launch list + full captures of the top kernels.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pt_r2b.log 2>&1; echo "rc=$?" >> gpurun_out/pt_r2b.log
python bench.py --steps 5 --warmup 3 --breakdown > gpurun_out/bench_c4_r2b.json 2> gpurun_out/bench_c4_r2b.err
for c in c3 c5 c6 c8; do timeout 400 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --breakdown > gpurun_out/bench_${c}_r2b.json 2> gpurun_out/bench_${c}_r2b.err; done
timeout 400 python bench.py --config c5 --prec --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c5p_r2b.json 2> gpurun_out/bench_c5p_r2b.err
timeout 400 python bench.py --config c8 --prec --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c8p_r2b.json 2> gpurun_out/bench_c8p_r2b.err
timeout 400 python bench.py --config c7 --steps 3 --warmup 2 > gpurun_out/bench_c7_r2b.json 2> gpurun_out/bench_c7_r2b.err
C="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_c4_r02.csv $C > gpurun_out/ncu_list.log 2>&1
python3 - <<'PY'
import csv, json
rows = [r for r in csv.reader(open("gpurun_out/launches_c4_r02.csv")) if len(r) > 10]
hdr = rows[0]; rows = rows[1:]
ki, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("ID")
d = [(int(r[ii]), r[ki], float(r[vi].replace(",", ""))) for r in rows if r[vi].replace(",", "").replace(".", "").isdigit()]
dg = [x for x in d if x[1].startswith("dgemm_kernel")]
big = max(range(len(dg)), key=lambda i: dg[i][2])
jac = [x for x in d if x[1].startswith("jacobi_persistent_k")]
jb = max(range(len(jac)), key=lambda i: jac[i][2])
json.dump({"dgemm_skip": big, "dgemm_ns": dg[big][2], "jacobi_skip": jb}, open("gpurun_out/ncu_pick.json", "w"))
PY
DS=$(python3 -c "import json; print(json.load(open('gpurun_out/ncu_pick.json'))['dgemm_skip'])")
JS=$(python3 -c "import json; print(json.load(open('gpurun_out/ncu_pick.json'))['jacobi_skip'])")
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dgemm_kernel -s $DS -c 1 -o gpurun_out/prof_r02_formW $C > gpurun_out/ncu_formW.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jacobi_persistent_k -s $JS -c 1 -o gpurun_out/prof_r02_jacobi $C > gpurun_out/ncu_jacobi.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_merged -c 1 -o gpurun_out/prof_r02_spmm $C > gpurun_out/ncu_spmm.log 2>&1
