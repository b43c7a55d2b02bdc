# Round-2 stage l: full GPU suite + smoke + bench lines on the final commit
mkdir -p gpurun_out
timeout 1200 python -X faulthandler -m pytest tests -m gpu -q -x -o faulthandler_timeout=400 > gpurun_out/pt_r2l.log 2>&1; echo "rc=$?" >> gpurun_out/pt_r2l.log
tail -3 gpurun_out/pt_r2l.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2l.log 2>&1; tail -1 gpurun_out/smoke_r2l.log
timeout 900 python bench.py > gpurun_out/bench_c4_r2l.json 2> gpurun_out/bench_c4_r2l.err
timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --breakdown > gpurun_out/bench_c3_r2l.json 2> gpurun_out/bench_c3_r2l.err
timeout 300 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_r2l.json 2> gpurun_out/bench_c5_r2l.err
python -c "
import json
for c in ('c4','c3','c5'):
    d=json.load(open(f'gpurun_out/bench_{c}_r2l.json')); print(c, d['ms_per_step'], d['value'], d['e2e']['value'], (d.get('roofline') or {}).get('frac'), d['clocks']['reasons'])"
