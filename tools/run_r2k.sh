# Round-2 stage k: the bench lines of the final commit (default run = c4, then c3, c5)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_c4_r2k.json 2> gpurun_out/bench_c4_r2k.err
timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --breakdown > gpurun_out/bench_c3_r2k.json 2> gpurun_out/bench_c3_r2k.err
timeout 300 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_r2k.json 2> gpurun_out/bench_c5_r2k.err
python -c "
import json
for c in ('c4','c3','c5'):
    d=json.load(open(f'gpurun_out/bench_{c}_r2k.json')); print(c, d['ms_per_step'], d['value'], d['e2e']['value'], (d.get('roofline') or {}).get('frac'), d['clocks']['reasons'])"
