mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pt_r2a.log 2>&1
python bench.py --steps 5 --warmup 3 --breakdown > gpurun_out/bench_c4_r2a.json 2> gpurun_out/bench_c4_r2a.err
for c in c3 c5 c6; do python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --breakdown > gpurun_out/bench_${c}_r2a.json 2> gpurun_out/bench_${c}_r2a.err; done
