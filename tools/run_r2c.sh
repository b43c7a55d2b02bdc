# Round-2 stage c: re-entry baseline — full GPU suite + bench lines c4/c3/c5.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pt_r2c.log 2>&1; echo "rc=$?" >> gpurun_out/pt_r2c.log
python bench.py --steps 5 --warmup 3 --breakdown > gpurun_out/bench_c4_r2c.json 2> gpurun_out/bench_c4_r2c.err
for c in c3 c5; do timeout 400 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --breakdown > gpurun_out/bench_${c}_r2c.json 2> gpurun_out/bench_${c}_r2c.err; done
tail -3 gpurun_out/pt_r2c.log
