# Round-2 stage h (final code): full GPU suite with a hard test timeout, bench lines
mkdir -p gpurun_out
timeout 1200 python -X faulthandler -m pytest tests -m gpu -q -x -o faulthandler_timeout=400 --durations=8 > gpurun_out/pt_r2h.log 2>&1; echo "rc=$?" >> gpurun_out/pt_r2h.log
tail -4 gpurun_out/pt_r2h.log
timeout 600 python bench.py --steps 5 --warmup 3 --breakdown > gpurun_out/bench_c4_r2h.json 2> gpurun_out/bench_c4_r2h.err
for c in c3 c5 c6; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --breakdown > gpurun_out/bench_${c}_r2h.json 2> gpurun_out/bench_${c}_r2h.err; done
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2h.log 2>&1; tail -1 gpurun_out/smoke_r2h.log
