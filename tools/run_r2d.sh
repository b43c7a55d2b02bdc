# Round-2 stage d: TMA-fed GEMM — GEMM feed timing, full GPU suite, bench lines c4/c3/c5.
mkdir -p gpurun_out
timeout 300 python tools/ubench/gemm_feed.py 5 > gpurun_out/gemm_feed.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pt_r2d.log 2>&1; echo "rc=$?" >> gpurun_out/pt_r2d.log
python bench.py --steps 5 --warmup 3 --breakdown > gpurun_out/bench_c4_r2d.json 2> gpurun_out/bench_c4_r2d.err
for c in c3 c5; do timeout 400 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --breakdown > gpurun_out/bench_${c}_r2d.json 2> gpurun_out/bench_${c}_r2d.err; done
cat gpurun_out/gemm_feed.txt | grep -v max; tail -3 gpurun_out/pt_r2d.log
