mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_convection.py -q -x -k "tall_panels or c5 or convection" --durations=5 > gpurun_out/pt_qrbig.log 2>&1; echo "rc=$?" >> gpurun_out/pt_qrbig.log
for c in c6 c3; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --breakdown > gpurun_out/bench_${c}_qrbig.json 2> gpurun_out/bench_${c}_qrbig.err; done
