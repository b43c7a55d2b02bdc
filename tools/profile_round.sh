# Round profile bundle (run under gpurun): GPU tests, full bench lines (c4 default, c5), then
# the per-launch list of one c4 step under ncu (after the same command exited 0 without ncu).
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python bench.py --config c5 --steps 1 --warmup 1 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline \
    > gpurun_out/ncu_launches.log 2>&1
