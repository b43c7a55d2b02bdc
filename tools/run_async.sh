mkdir -p gpurun_out
bash tools/debug/async_repro.sh
timeout 600 python -m pytest tests/test_gpu_async.py -q -x --durations=10 > gpurun_out/pt_async.log 2>&1
echo "rc=$?" >> gpurun_out/pt_async.log
