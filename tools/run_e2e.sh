mkdir -p gpurun_out
python tools/debug/e2e_diag.py > gpurun_out/e2e_diag2.txt 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_c4.json 2> gpurun_out/e2e_c4.err
python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_c3.json 2> gpurun_out/e2e_c3.err
timeout 900 python -m pytest tests/test_gpu_async.py tests/test_gpu_parity.py -q -x > gpurun_out/e2e_pt.log 2>&1; echo "rc=$?" >> gpurun_out/e2e_pt.log
