# NEXT-3/4 GPU parity under a hard timeout
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_picard.py tests/test_gpu_precond.py tests/test_gpu_parity.py -q -x -k "${K:-not golden}" --durations=10 > gpurun_out/pt_picard.log 2>&1
echo "rc=$?" >> gpurun_out/pt_picard.log
