# NEXT-3 GPU parity (tests/test_gpu_precond.py) under a hard timeout
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_precond.py -q -x -k "${K:-not golden}" --durations=10 > gpurun_out/pt_prec.log 2>&1
echo "rc=$?" >> gpurun_out/pt_prec.log
