# TMA-fed DMMA GEMM: parity tests of tk_gemm (both feeds) + timing on the c4 heavy shapes
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py -m gpu -q -x > gpurun_out/pt_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/pt_gemm.log
tail -15 gpurun_out/pt_gemm.log
timeout 300 python tools/ubench/gemm_feed.py 5 > gpurun_out/gemm_feed.txt 2>&1
cat gpurun_out/gemm_feed.txt
