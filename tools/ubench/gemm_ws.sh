# TMA-bulk-copy warp-specialised DMMA GEMM experiment (tools/ubench/gemm_ws.cu) on the c4 form_W shape
set -e
mkdir -p gpurun_out
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/gemm_ws tools/ubench/gemm_ws.cu \
  -Lpaper_1906_06785_b200 -lttk -Xlinker -rpath=$PWD/paper_1906_06785_b200
timeout 300 /tmp/gemm_ws 5 > gpurun_out/gemm_ws.txt 2>&1
