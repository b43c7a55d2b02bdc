# DMMA GEMM tile-configuration experiment (tools/ubench/gemm_tiles.cu) on the c4 GEMM shapes
set -e
mkdir -p gpurun_out
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/gemm_tiles tools/ubench/gemm_tiles.cu \
  -Lpaper_1906_06785_b200 -lttk -Xlinker -rpath=$PWD/paper_1906_06785_b200
timeout 400 /tmp/gemm_tiles 4 > gpurun_out/gemm_tiles.txt 2>&1
