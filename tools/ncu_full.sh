# ncu --set full captures of the top kernels at c4 (run under gpurun, after a plain run exits 0).
C="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
$C > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:jacobi_persistent -c 1 -o gpurun_out/prof_jacobi $C > gpurun_out/ncu1.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:spmm_multi -c 1 -o gpurun_out/prof_spmm $C > gpurun_out/ncu2.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:stoch_apply -c 1 -o gpurun_out/prof_stoch $C > gpurun_out/ncu3.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:dgemm_kernel -s 446 -c 1 -o gpurun_out/prof_gramW $C > gpurun_out/ncu4.log 2>&1
