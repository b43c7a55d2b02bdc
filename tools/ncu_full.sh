# ncu --set full captures of the top kernels at c4 (run under gpurun, after a plain run exits 0).
# dgemm launch indices (among dgemm_kernel launches of one step) from the launch list:
# 163 = bond1.form_W, 164 = bond1.gram_W, 215 = bond1.form_U1.
C="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
$C > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmm_merged -c 1 -o gpurun_out/prof_spmm $C > gpurun_out/ncu1.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:dgemm_kernel -s 163 -c 2 -o gpurun_out/prof_formW $C > gpurun_out/ncu2.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:dgemm_kernel -s 215 -c 1 -o gpurun_out/prof_formU1 $C > gpurun_out/ncu3.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:axpby_u1 -c 1 -o gpurun_out/prof_axpby $C > gpurun_out/ncu4.log 2>&1
