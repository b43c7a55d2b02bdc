# ncu --set full of the latency-bound small kernels (QR panel, Jacobi) at c4.
C="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
$C > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:qr_panel_warp -s 20 -c 1 -o gpurun_out/prof_qrpanel $C > gpurun_out/ncu5.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:jacobi_persistent -c 1 -o gpurun_out/prof_jacobi2 $C > gpurun_out/ncu6.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:pchol_panel -s 10 -c 1 -o gpurun_out/prof_pchol $C > gpurun_out/ncu7.log 2>&1
