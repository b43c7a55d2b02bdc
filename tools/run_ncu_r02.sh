# ncu --set full captures of the dominant kernels (indices from profiles/r02/launches_c4_r02.csv)
# and the DRAM traffic of the dgemm launches of one c4 bench step.
mkdir -p gpurun_out
C="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
$C > gpurun_out/plain_r02.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dgemm_kernel -s 153 -c 1 -o gpurun_out/prof_r02_formW $C > gpurun_out/ncu_formW.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jacobi_persistent_k -s 8 -c 1 -o gpurun_out/prof_r02_jacobi $C > gpurun_out/ncu_jacobi.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:dgemm_kernel --csv --log-file gpurun_out/dgemm_traffic_r02.csv $C > gpurun_out/ncu_traffic.log 2>&1
