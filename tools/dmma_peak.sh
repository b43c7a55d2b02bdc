# FP64 DMMA ceiling on this B200: register-only mma.sync m8n8k4 f64 chains (tools/ubench/dmma_peak.cu),
# with nvidia-smi SM clocks sampled while it runs.  Output -> gpurun_out/dmma_peak.txt
set -e
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/dmma_peak tools/ubench/dmma_peak.cu
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active,power.draw --format=csv,noheader -lms 100 > /tmp/dmma_clk.csv &
SMI=$!
/tmp/dmma_peak > /tmp/dmma_out.txt
/tmp/dmma_peak >> /tmp/dmma_out.txt
kill $SMI || true
{ echo "== tools/ubench/dmma_peak.cu (two runs)"; cat /tmp/dmma_out.txt; echo "== nvidia-smi samples (sm MHz, max MHz, throttle reasons, W)"; sort /tmp/dmma_clk.csv | uniq -c | sort -rn | head -8; nvidia-smi --query-gpu=name,driver_version --format=csv,noheader; } > gpurun_out/dmma_peak.txt
