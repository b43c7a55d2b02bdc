# Step-time distribution at c4 with and without a pre-reserved memory pool.
export TTK_BENCH_NOCLOCKS=1
B="python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --breakdown"
$B > gpurun_out/o_plain.json 2> gpurun_out/o_plain.err
TTK_POOL_RESERVE_GB=40 $B > gpurun_out/o_res.json 2> gpurun_out/o_res.err
