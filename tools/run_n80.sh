# 64 x 80 TMA tile (N = 80 j products): parity + timing + c4 / c3 bench lines
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_c4.py::test_c4_round_properties -m gpu -q -x > gpurun_out/pt_n80.log 2>&1; echo "rc=$?" >> gpurun_out/pt_n80.log
tail -4 gpurun_out/pt_n80.log
timeout 300 python tools/ubench/gemm_feed.py 5 2>&1 | grep -v max | grep form_U1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --breakdown > gpurun_out/bench_c4_n80.json 2> gpurun_out/bench_c4_n80.err
python -c "
import json
d=json.load(open('gpurun_out/bench_c4_n80.json'))
print('c4', d['ms_per_step'], d['roofline']['frac'], d['phases_ms_per_step'])"
