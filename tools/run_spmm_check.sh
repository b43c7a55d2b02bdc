# SpMM variants at c4 (column-merged V2 / scalar, per-term), apply parity, one ncu capture
python -m pytest tests/test_gpu_parity.py -q -x -k "apply" 2>&1 | tail -3 > gpurun_out/pt2.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --breakdown > gpurun_out/b2.json 2> gpurun_out/b2.err
TTK_SPMM_NATURAL=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --breakdown > gpurun_out/b2s.json 2> gpurun_out/b2s.err
ncu --set full --clock-control none --import-source on -k regex:spmm_merged -c 1 -o gpurun_out/prof_spmm_s python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_sm.log 2>&1
