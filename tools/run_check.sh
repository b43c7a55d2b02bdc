# GPU parity tests + a c4 bench line with the per-phase breakdown
python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/pt.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --breakdown > gpurun_out/b.json 2> gpurun_out/b.err
