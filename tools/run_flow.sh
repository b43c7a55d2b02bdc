# Dataflow Jacobi schedule: parity (bitwise vs the barrier schedule) + A/B timing
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_schedule.py -m gpu -q -x > gpurun_out/pt_flow.log 2>&1; echo "rc=$?" >> gpurun_out/pt_flow.log
tail -25 gpurun_out/pt_flow.log
for js in 0 1; do
  for c in c3 c4; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --breakdown --jacobi-schedule $js > gpurun_out/bench_${c}_js$js.json 2> gpurun_out/bench_${c}_js$js.err; done
  timeout 300 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --jacobi-schedule $js > gpurun_out/bench_c5_js$js.json 2> gpurun_out/bench_c5_js$js.err
done
python - <<'PY'
import json
for c in ("c3","c4","c5"):
    for js in (0,1):
        try:
            d=json.load(open(f"gpurun_out/bench_{c}_js{js}.json"))
            print(c, "js", js, round(d["ms_per_step"],2), "jacobi", (d.get("phases_ms_per_step") or {}).get("jacobi"))
        except Exception as e:
            print(c, js, "ERR", e)
PY
