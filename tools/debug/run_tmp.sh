timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "wide_time_bond or parity_c2 or parity_c3 or tall" 2>&1 | tail -2
for c in c3 c4; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --breakdown 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
p=d['phases_ms_per_step']
print('$c', round(d['ms_per_step'],2), 'pchol_panel', p.get('pchol_panel'), 'pchol', p.get('pchol'))"; done
timeout 300 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('c5', d['ms_per_step'])"
