for m in none round2 applyround h2d h2dbig; do echo "== $m"; timeout 60 python tools/debug/async_repro.py $m 2>&1 | tail -12; echo "rc=$?"; done > gpurun_out/async_repro.log 2>&1
