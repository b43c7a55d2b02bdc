# Round-2 stage j: last full check of the final commit (GPU suite with hard timeouts, smoke)
mkdir -p gpurun_out
timeout 1200 python -X faulthandler -m pytest tests -m gpu -q -x -o faulthandler_timeout=400 --durations=5 > gpurun_out/pt_r2j.log 2>&1; echo "rc=$?" >> gpurun_out/pt_r2j.log
tail -4 gpurun_out/pt_r2j.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2j.log 2>&1; tail -1 gpurun_out/smoke_r2j.log
