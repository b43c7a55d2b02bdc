# Diagnostics: per-call Jacobi sweeps / phase times for rounding variants (TTK_DEBUG).
export TTK_BENCH_NOCLOCKS=1
B="python bench.py --config ${CFG:-c4} --steps 1 --warmup 1 --no-cpu-baseline --breakdown"
for v in ${VARIANTS:-base}; do
  case $v in
    base) env TTK_DEBUG=1 $B ;;
    full) env TTK_DEBUG=1 TTK_FULL_PASS1_GRAM=1 $B ;;
    jac) env TTK_DEBUG=1 TTK_PASS1=jacobi $B ;;
    cskip) env TTK_DEBUG=1 TTK_CLUSTER_SKIP=1 $B ;;
    rskip) env TTK_DEBUG=1 TTK_CLUSTER_SKIP=1 TTK_RANK_SKIP=1 $B ;;
    b1id) env TTK_DEBUG=1 TTK_BOND1_PASS1_ID=1 $B ;;
  esac > gpurun_out/d_$v.json 2> gpurun_out/d_$v.err
done
