for js in 1; do TTK_JAC_DEBUG=1 timeout 120 python tools/debug/jac_debug.py c4 $js 2>&1 | grep "^JAC\|^---\|flow cta0" | tail -9; done
