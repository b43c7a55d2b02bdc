# Per-call Jacobi sizes/sweeps of one c5 GMRES cycle (TTK_DEBUG lines to gpurun_out/gdbg.err)
TTK_DEBUG=1 python - <<'PY' 2> gpurun_out/gdbg.err
import sys; sys.path.insert(0,'.')
import paper_1906_06785_b200 as ttk
from synth.configs import CONFIGS
from synth.operator import build_operator
from synth.tt import make_rhs_tt
cfg=CONFIGS['c5']; op=build_operator(cfg); b=make_rhs_tt(cfg, op.n_xi)
g=ttk.Operator.from_kronsum(op); ttk.gmres_cycle(g, ttk.TT.from_cores(*b), 20, cfg.tol)
PY
