"""Write oracle-derived golden files under tests/golden/ (calls ONLY oracle/ and synth/).

    python tools/make_golden.py c5      # c5 GMRES-cycle residual history (~20+ min on 8 cores)
    python tools/make_golden.py c5p     # c5's operator, 3 flexible steps with the mean-based
                                        # LSC preconditioner (NEXT-3; ~8 min)

The GPU parity test for c5 compares the CUDA path with this stored oracle history instead of
re-running the 20-minute CPU oracle inside the GPU test session.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.gmres import gmres_cycle  # noqa: E402
from oracle.precond import MeanLSC  # noqa: E402
from synth.configs import CONFIGS  # noqa: E402
from synth.operator import build_operator, mean_blocks  # noqa: E402
from synth.tt import make_rhs_tt  # noqa: E402


def c5():
    cfg = CONFIGS["c5"]
    op = build_operator(cfg)
    b = make_rhs_tt(cfg, op.n_xi)
    t0 = time.time()
    res = gmres_cycle(op, b, steps=cfg.gmres_steps, tol=cfg.tol)
    out = {
        "_about": "oracle/gmres.py gmres_cycle on config c5 (BASELINE.json configs[4]); written by "
                  "tools/make_golden.py, which calls only oracle/ and synth/",
        "config": "c5", "steps": int(res["steps"]), "tol": cfg.tol,
        "history": [float(h) for h in res["history"]],
        "explicit_residual": float(res["explicit"]),
        "ranks": [list(map(int, r)) for r in res["ranks"]],
        "oracle_seconds": time.time() - t0,
    }
    path = os.path.join(ROOT, "tests", "golden", "c5_gmres_oracle.json")
    json.dump(out, open(path, "w"), indent=1)
    print("wrote", path, out["oracle_seconds"])


def c5p():
    cfg = CONFIGS["c5"]
    op = build_operator(cfg)
    F0s, B = mean_blocks(cfg)  # the mean blocks of c5's own operator (its wind seed)
    b = make_rhs_tt(cfg, op.n_xi)
    steps = 3
    t0 = time.time()
    P = MeanLSC(F0s, B, cfg.tau, op.n_xi, op.n_t, tol=cfg.tol)
    res = gmres_cycle(op, b, steps=steps, tol=cfg.tol, prec=P.apply)
    out = {
        "_about": "oracle/gmres.py gmres_cycle with prec = oracle/precond.py MeanLSC(tol = 1e-6, "
                  "inner tol 1e-1, restart 10, 3 cycles) on config c5's operator and RHS; written "
                  "by tools/make_golden.py, which calls only oracle/ and synth/",
        "config": "c5", "steps": steps, "steps_done": int(res["steps"]), "tol": cfg.tol,
        "history": [float(h) for h in res["history"]],
        "explicit": float(res["explicit"]),
        "inner": [[int(c), float(r)] for c, r in P.inner_stats],
        "oracle_seconds": time.time() - t0,
    }
    path = os.path.join(ROOT, "tests", "golden", "c5p_gmres_oracle.json")
    json.dump(out, open(path, "w"), indent=1)
    print("wrote", path, out["oracle_seconds"])


if __name__ == "__main__":
    for name in sys.argv[1:] or ["c5"]:
        globals()[name]()
