"""Write oracle-derived golden files under tests/golden/ (calls ONLY oracle/ and synth/).

    python tools/make_golden.py c5      # c5 GMRES-cycle residual history (~20+ min on 8 cores)

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
from synth.configs import CONFIGS  # noqa: E402
from synth.operator import build_operator  # noqa: E402
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


if __name__ == "__main__":
    for name in sys.argv[1:] or ["c5"]:
        globals()[name]()
