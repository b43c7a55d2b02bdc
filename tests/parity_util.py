"""Shared comparison helpers of the GPU parity tests (R5, R7).  Test code only."""
import numpy as np

from oracle import tt as otT


def tt_diff_rel(a, b):
    """||a - b||_F / ||b||_F for TTs too large to densify: orthogonalise the TT a + (-b)
    with the oracle at tol 0 and read the norm off the last core (hard part 4)."""
    d = otT.round_tt(otT.axpby(1.0, a, -1.0, b), 0.0)
    nb = otT.round_tt(b, 0.0)
    return float(np.linalg.norm(d[2]) / max(np.linalg.norm(nb[2]), 1e-300))


def ranks_excused(sig, delta, r_gpu, r_orc, rmax):
    """DESIGN.md R5: a rank mismatch is a tie if the tail at the boundary is within 1e-10 ||x||
    of delta, if rmax binds and the singular values straddling it are within 1e-10 s_1, or if
    every singular value from the smaller rank's last kept one to the larger rank's is within
    1e-10 s_1 of the others (the tie rule of SPEC.md:109 decides on EXACT equality, which two
    backward-stable computations of a repeated value need not reproduce)."""
    if r_gpu == r_orc:
        return True
    nrm = np.linalg.norm(sig)
    lo = min(r_gpu, r_orc)
    hi = max(r_gpu, r_orc)
    run = sig[lo - 1:hi]
    if len(run) and np.max(run) - np.min(run) <= 1e-10 * sig[0]:
        return True
    tail = np.linalg.norm(sig[lo:])
    if abs(tail - delta) <= 1e-10 * nrm:
        return True
    if rmax and max(r_gpu, r_orc) == rmax and abs(sig[rmax - 1] - sig[min(rmax, len(sig) - 1)]) <= 1e-10 * sig[0]:
        return True
    return False
