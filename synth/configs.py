"""The five named configurations of BASELINE.json (``configs``), as read in DESIGN.md, plus c6
(NEXT-1: the TT convection operator, not a BASELINE.json config).

c1..c4: apply + round on a seeded operator and input TT.  c5: one 20-step low-rank GMRES
cycle on the c2 operator.  nu values for c3/c4 are unstated in BASELINE.json; the c2 rule
nu_k = 0.01 * 0.5^k is used (R9).  tau = 1/n_t except c1 (tau = 0.1, R12).
"""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass(frozen=True)
class Config:
    name: str
    index: int            # 0-based position in BASELINE.json configs; also the RNG seed
    grid: int             # N (interior nodes per direction); n_x = 3 N^2
    m: int                # number of random variables xi_1..xi_m
    p: int                # total degree d_psi
    n_t: int              # time steps
    tau: float            # backward-Euler step
    nus: tuple            # (nu_0, nu_1, ..., nu_m)
    wind_rank: int        # R_w: mean wind w_0 plus R_w - 1 stochastic wind modes
    ranks: tuple          # input TT ranks (r1, r2)
    tol: float            # rounding tolerance epsilon
    rmax: int             # rank cap (0 = none)
    input_kind: str       # "gauss" (N(0,1) cores) or "decay" (0.7^i spectra)
    gmres_steps: int = 0  # c5 only
    rhs_ranks: tuple = field(default=(0, 0))
    operator: str = "oseen"  # "convection": the TT convection operator N(u~) (NEXT-1, c6);
    #                          "picard": the Navier-Stokes Picard problem (NEXT-4, c7)
    velocity_ranks: tuple = field(default=(0, 0))  # ranks of the velocity TT u~ (c6)

    @property
    def n_x(self) -> int:
        return 3 * self.grid * self.grid

    @property
    def n_terms(self) -> int:
        if self.operator == "convection":  # one term per (alpha_1, alpha_2), eq:N_kron
            return self.velocity_ranks[0] * self.velocity_ranks[1]
        if self.operator == "picard":  # time-mass + Stokes block + m KL terms (N(u) is added)
            return 2 + self.m
        # time-mass + mean Oseen + m KL terms + (R_w - 1) wind terms (R8)
        return 2 + self.m + (self.wind_rank - 1)


def _nus(m: int) -> tuple:
    return tuple(0.01 * 0.5 ** k for k in range(m + 1))


CONFIGS = {
    "c1": Config("c1", 0, 16, 2, 2, 8, 0.1, (0.01, 0.003, 0.002), 1, (4, 4), 1e-10, 0, "gauss"),
    "c2": Config("c2", 1, 64, 4, 3, 64, 1.0 / 64, _nus(4), 1, (20, 20), 1e-8, 80, "decay"),
    "c3": Config("c3", 2, 256, 6, 3, 256, 1.0 / 256, _nus(6), 2, (40, 40), 1e-8, 120, "decay"),
    "c4": Config("c4", 3, 512, 8, 3, 512, 1.0 / 512, _nus(8), 5, (64, 64), 1e-6, 160, "decay"),
    "c5": Config("c5", 4, 64, 4, 3, 64, 1.0 / 64, _nus(4), 1, (20, 20), 1e-6, 0, "decay",
                 gmres_steps=20, rhs_ranks=(8, 8)),
    # NEXT-1, not a BASELINE.json config: apply + round of the TT convection
    # operator N(u~) of eq:N_kron on the c2 sizes, u~ a seeded decaying
    # velocity TT of ranks (8, 8) -> 64 terms, x the c2-style input (20, 20) -> (1280, 1280)
    "c6": Config("c6", 5, 64, 4, 3, 64, 1.0 / 64, _nus(4), 1, (20, 20), 1e-8, 80, "decay",
                 operator="convection", velocity_ranks=(8, 8)),
    # NEXT-4, not BASELINE.json configs: the inexact Picard iteration of Alg. 1
    # (eq:inexact_solve :536-538) on the all-at-once stochastic Galerkin
    # Navier-Stokes system (eq:ns_sys_all) with a seeded body force; nu_0 = 1/50 as in the
    # paper's Table 1, KL viscosity nu_l = 0.002 / l; tol = eps_gmres.
    # c7: the oracle-parity size; c8: GPU-scale (checked through properties)
    "c7": Config("c7", 6, 4, 1, 2, 4, 1.0 / 4, (0.02, 0.002), 1, (1, 1), 1e-5, 0, "gauss",
                 operator="picard"),
    "c8": Config("c8", 7, 16, 2, 2, 8, 1.0 / 8, (0.02, 0.002, 0.001), 1, (1, 1), 1e-4, 0,
                 "gauss", operator="picard"),
}


def get_config(name: str) -> Config:
    return CONFIGS[name]
