"""B200-native (sm_100a, fp64) tensor-train hot path of arXiv:1906.06785.

apply A = sum_k T_k (x) G_k (x) K_k to a 3-core TT, TT-round, TT dot/axpby, one low-rank GMRES
cycle — all in libttk.so (hand-written CUDA, C ABI in include/ttk.h).  This package is the
thin Python binding; it never imports the CPU oracle and has no CPU fallback.
"""
from .ttk import (TK_EARG, TK_ECAP, TK_ECUDA, TK_ENUMERIC, TK_ESHAPE, TK_OK, TT,  # noqa: F401
                  BlockTridiag, Context, Convection, MeanLSC, Operator, RoundInfo, TkError,
                  default_context, gmres_cycle, gmres_solve, lib, picard, round_workspace_bytes, tt_apply_op, tt_apply_round,
                  tt_axpby, tt_dot, tt_norm, tt_round)
