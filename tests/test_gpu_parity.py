"""GPU-vs-oracle parity through the C ABI (libttk.so) — the parity tests proper.

Bars (BASELINE.json north_star):
  apply      : exact arithmetic path, rel. error <= 1e-13 per core
  round      : relative Frobenius error of the reconstructed tensor <= 1e-10, singular values
               |s_gpu - s_orc| <= 1e-10 s_1, identical ranks away from ties (R5)
  dot / norm : <= 1e-12 relative;  axpby exact
  GMRES (c5) : residual history within 1e-8 relative (to beta)
"""
import json
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1906_06785_b200 as ttk  # noqa: E402
from oracle import tt as otT  # noqa: E402
from oracle.gmres import gmres_cycle as o_gmres  # noqa: E402
from synth.configs import CONFIGS  # noqa: E402
from synth.operator import build_operator, random_operator  # noqa: E402
from synth.tt import make_input_tt, make_rhs_tt, random_tt  # noqa: E402
from parity_util import ranks_excused, tt_diff_rel  # noqa: E402,F401

TOL_TENSOR = 1e-10
TOL_SIGMA = 1e-10


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def ctx():
    return ttk.default_context()


def gpu_op(op, ctx):
    return ttk.Operator.from_kronsum(op, ctx)


# ----------------------------------------------------------------------------- apply
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_apply_parity_configs(name, ctx):
    cfg = CONFIGS[name]
    op = build_operator(cfg)
    x = make_input_tt(cfg, op.n_xi)
    y_o = otT.apply_op(op, x)
    y_g = ttk.tt_apply_op(gpu_op(op, ctx), ttk.TT.from_cores(*x)).cores_numpy()
    for a, b in zip(y_g, y_o):
        assert a.shape == b.shape
        assert rel(a, b) <= 1e-13


@pytest.mark.parametrize("seed", range(6))
def test_apply_parity_random_ragged(seed, ctx):
    rng = np.random.default_rng(seed)
    n_x = int(rng.integers(1, 300))
    n_xi, n_t = int(rng.integers(1, 12)), int(rng.integers(1, 40))
    T = int(rng.integers(1, 5))
    r1 = [1, 3, 17, 33, 65, 97][seed]
    r2 = int(rng.integers(1, 9))
    op = random_operator(rng, n_x, n_xi, n_t, T, density=0.05, max_band=3)
    x = random_tt(rng, n_x, n_xi, n_t, r1, r2)
    y_o = otT.apply_op(op, x)
    y_g = ttk.tt_apply_op(gpu_op(op, ctx), ttk.TT.from_cores(*x)).cores_numpy()
    for a, b in zip(y_g, y_o):
        assert rel(a, b) <= 1e-13


@pytest.mark.parametrize("T,n_x,density,r1,perterm", [
    (17, 60, 0.1, 8, False),    # T > 16: the per-term kernel
    (16, 80, 0.6, 64, False),   # rows with > 32 distinct columns and > 256 values (unstaged)
    (9, 200, 0.02, 66, False),  # two column chunks, ragged second chunk
    (5, 150, 0.3, 7, False),    # odd r: scalar lanes
    (6, 150, 0.3, 40, True),    # tk_op_set_spmm_kernel(op, 1)
])
def test_apply_spmm_paths(T, n_x, density, r1, perterm, ctx):
    """Both SpMM kernels (column-merged for T <= 16, per-term otherwise or on request) and the
    merged kernel's group / staging limits, vs the oracle apply."""
    rng = np.random.default_rng(T * 1000 + n_x)
    op = random_operator(rng, n_x, 3, 5, T, density=density, max_band=1)
    x = random_tt(rng, n_x, 3, 5, r1, 2)
    y_o = otT.apply_op(op, x)
    gop = gpu_op(op, ctx)
    if perterm:
        assert gop.set_spmm_kernel(1) is False
    y_g = ttk.tt_apply_op(gop, ttk.TT.from_cores(*x)).cores_numpy()
    for a, b in zip(y_g, y_o):
        assert rel(a, b) <= 1e-13


def test_apply_spmm_long_records(ctx):
    """Merged SpMM rows whose record exceeds the 96 staged words (<= 32 distinct columns but
    16 terms on each: ~20 x 16 values per row) take the unstaged path: values from global."""
    import scipy.sparse as sp
    from synth.operator import KronSumOp, Term
    rng = np.random.default_rng(31)
    n_x, T = 90, 16
    pat = sp.random(n_x, n_x, density=0.22, random_state=rng, format="csr")
    terms = []
    for k in range(T):
        K = pat.copy()
        K.data = rng.standard_normal(K.nnz)
        K.indices = K.indices.astype(np.int32)
        K.indptr = K.indptr.astype(np.int32)
        K.sort_indices()
        terms.append(Term(f"t{k}", 0, 0, rng.standard_normal((1, 4)), rng.standard_normal((3, 3)), K))
    op = KronSumOp(n_x, 3, 4, terms)
    assert max(np.diff(pat.indptr)) <= 32 and max(np.diff(pat.indptr)) * (T + 1) > 96
    x = random_tt(rng, n_x, 3, 4, 40, 2)
    y_o = otT.apply_op(op, x)
    y_g = ttk.tt_apply_op(gpu_op(op, ctx), ttk.TT.from_cores(*x)).cores_numpy()
    for a, b in zip(y_g, y_o):
        assert rel(a, b) <= 1e-13


def test_apply_capacity_and_shape_errors(ctx):
    rng = np.random.default_rng(3)
    op = random_operator(rng, 10, 3, 4, 2)
    g = gpu_op(op, ctx)
    x = ttk.TT.from_cores(*random_tt(rng, 10, 3, 4, 2, 2))
    small = ttk.TT(10, 3, 4, 2, 2)
    with pytest.raises(ttk.TkError) as e:
        ttk.tt_apply_op(g, x, out=small)
    assert e.value.code == -2
    bad = ttk.TT.from_cores(*random_tt(rng, 11, 3, 4, 2, 2))
    with pytest.raises(ttk.TkError) as e:
        ttk.tt_apply_op(g, bad)
    assert e.value.code == -1


# ----------------------------------------------------------------------------- round
def check_round(y_cores, tol, rmax, ctx, dense=True, gpu=None):
    """Oracle round of y_cores vs the GPU: tk_round on the same cores, or gpu() -> (TT, info)
    (the fused tk_apply_round on the operator and input that produced y_cores)."""
    o, info = otT.round_tt(y_cores, tol, rmax, return_info=True)
    if gpu is None:
        g = ttk.TT.from_cores(*y_cores)
        g, ginfo = ttk.tt_round(g, tol, rmax, ctx, want_info=True)
    else:
        g, ginfo = gpu()
    gc = g.cores_numpy()
    assert ranks_excused(info["sigma1"], info["delta"], ginfo.ranks[0], info["ranks"][0], rmax)
    # kept singular values to 1e-10 s_1 and the discarded tail norms to 1e-10 ||x|| (DESIGN.md
    # R6: values below the cut only enter through their tail sum)
    k = min(ginfo.ranks[0], info["ranks"][0])
    assert np.max(np.abs(ginfo.sigma1[:k] - info["sigma1"][:k])) <= TOL_SIGMA * info["sigma1"][0]
    if ginfo.ranks == info["ranks"]:
        k2 = ginfo.ranks[1]
        assert np.max(np.abs(ginfo.sigma2[:k2] - info["sigma2"][:k2])) <= TOL_SIGMA * max(info["sigma2"][0], 1e-300)
        for a, b in zip(ginfo.discarded, info["discarded"]):
            assert abs(a - b) <= TOL_SIGMA * info["norm"]
        err = rel(otT.full(gc), otT.full(o)) if dense else tt_diff_rel(gc, o)
        assert err <= TOL_TENSOR, err
    assert ginfo.norm == pytest.approx(info["norm"], rel=1e-12)
    # invariants of the GPU output
    u1, u2, u3 = gc
    assert np.max(np.abs(u1.T @ u1 - np.eye(u1.shape[1]))) <= 1e-10
    m2 = u2.reshape(-1, u2.shape[2])
    assert np.max(np.abs(m2.T @ m2 - np.eye(m2.shape[1]))) <= 1e-10
    return ginfo, info


@pytest.mark.parametrize("rmax", [0, 2, 3])
def test_round_tie_spectrum(rmax, ctx):
    """Exactly repeated singular values at the delta cut and at rmax (sigma = [1, .5, .5, .5, .1],
    delta = 0.6: the tail rule gives 3, the tie rule 4, rmax caps last).  Which vectors of a
    tied subspace are kept is not unique, so this compares what is: the ranks (equal or
    excused by R5's tie clauses), the kept sigma, the bond-1 discarded norm, ||x~|| and — when
    rmax cuts through the tie, where the error is unique — ||x~ - x|| to 1e-10 ||x||."""
    rng = np.random.default_rng(77 + rmax)
    sig = np.array([1.0, 0.5, 0.5, 0.5, 0.1])
    n = (40, 7, 9)
    u1 = np.linalg.qr(rng.standard_normal((n[0], 5)))[0]
    q = np.linalg.qr(rng.standard_normal((n[1], 5)))[0]
    w = np.linalg.qr(rng.standard_normal((n[2], 5)))[0].T
    u2 = np.zeros((5, n[1], 5))
    for a in range(5):
        u2[a, :, a] = sig[a] * q[:, a]
    x = (u1, u2, w)
    nrm = np.linalg.norm(sig)
    tol = 0.6 * math.sqrt(2) / nrm
    o, info = otT.round_tt(x, tol, rmax, return_info=True)
    g, ginfo = ttk.tt_round(ttk.TT.from_cores(*x), tol, rmax, ctx, want_info=True)
    assert ranks_excused(info["sigma1"], info["delta"], ginfo.ranks[0], info["ranks"][0], rmax)
    if rmax:
        assert ginfo.ranks[0] == info["ranks"][0] == min(4, rmax)
    assert np.max(np.abs(ginfo.sigma1[:5] - sig)) <= TOL_SIGMA
    r1 = ginfo.ranks[0]
    assert ginfo.discarded[0] == pytest.approx(np.linalg.norm(sig[r1:]), abs=1e-10 * nrm)
    xf = otT.full(x)
    e_g = np.linalg.norm(otT.full(g.cores_numpy()) - xf)
    e_o = np.linalg.norm(otT.full(o) - xf)
    # the bond-2 spectrum depends on WHICH vectors of the tied subspace bond 1 kept, so past
    # bond 1 only validity is checked: the error is the nested-projection sum of the two
    # reported discarded norms, on both sides, and within the bound when rmax does not bind
    d1, d2 = ginfo.discarded
    assert abs(e_g ** 2 - (d1 ** 2 + d2 ** 2)) <= 1e-10 * nrm ** 2
    o1, o2 = info["discarded"]
    assert abs(e_o ** 2 - (o1 ** 2 + o2 ** 2)) <= 1e-10 * nrm ** 2
    if not rmax:
        assert e_g <= tol * nrm * (1 + 1e-10)


@pytest.mark.parametrize("tol", [1e-10, 1e-6, 1e-3, 0.1])
def test_round_parity_c1(tol, ctx):
    cfg = CONFIGS["c1"]
    op = build_operator(cfg)
    y = otT.apply_op(op, make_input_tt(cfg, op.n_xi))
    check_round(y, tol, 0, ctx)


def test_round_parity_c2(ctx):
    cfg = CONFIGS["c2"]
    op = build_operator(cfg)
    y = otT.apply_op(op, make_input_tt(cfg, op.n_xi))
    check_round(y, cfg.tol, cfg.rmax, ctx, dense=False)


@pytest.mark.parametrize("seed", range(12))
def test_round_parity_random(seed, ctx):
    rng = np.random.default_rng(500 + seed)
    n = [int(v) for v in rng.integers(1, 30, size=3)]
    r1, r2 = [int(v) for v in rng.integers(1, 24, size=2)]
    x = random_tt(rng, *n, r1, r2)
    tol = [1e-12, 1e-8, 1e-4, 0.2][seed % 4]
    check_round(x, tol, 0, ctx)


@pytest.mark.parametrize("r1,n_xi,n_t", [(1000, 30, 60), (1700, 45, 40), (2100, 44, 50),
                                        (2500, 200, 20)])
def test_round_parity_tall_panels(r1, n_xi, n_t, ctx):
    """Wide space bonds (R1 > 896 rows in the Householder panels of pass 1 and of the middle
    core's orth_rows): the shared-memory and the register + shared-memory overflow panel kernels
    (qr_panel_warp_k, qr_panel_big_k) — the c5 / c6 apply rounds reach k = 2240; the last case
    (k = 2400 > 2256) also uses the big kernel's global-memory tail."""
    rng = np.random.default_rng(800 + r1)
    x = random_tt(rng, 2600, n_xi, n_t, r1, 12, kind="decay")
    check_round(x, 1e-8, 0, ctx, dense=False)


@pytest.mark.parametrize("r2", [128, 160, 192, 200, 256, 520])
def test_round_wide_time_bond(r2, ctx):
    """R2 >= 128 runs the rank-revealing orth_rows on the R2 x n_t time core (pivoted Cholesky of
    an R2 x R2 Gram): every panel-kernel shared-memory size class, including the exact 48 KB
    edge at R2 = 192 (32 panel rows x 192 doubles) that once failed to launch."""
    rng = np.random.default_rng(700 + r2)
    # n_t = 130 >= 128: the rank-revealing path is taken for every R2 (for n_t < 128 and
    # R2 >= n_t the library keeps Q3 = I, as the oracle does)
    x = random_tt(rng, 40, 3, 130, 5, r2)
    check_round(x, 1e-8, 0, ctx)
    y = random_tt(rng, 40, 3, 6, 5, r2)   # Q3 = I branch
    check_round(y, 1e-8, 0, ctx)


def test_round_rank_one_and_zero(ctx):
    rng = np.random.default_rng(9)
    x = random_tt(rng, 5, 4, 3, 1, 1)
    check_round(x, 1e-8, 0, ctx)
    z = (np.zeros((6, 2)), np.zeros((2, 3, 2)), np.zeros((2, 5)))
    g, info = ttk.tt_round(ttk.TT.from_cores(*z), 1e-3, 0, ctx, want_info=True)
    assert g.ranks == (1, 1) and info.norm == 0.0
    assert not np.any(np.concatenate([c.ravel() for c in g.cores_numpy()]))


def test_round_bad_tol(ctx):
    rng = np.random.default_rng(1)
    g = ttk.TT.from_cores(*random_tt(rng, 4, 3, 3, 2, 2))
    with pytest.raises(ttk.TkError) as e:
        ttk.tt_round(g, -1.0, 0, ctx)
    assert e.value.code == -3


# ----------------------------------------------------------------------------- dot / axpby
@pytest.mark.parametrize("seed", range(5))
def test_dot_norm_axpby_parity(seed, ctx):
    rng = np.random.default_rng(70 + seed)
    n = [int(v) for v in rng.integers(1, 200, size=3)]
    x = random_tt(rng, *n, int(rng.integers(1, 20)), int(rng.integers(1, 20)))
    y = random_tt(rng, *n, int(rng.integers(1, 20)), int(rng.integers(1, 20)))
    gx, gy = ttk.TT.from_cores(*x), ttk.TT.from_cores(*y)
    assert ttk.tt_dot(gx, gy, ctx).item() == pytest.approx(otT.dot(x, y), rel=1e-12, abs=1e-12)
    assert ttk.tt_norm(gx, ctx).item() == pytest.approx(otT.norm(x), rel=1e-12)
    z = ttk.tt_axpby(1.5, gx, -0.25, gy, ctx)
    zo = otT.axpby(1.5, x, -0.25, y)
    for a, b in zip(z.cores_numpy(), zo):
        assert np.array_equal(a, b)
    a_dev = torch.tensor([2.0], dtype=torch.float64, device="cuda")
    z2 = ttk.tt_axpby(a_dev, gx, 1.0, gy, ctx)
    assert np.array_equal(z2.cores_numpy()[2], otT.axpby(2.0, x, 1.0, y)[2])


# ----------------------------------------------------------------------------- c3 (large)
@pytest.mark.slow
def test_round_parity_c3(ctx):
    cfg = CONFIGS["c3"]
    op = build_operator(cfg)
    x = make_input_tt(cfg, op.n_xi)
    y = otT.apply_op(op, x)
    yg = ttk.tt_apply_op(gpu_op(op, ctx), ttk.TT.from_cores(*x))
    for a, b in zip(yg.cores_numpy(), y):
        assert rel(a, b) <= 1e-13
    check_round(y, cfg.tol, cfg.rmax, ctx, dense=False)


# ----------------------------------------------------------------------------- fused apply+round
@pytest.mark.parametrize("name,tol", [("c1", 1e-10), ("c1", 1e-3), ("c2", None)])
def test_apply_round_parity(name, tol, ctx):
    """tk_apply_round (block-diagonal middle core never materialised) vs oracle apply + round."""
    cfg = CONFIGS[name]
    op = build_operator(cfg)
    x = make_input_tt(cfg, op.n_xi)
    tol = cfg.tol if tol is None else tol
    y = otT.apply_op(op, x)
    g = gpu_op(op, ctx)
    check_round(y, tol, cfg.rmax, ctx, dense=(name == "c1"),
                gpu=lambda: ttk.tt_apply_round(g, ttk.TT.from_cores(*x), tol, cfg.rmax,
                                               want_info=True))


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_apply_round_parity_random(seed, ctx):
    """Random operators (T terms, ragged CSR, banded T_k) and odd ranks through the fused path."""
    rng = np.random.default_rng(seed)
    T = int(rng.integers(1, 5))
    n_x, n_xi, n_t = int(rng.integers(20, 90)), int(rng.integers(2, 9)), int(rng.integers(3, 17))
    r1, r2 = int(rng.integers(1, 6)), int(rng.integers(1, 6))
    op = random_operator(rng, n_x, n_xi, n_t, T)
    x = random_tt(rng, n_x, n_xi, n_t, r1, r2)
    y = otT.apply_op(op, x)
    g = gpu_op(op, ctx)
    tol = float(10.0 ** rng.uniform(-10, -2))
    check_round(y, tol, 0, ctx, dense=True,
                gpu=lambda: ttk.tt_apply_round(g, ttk.TT.from_cores(*x), tol, 0, want_info=True))


@pytest.mark.parametrize("shape", [
    # (n_x, n_xi, n_t, T, r1, r2): n_t > T r2 (time core orthogonalised, L3 != identity)
    (40, 3, 24, 2, 3, 2),
    # n_xi k3 <= T r1 (Q2 = identity) and T = 1
    (35, 2, 3, 1, 5, 4),
    # rank one everywhere, several terms
    (50, 4, 6, 3, 1, 1),
])
def test_apply_round_parity_shapes(shape, ctx):
    """Both branches of the identity shortcuts (Q3, Q2) through the fused path."""
    n_x, n_xi, n_t, T, r1, r2 = shape
    rng = np.random.default_rng(sum(shape))
    op = random_operator(rng, n_x, n_xi, n_t, T)
    x = random_tt(rng, n_x, n_xi, n_t, r1, r2)
    y = otT.apply_op(op, x)
    g = gpu_op(op, ctx)
    for tol, rmax in ((1e-12, 0), (1e-4, 0), (1e-6, 2)):
        check_round(y, tol, rmax, ctx, dense=True,
                    gpu=lambda: ttk.tt_apply_round(g, ttk.TT.from_cores(*x), tol, rmax,
                                                   want_info=True))


def test_apply_round_zero_input(ctx):
    """The zero tensor through the fused path canonicalises to ranks (1, 1), zero cores."""
    rng = np.random.default_rng(21)
    op = random_operator(rng, 30, 3, 5, 2)
    x = [np.zeros((30, 2)), np.zeros((2, 3, 2)), np.zeros((2, 5))]
    g = gpu_op(op, ctx)
    y, info = ttk.tt_apply_round(g, ttk.TT.from_cores(*x), 1e-8, 0, want_info=True)
    assert y.ranks == (1, 1)
    assert info.norm == 0.0
    assert all(np.all(c == 0) for c in y.cores_numpy())


@pytest.mark.slow
def test_apply_round_parity_c3(ctx):
    cfg = CONFIGS["c3"]
    op = build_operator(cfg)
    x = make_input_tt(cfg, op.n_xi)
    y = otT.apply_op(op, x)
    g = gpu_op(op, ctx)
    check_round(y, cfg.tol, cfg.rmax, ctx, dense=False,
                gpu=lambda: ttk.tt_apply_round(g, ttk.TT.from_cores(*x), cfg.tol, cfg.rmax,
                                               want_info=True))


# ----------------------------------------------------------------------------- GMRES c5
def _c5_reference(op, b, cfg):
    """The oracle's c5 history: stored by tools/make_golden.py (oracle-only script) because the
    CPU oracle needs ~20 minutes; recomputed live if the file is missing."""
    path = os.path.join(os.path.dirname(__file__), "golden", "c5_gmres_oracle.json")
    if os.path.exists(path):
        g = json.load(open(path))
        return dict(history=np.array(g["history"]), steps=g["steps"], explicit=g["explicit_residual"])
    return o_gmres(op, b, steps=cfg.gmres_steps, tol=cfg.tol)


def test_gmres_cycle_parity_c5(ctx):
    cfg = CONFIGS["c5"]
    op = build_operator(cfg)
    b = make_rhs_tt(cfg, op.n_xi)
    ref = _c5_reference(op, b, cfg)
    res = ttk.gmres_cycle(gpu_op(op, ctx), ttk.TT.from_cores(*b), steps=cfg.gmres_steps, tol=cfg.tol)
    assert res["steps"] == ref["steps"]
    h, hr = res["history"], ref["history"]
    assert np.max(np.abs(h - hr)) <= 1e-8 * hr[0], (h, hr)
    assert res["explicit"] == pytest.approx(ref["explicit"], rel=1e-6, abs=1e-8 * hr[0])
    print("c5 GMRES ms/step:", np.round(res["step_ms"], 2).tolist())


# ----------------------------------------------------------------------------- optional grouping
@pytest.mark.parametrize("name", ["c2", "c3"])
def test_apply_round_grouped_space(name, ctx):
    """SURVEY 8d optional exact factor grouping (tk_op_group_space): the KL terms nu_l L with
    nu_l = nu_0 2^-l are bitwise proportional, so the space core is produced as Y1' E; the
    rounded result must meet the same parity bars as the literal path."""
    cfg = CONFIGS[name]
    op = build_operator(cfg)
    x = make_input_tt(cfg, op.n_xi)
    g = gpu_op(op, ctx)
    G = g.group_space(True)
    assert G == 3 if name == "c2" else G == 4  # time-mass, Oseen, KL group (+ c3's wind term)
    y = otT.apply_op(op, x)
    check_round(y, cfg.tol, cfg.rmax, ctx, dense=False,
                gpu=lambda: ttk.tt_apply_round(g, ttk.TT.from_cores(*x), cfg.tol, cfg.rmax,
                                               want_info=True))


def test_apply_round_grouped_random(ctx):
    """Constructed proportional terms (K_2 = 0.5 K_0, K_3 = -0.25 K_1) on a random operator."""
    from synth.operator import KronSumOp, Term
    rng = np.random.default_rng(21)
    base = random_operator(rng, 70, 4, 9, 2, density=0.1, max_band=1)
    t0, t1 = base.terms
    terms = [t0, t1,
             Term("p0", 0, 0, rng.standard_normal((1, 9)), rng.standard_normal((4, 4)), t0.K * 0.5),
             Term("p1", 1, 0, rng.standard_normal((2, 9)), rng.standard_normal((4, 4)), t1.K * -0.25)]
    op = KronSumOp(70, 4, 9, terms)
    x = random_tt(rng, 70, 4, 9, 3, 2)
    g = gpu_op(op, ctx)
    assert g.group_space(True) == 2
    y = otT.apply_op(op, x)
    check_round(y, 1e-8, 0, ctx, dense=True,
                gpu=lambda: ttk.tt_apply_round(g, ttk.TT.from_cores(*x), 1e-8, 0, want_info=True))
