"""Oracle pins: one-call MLL + gradient (Eq. 2, Eq. 4-6)."""
import math

import numpy as np
import pytest

from tests import dense_ref as ref


def test_single_point_closed_form(orc):
    """n = 1, no preconditioner: one CG step is exact and z^2 = 1, so every term is exact."""
    X = np.array([[0.3]], np.float32)
    y = np.array([1.7], np.float32)
    ls_, ln = math.log(1.3), math.log(0.4)
    s, s2 = 1.3, 0.16
    yv = float(y[0])
    r = orc.mll_and_grad(ref.RBF, X, y, [0.0], ls_, ln, t=4, k=0, p=3)
    kh = s + s2
    assert r["mll"] == pytest.approx(-0.5 * (yv * yv / kh + math.log(kh) + math.log(2 * math.pi)),
                                     rel=1e-14)
    # d/dlog l = 0 (r = 0); d/dlog s and d/dlog sigma from the scalar formula
    g = r["grad"]
    assert g[0] == pytest.approx(0.0, abs=1e-15)
    assert g[1] == pytest.approx(0.5 * (yv * yv * s / kh**2 - s / kh), rel=1e-13)
    assert g[2] == pytest.approx(0.5 * (yv * yv * 2 * s2 / kh**2 - 2 * s2 / kh), rel=1e-13)


@pytest.mark.parametrize("kind", [0, 1])
def test_zero_preconditioner_error(orc, kind):
    """k >= numerical rank: P ~= Khat, so one iteration converges, T = [1] and
    log|Khat| = log|P| (SURVEY [X24]); the MLL then equals the dense value."""
    rng = np.random.default_rng(0)
    n = 64
    X = rng.random((n, 1)).astype(np.float32)
    y = rng.standard_normal(n).astype(np.float32)
    lls, ls_, ln = np.log([0.5]), 0.0, 0.5 * math.log(0.1)
    r = orc.mll_and_grad(kind, X, y, lls, ls_, ln, t=6, k=n, p=4, tol=1e-10)
    if kind == 0:
        assert r["k_used"] < n                   # early stop at the numerical rank (R23)
    assert abs(r["logdet_ratio"]) < 1e-6
    assert r["mll"] == pytest.approx(ref.dense_mll(kind, X.astype(float), y, lls, ls_, ln), rel=1e-8)
    assert int(r["iters"]) <= 2


@pytest.mark.parametrize("kind", [0, 1])
def test_exact_solve_at_p_equals_n(orc, kind):
    rng = np.random.default_rng(1)
    n = 25
    X = rng.standard_normal((n, 2)).astype(np.float32)
    y = rng.standard_normal(n).astype(np.float32)
    lls, ls_, ln = np.array([0.2, -0.1]), 0.1, 0.5 * math.log(0.3)
    r = orc.mll_and_grad(kind, X, y, lls, ls_, ln, t=5, k=3, p=n)
    A = ref.khat(kind, X.astype(float), lls, ls_, ln)
    np.testing.assert_allclose(r["U"][:, 0], np.linalg.solve(A, y.astype(float)), rtol=1e-8)
    assert r["quad_y"] == pytest.approx(y.astype(float) @ np.linalg.solve(A, y.astype(float)), rel=1e-9)


@pytest.mark.parametrize("kind,ard", [(0, True), (1, False)])
def test_estimator_unbiased_over_reseeds(orc, kind, ard):
    """Full stochastic estimator (preconditioned probes, omega weights, P^-1 trace
    correction) averaged over reseeds -> dense MLL and its FD gradient (SURVEY [X22])."""
    rng = np.random.default_rng(2)
    n = 40
    X = rng.standard_normal((n, 2)).astype(np.float32)
    y = rng.standard_normal(n).astype(np.float32)
    lls = np.array([0.1, 0.4]) if ard else np.array([0.2])
    ls_, ln = 0.15, 0.5 * math.log(0.2)
    mlls, grads = [], []
    for seed in range(150):
        r = orc.mll_and_grad(kind, X, y, lls, ls_, ln, t=8, k=4, p=n, seed=seed)
        mlls.append(r["mll"])
        grads.append(r["grad"])
    mlls, grads = np.array(mlls), np.array(grads)
    Xd = X.astype(float)
    exact = ref.dense_mll(kind, Xd, y, lls, ls_, ln)
    gexact = ref.dense_mll_grad_fd(kind, Xd, y, lls, ls_, ln)
    se = mlls.std(ddof=1) / math.sqrt(len(mlls))
    assert abs(mlls.mean() - exact) < 4 * se + 1e-9
    gse = grads.std(0, ddof=1) / math.sqrt(len(grads))
    assert np.all(np.abs(grads.mean(0) - gexact) < 4 * gse + 1e-7), (grads.mean(0), gexact, gse)
