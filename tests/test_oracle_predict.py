"""Oracle pins: predictive mean and pointwise variance, Eq. 1.

The oracle solves [y | k_{X x*}] with one mBCG call; these tests pin it to the
dense Cholesky formulas (library solves on the textbook definition), to the
interpolation limit, to the far-field limit and to linearity in y.
"""
import math

import numpy as np
import pytest

from tests import dense_ref as ref


def dense_predict(kind, X, y, Xs, log_ls, log_s, log_noise):
    """mean = K_{*X} Khat^{-1} y, var = diag(K_{**} - K_{*X} Khat^{-1} K_{X*}) via Cholesky."""
    A = ref.khat(kind, X, log_ls, log_s, log_noise)
    Ks = ref.kernel_matrix(kind, X, Xs, log_ls, log_s)            # n x ns
    Lc = np.linalg.cholesky(A)
    a = np.linalg.solve(Lc.T, np.linalg.solve(Lc, np.asarray(y, np.float64)))
    W = np.linalg.solve(Lc, Ks)
    kss = np.diag(ref.kernel_matrix(kind, Xs, Xs, log_ls, log_s))
    return Ks.T @ a, kss - (W * W).sum(0)


def problem(n=30, ns=7, d=2, seed=0):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d)).astype(np.float32)
    y = np.sin(X.sum(1)).astype(np.float32) + 0.1 * rng.standard_normal(n).astype(np.float32)
    Xs = rng.standard_normal((ns, d)).astype(np.float32)
    return X, y, Xs


@pytest.mark.parametrize("kind,log_ls", [(ref.RBF, math.log(1.2)), (ref.MATERN52, math.log(1.5)),
                                         (ref.RBF, np.log([0.8, 1.7]))])
@pytest.mark.parametrize("k", [0, 5])
def test_matches_dense_cholesky(orc, kind, log_ls, k):
    # p = n and a tiny tol: mBCG is an exact solver (SPEC predict example, n=30, n*=7)
    X, y, Xs = problem()
    m, v = orc.predict(kind, X, y, Xs, log_ls, 0.2, math.log(0.3), k, 30, 1e-13)
    md, vd = dense_predict(kind, X.astype(np.float64), y, Xs.astype(np.float64), log_ls, 0.2,
                           math.log(0.3))
    np.testing.assert_allclose(m, md, rtol=0, atol=1e-9)
    np.testing.assert_allclose(v, vd, rtol=0, atol=1e-9)


def test_interpolation_limit(orc):
    # x* = a training point and sigma^2 -> 0: mean -> its label, variance -> 0 (SPEC predict).
    # k = n makes the preconditioner (nearly) Khat itself, so mBCG converges at once.
    X, y, _ = problem(n=25)
    Xs = X[[3, 11]]
    m, v = orc.predict(ref.RBF, X, y, Xs, math.log(1.0), 0.0, math.log(1e-5), 25, 25, 1e-14)
    np.testing.assert_allclose(m, y[[3, 11]], atol=1e-3)
    assert np.all(np.abs(v) <= 1e-3)


def test_far_field(orc):
    # k_{X x*} = 0 exactly in fp64 far away: mean = 0 (zero prior mean, R19), var = s
    X, y, _ = problem()
    Xs = np.full((2, 2), 1e3, np.float32)
    m, v = orc.predict(ref.RBF, X, y, Xs, math.log(1.0), math.log(2.5), math.log(0.3), 5, 10)
    np.testing.assert_array_equal(m, 0.0)
    np.testing.assert_allclose(v, 2.5, rtol=1e-15)


def test_columns_independent_and_single_point(orc):
    # mBCG columns are independent CG runs: n* = 1 gives the same numbers as within a batch
    X, y, Xs = problem()
    m7, v7 = orc.predict(ref.RBF, X, y, Xs, math.log(1.2), 0.0, math.log(0.3), 5, 12)
    m1, v1 = orc.predict(ref.RBF, X, y, Xs[4:5], math.log(1.2), 0.0, math.log(0.3), 5, 12)
    assert m1[0] == m7[4] and v1[0] == v7[4]


def test_mean_linear_in_y(orc):
    X, y1, Xs = problem(seed=1)
    y2 = np.cos(3 * X[:, 0]).astype(np.float32)
    args = (ref.RBF, X)
    kw = dict(log_ls=math.log(1.1), log_s=0.0, log_noise=math.log(0.4), k=0, p=30, tol=1e-13)
    ma, _ = orc.predict(*args, y1, Xs, **kw)
    mb, _ = orc.predict(*args, y2, Xs, **kw)
    mc, _ = orc.predict(*args, (y1.astype(np.float64) + y2).astype(np.float32), Xs, **kw)
    ysum_err = (y1.astype(np.float64) + y2) - (y1 + y2).astype(np.float32)
    assert np.abs(ysum_err).max() < 1e-6
    np.testing.assert_allclose(mc, ma + mb, atol=1e-6)


def dense_cov(kind, X, Xs, log_ls, log_s, log_noise):
    """K_{**} - K_{*X} Khat^{-1} K_{X*} via Cholesky (the textbook GP posterior covariance)."""
    A = ref.khat(kind, X, log_ls, log_s, log_noise)
    Ks = ref.kernel_matrix(kind, X, Xs, log_ls, log_s)
    W = np.linalg.solve(np.linalg.cholesky(A), Ks)
    return ref.kernel_matrix(kind, Xs, Xs, log_ls, log_s) - W.T @ W


@pytest.mark.parametrize("kind,log_ls", [(ref.RBF, math.log(1.2)), (ref.MATERN52, np.log([0.9, 1.6]))])
@pytest.mark.parametrize("k", [0, 5])
def test_covariance_matches_dense_cholesky(orc, kind, log_ls, k):
    """Full posterior covariance between test points (Eq. 1): the dense Cholesky formula at
    p = n; its diagonal is the pointwise variance and the mean is unchanged."""
    X, y, Xs = problem(ns=9)
    m, C = orc.predict_cov(kind, X, y, Xs, log_ls, 0.2, math.log(0.3), k, 30, 1e-13)
    Cd = dense_cov(kind, X.astype(np.float64), Xs.astype(np.float64), log_ls, 0.2, math.log(0.3))
    np.testing.assert_allclose(C, Cd, rtol=0, atol=1e-9)
    m2, v = orc.predict(kind, X, y, Xs, log_ls, 0.2, math.log(0.3), k, 30, 1e-13)
    np.testing.assert_array_equal(m, m2)
    np.testing.assert_allclose(np.diag(C), v, rtol=0, atol=1e-12)
    assert np.min(np.linalg.eigvalsh(0.5 * (C + C.T))) > -1e-9     # PSD


def test_covariance_of_coincident_points(orc):
    """Two identical test points have covariance equal to their variance; far-apart test points
    (no training data nearby) are uncorrelated."""
    X, y, _ = problem()
    Xs = np.array([[0.3, -0.2], [0.3, -0.2], [1e3, 1e3]], np.float32)
    m, C = orc.predict_cov(ref.RBF, X, y, Xs, math.log(1.0), 0.0, math.log(0.2), 5, 30, 1e-13)
    assert C[0, 1] == pytest.approx(C[0, 0], rel=1e-12)
    assert C[0, 2] == pytest.approx(0.0, abs=1e-12)
    assert C[2, 2] == pytest.approx(1.0, rel=1e-12)
