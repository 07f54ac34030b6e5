"""Oracle pins: the SoR / SGPR operator through mBCG (row f4; App. B).
K_SoR = K_XU (K_UU + 1e-6 s I)^{-1} K_UX (reading R28), Khat_SoR = K_SoR + sigma^2 I.
Pinned to dense numpy formulas on the textbook kernel matrices, to the m = n limit,
to the dense pivoted-Cholesky routine on the materialised matrix and to a dense solve."""
import math

import numpy as np
import pytest

from tests import dense_ref as ref


def data(n=60, m=9, d=2, seed=0):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d)).astype(np.float32)
    Xu = rng.standard_normal((m, d)).astype(np.float32)
    return X, Xu, rng


def dense_sor(kind, X, Xu, log_ls, log_s):
    Kxu = ref.kernel_matrix(kind, X.astype(np.float64), Xu.astype(np.float64), log_ls, log_s)
    Kuu = ref.kernel_matrix(kind, Xu.astype(np.float64), Xu.astype(np.float64), log_ls, log_s)
    Kuu = Kuu + 1e-6 * math.exp(log_s) * np.eye(len(Xu))
    return Kxu @ np.linalg.solve(Kuu, Kxu.T)


@pytest.mark.parametrize("kind,log_ls", [(ref.RBF, math.log(1.3)), (ref.MATERN52, math.log(0.9)),
                                         (ref.RBF, np.log([0.7, 2.0]))])
def test_matmul_matches_dense(orc, kind, log_ls):
    X, Xu, rng = data()
    M = rng.standard_normal((60, 4))
    out = orc.sor_matmul(kind, X, Xu, log_ls, 0.3, math.log(0.4), M)
    K = dense_sor(kind, X, Xu, log_ls, 0.3)
    np.testing.assert_allclose(out, K @ M + 0.16 * M, rtol=0, atol=1e-9 * np.abs(K @ M).max())
    out0 = orc.sor_matmul(kind, X, Xu, log_ls, 0.3, math.log(0.4), M, with_noise=False)
    np.testing.assert_allclose(out0, K @ M, rtol=0, atol=1e-9 * np.abs(K @ M).max())


def test_all_points_inducing_recovers_exact_kernel(orc):
    # U = X: K_SoR = K (K + jI)^{-1} K = K - j K (K + jI)^{-1}, within j = 1e-6 s of K
    X, _, rng = data(n=25)
    M = np.eye(25)
    K_sor = orc.sor_matmul(ref.RBF, X, X, math.log(0.8), 0.0, 0.0, M, with_noise=False)
    K = ref.kernel_matrix(ref.RBF, X.astype(np.float64), X.astype(np.float64), math.log(0.8), 0.0)
    assert np.abs(K_sor - K).max() <= 1.5e-6


def test_pivchol_matches_dense_routine(orc):
    # pivoted Cholesky through SoR rows == the dense routine on the materialised K_SoR;
    # k = m reproduces the rank-m matrix
    X, Xu, _ = data()
    K = dense_sor(ref.RBF, X, Xu, math.log(1.1), 0.0)
    L, piv, ku, res = orc.pivchol_sor(ref.RBF, X, Xu, math.log(1.1), 0.0, 6)
    Ld, pivd, kud, resd = orc.pivchol_dense(K, 6)
    np.testing.assert_array_equal(piv, pivd)
    np.testing.assert_allclose(L, Ld, atol=1e-8)
    L9, _, ku9, res9 = orc.pivchol_sor(ref.RBF, X, Xu, math.log(1.1), 0.0, 9)
    assert ku9 == 9 and abs(res9) < 1e-8
    np.testing.assert_allclose(L9 @ L9.T, K, atol=1e-8)


def test_mbcg_exact_solve(orc):
    X, Xu, rng = data(n=40)
    B = rng.standard_normal((40, 3))
    A = dense_sor(ref.RBF, X, Xu, math.log(1.0), 0.0) + 0.09 * np.eye(40)
    L = orc.pivchol_sor(ref.RBF, X, Xu, math.log(1.0), 0.0, 4)[0]
    r = orc.mbcg_sor(ref.RBF, X, Xu, math.log(1.0), 0.0, math.log(0.3), B, 40, tol=1e-13, L=L)
    np.testing.assert_allclose(r["U"], np.linalg.solve(A, B), rtol=0, atol=1e-8)
    # a rank-m operator plus sigma^2 I has at most m + 1 distinct eigenvalues: plain CG is
    # exact after m + 1 = 10 iterations
    r0 = orc.mbcg_sor(ref.RBF, X, Xu, math.log(1.0), 0.0, math.log(0.3), B, 10)
    np.testing.assert_allclose(r0["U"], np.linalg.solve(A, B), rtol=0, atol=1e-7)
