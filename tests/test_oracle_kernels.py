"""Oracle pins: kernel values, derivatives and the blackbox matmul (CPU only)."""
import json
import math
import os

import numpy as np
import pytest

from tests import dense_ref as ref

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_rbf_golden_sqrt2(orc):
    g = json.load(open(os.path.join(GOLD, "closed_forms.json")))["rbf_unit_sqrt2"]
    v = orc.kernel(orc.RBF, g["x"], g["x2"], g["log_ls"], g["log_s"])
    assert v == pytest.approx(g["value"], rel=1e-15)


@pytest.mark.parametrize("kind", [0, 1])
def test_kernel_at_zero_distance_is_outputscale(orc, kind):
    x = np.array([0.3, -1.2, 2.0])
    assert orc.kernel(kind, x, x, [0.4], math.log(2.5)) == pytest.approx(2.5, rel=1e-15)


def test_matern52_matches_bessel_definition(orc):
    rng = np.random.default_rng(0)
    for _ in range(20):
        x, x2 = rng.standard_normal(3), rng.standard_normal(3)
        lls = rng.uniform(-1, 1, 3)
        v = orc.kernel(orc.MATERN52, x, x2, lls, 0.3)
        r = ref.scaled_r(x[None], x2[None], lls)[0, 0]
        assert v == pytest.approx(math.exp(0.3) * ref.matern_bessel(np.array([r]))[0], rel=1e-12)


@pytest.mark.parametrize("kind", [0, 1])
def test_ard_equal_lengthscales_equals_isotropic(orc, kind):
    rng = np.random.default_rng(1)
    x, x2 = rng.standard_normal(4), rng.standard_normal(4)
    a = orc.kernel(kind, x, x2, [0.7] * 4, 0.0)
    b = orc.kernel(kind, x, x2, [0.7], 0.0)
    assert a == pytest.approx(b, rel=1e-15)
    # lengthscale per dimension really is per dimension: scaling coordinates
    lls = np.array([0.1, -0.3, 0.5, 0.0])
    c1 = orc.kernel(kind, x, x2, lls, 0.0)
    c2 = orc.kernel(kind, x / np.exp(lls), x2 / np.exp(lls), [0.0], 0.0)
    assert c1 == pytest.approx(c2, rel=1e-13)


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("ard", [False, True])
def test_kernel_grad_matches_finite_differences(orc, kind, ard):
    rng = np.random.default_rng(2)
    d = 3
    x, x2 = rng.standard_normal(d), rng.standard_normal(d)
    lls = rng.uniform(-0.5, 0.5, d) if ard else np.array([0.2])
    ls_ = 0.4
    g = orc.kernel_grad(kind, x, x2, lls, ls_)
    h = 1e-6
    for q in range(lls.size):
        lp, lm = lls.copy(), lls.copy()
        lp[q] += h
        lm[q] -= h
        fd = (orc.kernel(kind, x, x2, lp, ls_) - orc.kernel(kind, x, x2, lm, ls_)) / (2 * h)
        assert g[q] == pytest.approx(fd, rel=1e-6, abs=1e-10)
    fd = (orc.kernel(kind, x, x2, lls, ls_ + h) - orc.kernel(kind, x, x2, lls, ls_ - h)) / (2 * h)
    assert g[-1] == pytest.approx(fd, rel=1e-6)


@pytest.mark.parametrize("kind", [0, 1])
def test_kernel_matmul_matches_dense_library_product(orc, kind):
    rng = np.random.default_rng(3)
    n, d, c = 57, 3, 5
    X = rng.standard_normal((n, d)).astype(np.float32)
    M = rng.standard_normal((n, c))
    lls, ls_, ln = np.array([0.1, 0.3, -0.2]), 0.2, -0.6
    out = orc.kernel_matmul(kind, X, lls, ls_, ln, M)
    A = ref.khat(kind, X.astype(np.float64), lls, ls_, ln)
    np.testing.assert_allclose(out, A @ M, rtol=1e-12, atol=1e-12)
    rows = np.array([5, 0, 56, 17])
    np.testing.assert_array_equal(orc.kernel_matmul(kind, X, lls, ls_, ln, M, rows=rows), out[rows])


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("ard", [False, True])
def test_dkernel_matmul_matches_fd_of_kernel_matrix(orc, kind, ard):
    rng = np.random.default_rng(4)
    n, d, c = 23, 2, 3
    X = rng.standard_normal((n, d)).astype(np.float32)
    M = rng.standard_normal((n, c))
    lls = np.array([0.1, -0.2]) if ard else np.array([0.15])
    ls_ = -0.1
    out = orc.dkernel_matmul(kind, X, lls, ls_, M)
    Xd = X.astype(np.float64)
    h = 1e-6
    for q in range(lls.size):
        lp, lm = lls.copy(), lls.copy()
        lp[q] += h
        lm[q] -= h
        dK = (ref.kernel_matrix(kind, Xd, Xd, lp, ls_) - ref.kernel_matrix(kind, Xd, Xd, lm, ls_)) / (2 * h)
        np.testing.assert_allclose(out[q], dK @ M, rtol=1e-6, atol=1e-8)
    np.testing.assert_allclose(out[-1], ref.kernel_matrix(kind, Xd, Xd, lls, ls_) @ M, rtol=1e-12)
