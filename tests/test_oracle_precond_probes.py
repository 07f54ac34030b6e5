"""Oracle pins: Woodbury solve, determinant lemma, probe generator (App. B)."""
import json
import math
import os

import numpy as np
import pytest

from tests import dense_ref as ref

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _problem(seed=0, n=30, k=4):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, 2))
    K = ref.kernel_matrix(ref.RBF, X, X, math.log(0.9), 0.0)
    return K, rng


def test_woodbury_equals_dense_solve(orc):
    K, rng = _problem()
    L, piv, ku, _ = orc.pivchol_dense(K, 4)
    s2 = 0.07
    R = rng.standard_normal((K.shape[0], 3))
    Z = orc.precond_solve(L, s2, R)
    P = L @ L.T + s2 * np.eye(K.shape[0])
    np.testing.assert_allclose(Z, np.linalg.solve(P, R), rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(orc.precond_solve(L, s2, P @ R), R, rtol=1e-9, atol=1e-9)


def test_determinant_lemma_equals_slogdet(orc):
    K, _ = _problem(1)
    for k in (1, 4, 9):
        L, *_ = orc.pivchol_dense(K, k)
        s2 = 0.05
        _, ld = orc.precond_setup(L, s2)
        sign, ref_ld = np.linalg.slogdet(L @ L.T + s2 * np.eye(K.shape[0]))
        assert sign > 0
        assert ld == pytest.approx(ref_ld, rel=1e-12, abs=1e-10)


def test_zero_columns_is_scaled_identity(orc):
    n = 7
    L = np.zeros((n, 0))
    R = np.arange(n * 2, dtype=float).reshape(n, 2)
    np.testing.assert_allclose(orc.precond_solve(L, 0.25, R), R / 0.25)
    _, ld = orc.precond_setup(L, 0.25)
    assert ld == pytest.approx(n * math.log(0.25))


def test_splitmix64_published_vectors(orc):
    g = json.load(open(os.path.join(GOLD, "splitmix64.json")))
    G = 0x9E3779B97F4A7C15
    for st in g["streams"]:
        for ctr, want in enumerate(st["outputs"], start=1):
            assert orc.splitmix64_mix((st["seed"] + ctr * G) & (2**64 - 1)) == want


def test_rademacher_layout_and_balance(orc):
    n, k, t, seed = 1000, 7, 5, 11
    eps = orc.rademacher(seed, n, k, t)
    assert set(np.unique(eps)) == {-1, 1}
    assert abs(eps.mean()) < 0.05
    # counter layout: entry (i, col) is draw number col*(n+k) + i + 1 of the stream
    G = 0x9E3779B97F4A7C15
    for i, col in [(0, 0), (999, 4), (1003, 2)]:
        h = orc.splitmix64_mix((seed + (col * (n + k) + i + 1) * G) & (2**64 - 1))
        assert eps[i, col] == (-1 if h >> 63 else 1)


def test_probe_covariance_is_preconditioner(orc):
    """z = L eps1 + sigma eps2 has Cov(z) = L L^T + sigma^2 I (reading R13)."""
    n, k, t = 6, 2, 40000
    rng = np.random.default_rng(3)
    L = rng.standard_normal((n, k))
    sigma = 0.7
    eps = orc.rademacher(5, n, k, t)
    Z = orc.probes(eps, L, sigma)
    np.testing.assert_allclose(Z, L @ eps[n:].astype(float) + sigma * eps[:n], atol=1e-14)
    C = Z @ Z.T / t
    P = L @ L.T + sigma**2 * np.eye(n)
    se = np.sqrt((P**2 + np.outer(np.diag(P), np.diag(P))) / t)   # Gaussian-ish SE bound
    assert np.all(np.abs(C - P) < 5 * se + 1e-3)
