"""Oracle pins: mBCG (Alg. S2), Lanczos recovery,
tridiagonal eigensolve and SLQ (Eq. 5-6)."""
import json
import math
import os

import numpy as np
import pytest

from tests import dense_ref as ref

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def spd(n, seed, cond=50.0):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    w = np.geomspace(1.0, cond, n)
    return (Q * w) @ Q.T


def kernel_problem(n=40, seed=0, s2=0.05):
    rng = np.random.default_rng(seed)
    X = rng.random((n, 2))
    K = ref.kernel_matrix(ref.RBF, X, X, math.log(0.3), 0.0)
    return K, K + s2 * np.eye(n), s2, rng


def test_identity_operator_golden(orc):
    g = json.load(open(os.path.join(GOLD, "closed_forms.json")))["mbcg_identity"]
    n = g["n"]
    B = np.random.default_rng(0).standard_normal((n, 3))
    r = orc.mbcg_dense(np.eye(n), B, p=5, tol=1e-12)
    np.testing.assert_allclose(r["U"], B, atol=1e-15)
    assert list(r["iters"]) == [1, 1, 1]
    np.testing.assert_allclose(r["alpha"][0], g["alpha0"])
    dg, of = orc.tridiag_from_cg(r["alpha"][:1, 1], r["beta"][:0, 1])
    np.testing.assert_allclose(np.diag(dg), g["T"])


def test_scalar_operator(orc):
    n, c_ = 9, 3.5
    B = np.random.default_rng(1).choice([-1.0, 1.0], size=(n, 4))
    r = orc.mbcg_dense(c_ * np.eye(n), B, p=3, tol=1e-12)
    np.testing.assert_allclose(r["U"], B / c_, rtol=1e-15)
    assert r["alpha"][0, 0] == pytest.approx(1 / c_)
    ld, per = orc.slq_logdet(r)
    assert ld == pytest.approx(n * math.log(c_), rel=1e-14)


def test_diagonal_exact_in_n_steps(orc):
    A = np.diag(np.arange(1.0, 6.0))
    r = orc.mbcg_dense(A, np.ones((5, 1)), p=5)
    np.testing.assert_allclose(r["U"][:, 0], 1 / np.arange(1.0, 6.0), rtol=1e-12)


@pytest.mark.parametrize("precond", [False, True])
def test_p_equals_n_gives_dense_solve(orc, precond):
    K, A, s2, rng = kernel_problem(30, 1, s2=0.3)
    B = rng.standard_normal((30, 5))
    L = orc.pivchol_dense(K, 5)[0] if precond else None
    r = orc.mbcg_dense(A, B, p=30, L=L, noise_var=s2)
    np.testing.assert_allclose(r["U"], np.linalg.solve(A, B), rtol=1e-7, atol=1e-8)


def test_columns_are_independent_pcg_runs(orc):
    K, A, s2, rng = kernel_problem(35, 2)
    L = orc.pivchol_dense(K, 4)[0]
    B = rng.standard_normal((35, 5))
    r = orc.mbcg_dense(A, B, p=12, L=L, noise_var=s2)
    for col in range(5):
        r1 = orc.mbcg_dense(A, B[:, col:col + 1], p=12, L=L, noise_var=s2)
        np.testing.assert_array_equal(r["U"][:, col], r1["U"][:, 0])
        np.testing.assert_array_equal(r["alpha"][:, col], r1["alpha"][:, 0])
    # the y-solve does not depend on probe content
    B2 = B.copy()
    B2[:, 1:] = rng.standard_normal((35, 4))
    np.testing.assert_array_equal(orc.mbcg_dense(A, B2, p=12, L=L, noise_var=s2)["U"][:, 0],
                                  r["U"][:, 0])


@pytest.mark.parametrize("precond", [False, True])
def test_tridiagonal_equals_explicit_lanczos(orc, precond):
    """T from CG coefficients == Lanczos on P^{-1/2} Khat P^{-1/2} from P^{-1/2} b."""
    K, A, s2, rng = kernel_problem(40, 3)
    k = 5 if precond else 0
    L = orc.pivchol_dense(K, k)[0] if precond else None
    P = (L @ L.T + s2 * np.eye(40)) if precond else np.eye(40)
    b = rng.choice([-1.0, 1.0], size=(40, 1))
    m = 8
    r = orc.mbcg_dense(A, b, p=m, L=L, noise_var=s2)
    dg, of = orc.tridiag_from_cg(r["alpha"][:m, 0], r["beta"][:m - 1, 0])
    Pm = ref.sym_sqrt_inv(P)
    la, lb = ref.lanczos_full_reorth(Pm @ A @ Pm, Pm @ b[:, 0], m)
    np.testing.assert_allclose(dg, la, rtol=1e-9)
    np.testing.assert_allclose(np.abs(of), np.abs(lb), rtol=1e-8)


def test_ritz_values_inside_spectrum_and_exact_at_p_n(orc):
    K, A, s2, rng = kernel_problem(24, 4, s2=0.2)
    L = orc.pivchol_dense(K, 3)[0]
    P = L @ L.T + s2 * np.eye(24)
    lam = np.linalg.eigvals(np.linalg.solve(P, A)).real
    b = rng.choice([-1.0, 1.0], size=(24, 1))
    for m in (3, 8):
        r = orc.mbcg_dense(A, b, p=m, L=L, noise_var=s2)
        ev, _ = orc.tridiag_eig(*orc.tridiag_from_cg(r["alpha"][:m, 0], r["beta"][:m - 1, 0]))
        assert ev.min() >= lam.min() * (1 - 1e-9) and ev.max() <= lam.max() * (1 + 1e-9)
    # lambda(P^-1 Khat) >= 1 since Khat - P = K - LL^T is PSD
    assert lam.min() > 1 - 1e-9


def test_cg_error_bound(orc):
    """Obs. S2: ||u*-u_p||_A <= 2 ((sqrt k - 1)/(sqrt k + 1))^p ||u*||_A."""
    A = spd(40, 5, cond=200.0)
    b = np.random.default_rng(5).standard_normal((40, 1))
    us = np.linalg.solve(A, b[:, 0])
    kap = np.linalg.cond(A)
    rate = (math.sqrt(kap) - 1) / (math.sqrt(kap) + 1)
    anorm = lambda v: math.sqrt(v @ A @ v)
    for p in (1, 5, 10, 20, 30):
        u = orc.mbcg_dense(A, b, p=p)["U"][:, 0]
        assert anorm(us - u) <= 2 * rate**p * anorm(us) * (1 + 1e-9)


def test_tridiag_eig_golden_and_random(orc):
    g = json.load(open(os.path.join(GOLD, "closed_forms.json")))["tridiag_2x2"]
    ev, v0 = orc.tridiag_eig(g["diag"], g["off"])
    np.testing.assert_allclose(ev, g["evals"], rtol=1e-14)
    np.testing.assert_allclose(np.abs(v0), g["abs_v0"], rtol=1e-14)
    ev, v0 = orc.tridiag_eig([2.5], [])
    assert list(ev) == [2.5] and list(np.abs(v0)) == [1.0]
    rng = np.random.default_rng(6)
    for m in (5, 12, 20):
        dg, of = rng.uniform(1, 3, m), rng.uniform(-1, 1, m - 1)
        T = np.diag(dg) + np.diag(of, 1) + np.diag(of, -1)
        w, V = np.linalg.eigh(T)
        ev, v0 = orc.tridiag_eig(dg, of)
        np.testing.assert_allclose(ev, w, rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(np.abs(v0), np.abs(V[0]), rtol=1e-8, atol=1e-10)


@pytest.mark.parametrize("precond", [False, True])
def test_slq_exact_per_probe_at_p_n(orc, precond):
    """At p = n, omega e1^T log(T) e1 = w^T log(P^-1/2 Khat P^-1/2) w, w = P^-1/2 z exactly."""
    n = 20
    K, A, s2, rng = kernel_problem(n, 7, s2=0.3)
    L = orc.pivchol_dense(K, 3)[0] if precond else None
    P = (L @ L.T + s2 * np.eye(n)) if precond else np.eye(n)
    Z = rng.choice([-1.0, 1.0], size=(n, 3))
    r = orc.mbcg_dense(A, Z, p=n, L=L, noise_var=s2)
    _, per = orc.slq_logdet(r, col0=0)
    Pm = ref.sym_sqrt_inv(P)
    w_, V_ = np.linalg.eigh(Pm @ A @ Pm)
    logA = (V_ * np.log(w_)) @ V_.T
    for i in range(3):
        w = Pm @ Z[:, i]
        assert per[i] == pytest.approx(w @ logA @ w, rel=1e-9)
    np.testing.assert_allclose(r["rho0"], np.einsum("ij,ij->j", Z, np.linalg.solve(P, Z)), rtol=1e-12)


def test_slq_unbiased_over_reseeds(orc):
    """Mean over reseeded preconditioned probes -> log|P^-1 Khat| (Thm 2 / Eq. 6, reading R12)."""
    n = 30
    K, A, s2, _ = kernel_problem(n, 8, s2=0.1)
    L = orc.pivchol_dense(K, 3)[0]
    P = L @ L.T + s2 * np.eye(n)
    exact = np.linalg.slogdet(A)[1] - np.linalg.slogdet(P)[1]
    t = 400
    eps = orc.rademacher(9, n, 3, t)
    Z = orc.probes(eps, L, math.sqrt(s2))
    r = orc.mbcg_dense(A, Z, p=n, L=L, noise_var=s2)
    ld, per = orc.slq_logdet(r, col0=0)
    se = per.std(ddof=1) / math.sqrt(t)
    assert abs(ld - exact) < 3.5 * se


# ------------------------------------------------ residual history (row f3)
def test_relres_history_is_true_residual(orc):
    # entry j = ||B - A U_(j+1)|| / ||B|| with U_(j+1) from an independent run stopped after
    # j + 1 iterations (the recurrence residual equals the true residual up to rounding)
    K, A, s2, rng = kernel_problem(n=40, seed=3)
    B = rng.standard_normal((40, 3))
    L = np.linalg.cholesky(K + 1e-9 * np.eye(40))[:, :4]
    full = orc.mbcg_dense(A, B, 12, L=L, noise_var=s2)
    for j in range(12):
        Uj = orc.mbcg_dense(A, B, j + 1, L=L, noise_var=s2)["U"]
        true = np.linalg.norm(B - A @ Uj, axis=0) / np.linalg.norm(B, axis=0)
        np.testing.assert_allclose(full["relres_hist"][j], true, rtol=1e-8, atol=1e-14)


def test_relres_history_frozen_columns_zero(orc):
    K, A, s2, rng = kernel_problem(n=30, seed=4)
    B = rng.standard_normal((30, 2))
    r = orc.mbcg_dense(A, B, 30, tol=1e-6)
    for col in range(2):
        it = r["iters"][col]
        assert it < 30 and r["relres_hist"][it - 1, col] < 1e-6
        assert np.all(r["relres_hist"][it:, col] == 0.0)


def test_preconditioning_lowers_residual(orc):
    # the paper's claim for pivoted-Cholesky preconditioning of smooth kernels:
    # at a fixed iteration the rank-k preconditioned residual is far below the plain one
    rng = np.random.default_rng(5)
    X = rng.random((200, 1))
    K = ref.kernel_matrix(ref.RBF, X, X, math.log(0.2), 0.0)
    A = K + 0.01 * np.eye(200)
    B = rng.standard_normal((200, 1))
    L, piv, ku, _ = orc.pivchol_dense(K, 12)
    plain = orc.mbcg_dense(A, B, 10)["relres_hist"][:, 0]
    pre = orc.mbcg_dense(A, B, 10, L=L[:, :ku], noise_var=0.01)["relres_hist"][:, 0]
    assert pre[9] < 1e-2 * plain[9], (pre[9], plain[9])
