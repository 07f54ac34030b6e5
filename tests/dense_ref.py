"""Dense library-routine references used to PIN the oracle (tests only).

Each helper is built from library primitives (scipy.spatial.distance.cdist,
scipy.special.kv, numpy.linalg cholesky/solve/slogdet/eigh) applied to the
textbook definitions, so a mistake inside oracle/bbmm_oracle.c (a dropped
term, wrong sign, transposed operand, wrong index) shows up as a mismatch.
"""
from __future__ import annotations

import math

import numpy as np
from scipy.spatial.distance import cdist
from scipy.special import gamma, kv

RBF, MATERN52 = 0, 1


def scaled_r(X1, X2, log_ls):
    ls = np.exp(np.atleast_1d(np.asarray(log_ls, np.float64)))
    X1 = np.asarray(X1, np.float64) / ls
    X2 = np.asarray(X2, np.float64) / ls
    return cdist(X1, X2)          # Euclidean distance in lengthscale units


def matern_bessel(r, nu=2.5):
    """General Matern correlation via the modified Bessel function K_nu."""
    r = np.asarray(r, np.float64)
    out = np.ones_like(r)
    nz = r > 0
    z = math.sqrt(2 * nu) * r[nz]
    out[nz] = (2 ** (1 - nu) / gamma(nu)) * z ** nu * kv(nu, z)
    return out


def kernel_matrix(kind, X1, X2, log_ls, log_s):
    r = scaled_r(X1, X2, log_ls)
    s = math.exp(log_s)
    if kind == RBF:
        return s * np.exp(-0.5 * r * r)
    return s * matern_bessel(r)


def khat(kind, X, log_ls, log_s, log_noise):
    K = kernel_matrix(kind, X, X, log_ls, log_s)
    return K + math.exp(2 * log_noise) * np.eye(X.shape[0])


def dense_mll(kind, X, y, log_ls, log_s, log_noise):
    """Exact log marginal likelihood via Cholesky (the standard closed form)."""
    A = khat(kind, X, log_ls, log_s, log_noise)
    y = np.asarray(y, np.float64)
    Lc = np.linalg.cholesky(A)
    a = np.linalg.solve(Lc.T, np.linalg.solve(Lc, y))
    return -0.5 * (y @ a + 2 * np.log(np.diag(Lc)).sum() + len(y) * math.log(2 * math.pi))


def dense_mll_grad_fd(kind, X, y, log_ls, log_s, log_noise, h=1e-5):
    """Central finite differences of dense_mll over theta = (log_ls.., log_s, log_noise)."""
    th = np.concatenate([np.atleast_1d(log_ls).astype(np.float64), [log_s, log_noise]])
    nl = th.size - 2
    g = np.zeros_like(th)
    for q in range(th.size):
        tp, tm = th.copy(), th.copy()
        tp[q] += h
        tm[q] -= h
        fp = dense_mll(kind, X, y, tp[:nl], tp[nl], tp[nl + 1])
        fm = dense_mll(kind, X, y, tm[:nl], tm[nl], tm[nl + 1])
        g[q] = (fp - fm) / (2 * h)
    return g


def sym_sqrt_inv(P):
    w, Q = np.linalg.eigh(P)
    return (Q / np.sqrt(w)) @ Q.T


def lanczos_full_reorth(A, v, m):
    """Explicit Lanczos with full re-orthogonalisation (two passes)."""
    n = A.shape[0]
    Q = np.zeros((n, m))
    alpha = np.zeros(m)
    beta = np.zeros(max(m - 1, 0))
    q = v / np.linalg.norm(v)
    for j in range(m):
        Q[:, j] = q
        w = A @ q
        alpha[j] = q @ w
        for _ in range(2):
            w = w - Q[:, :j + 1] @ (Q[:, :j + 1].T @ w)
        if j < m - 1:
            beta[j] = np.linalg.norm(w)
            q = w / beta[j]
    return alpha, beta
