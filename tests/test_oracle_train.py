"""Oracle pins: Adam hyperparameter training (row f2; "All methods use the same
optimizer (Adam)", settings by reading R26 = SPEC defaults).

Pinned to the textbook Adam recursion written out in numpy (Kingma & Ba), replayed
on the MLL oracle's own gradients, and to SPEC's descent example against training
with exact dense (Cholesky + finite-difference) gradients."""
import math

import numpy as np

from tests import dense_ref as ref


def gp_data(n=200, seed=0):
    # 1-D data drawn from a known RBF GP: l* = 0.3, s* = 1, sigma^2 = 0.01 (SPEC train example)
    rng = np.random.default_rng(seed)
    X = np.sort(rng.random(n)).reshape(-1, 1)
    K = ref.kernel_matrix(ref.RBF, X, X, math.log(0.3), 0.0) + 1e-8 * np.eye(n)
    f = np.linalg.cholesky(K) @ rng.standard_normal(n)
    y = f + 0.1 * rng.standard_normal(n)
    return X.astype(np.float32), y.astype(np.float32)


TH0 = (math.log(1.0), 0.0, math.log(0.5))       # initial (log l, log s, log sigma)
KW = dict(t=10, k=5, p=20)


def adam_replay(orc, X, y, steps, lr=0.1, b1=0.9, b2=0.999, eps=1e-8, seed=1):
    th = np.array(TH0, np.float64)
    m = np.zeros(3)
    v = np.zeros(3)
    for s in range(steps):
        r = orc.mll_and_grad(ref.RBF, X, y, th[:1], th[1], th[2], seed=seed + s, **KW)
        g = -np.asarray(r["grad"])
        m = b1 * m + (1 - b1) * g
        v = b2 * v + (1 - b2) * g * g
        th = th - lr * (m / (1 - b1 ** (s + 1))) / (np.sqrt(v / (1 - b2 ** (s + 1))) + eps)
    return th


def test_zero_steps_is_identity(orc):
    X, y = gp_data()
    th, tr = orc.train_adam(ref.RBF, X, y, *TH0, steps=0, **KW)
    np.testing.assert_array_equal(th, TH0)
    assert tr.shape[0] == 0


def test_first_step_closed_form(orc):
    # bias-corrected moments equal g and g^2 at step 1: theta_1 = theta_0 - lr g / (|g| + eps)
    X, y = gp_data()
    th, tr = orc.train_adam(ref.RBF, X, y, *TH0, steps=1, **KW)
    r = orc.mll_and_grad(ref.RBF, X, y, TH0[0], TH0[1], TH0[2], seed=1, **KW)
    g = -np.asarray(r["grad"])
    np.testing.assert_allclose(th, np.array(TH0) - 0.1 * g / (np.abs(g) + 1e-8), rtol=0, atol=1e-14)
    assert tr[0, 0] == r["mll"] and np.all(tr[0, 1:] == TH0)


def test_matches_numpy_adam_replay(orc):
    X, y = gp_data()
    th, tr = orc.train_adam(ref.RBF, X, y, *TH0, steps=4, **KW)
    np.testing.assert_allclose(th, adam_replay(orc, X, y, 4), rtol=0, atol=1e-12)


def test_descends_like_exact_dense_training(orc):
    # SPEC: trained nll <= initial nll over 100 steps, and the final nll within 2 % of
    # Adam driven by exact dense gradients (Cholesky MLL, central differences)
    X, y = gp_data()
    X64 = X.astype(np.float64)
    steps = 100
    th, tr = orc.train_adam(ref.RBF, X, y, *TH0, steps=steps, **KW)
    nll0 = -ref.dense_mll(ref.RBF, X64, y, *TH0)
    nll_b = -ref.dense_mll(ref.RBF, X64, y, th[:1], th[1], th[2])
    assert nll_b < nll0
    thd = np.array(TH0, np.float64)
    m = np.zeros(3)
    v = np.zeros(3)
    for s in range(steps):
        g = -ref.dense_mll_grad_fd(ref.RBF, X64, y, thd[:1], thd[1], thd[2])
        m = 0.9 * m + 0.1 * g
        v = 0.999 * v + 0.001 * g * g
        thd = thd - 0.1 * (m / (1 - 0.9 ** (s + 1))) / (np.sqrt(v / (1 - 0.999 ** (s + 1))) + 1e-8)
    nll_d = -ref.dense_mll(ref.RBF, X64, y, thd[:1], thd[1], thd[2])
    assert abs(nll_b - nll_d) <= 0.02 * abs(nll_d), (nll_b, nll_d, th, thd)
