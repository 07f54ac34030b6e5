"""Oracle pins: pivoted Cholesky (App. B)."""
import json
import os

import numpy as np
import pytest

from tests import dense_ref as ref

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def brute_force_pivchol(K, k):
    """App. B written with explicit permutation matrices:
    permute the max-diagonal entry of the Schur complement to the top-left,
    peel q = [k11; b]/sqrt(k11), recurse on S = K22 - b b^T / k11, and map
    every q back through the accumulated permutations Q_i."""
    n = K.shape[0]
    S = K.copy()
    perm = np.arange(n)            # perm[pos] = original index at position pos
    L = np.zeros((n, k))
    pivots = []
    for m in range(k):
        sub = S[m:, m:]
        jrel = int(np.argmax(np.diag(sub)))   # first maximum = lowest position
        j = m + jrel
        Pm = np.eye(n)                         # permutation pi_m swapping m <-> j
        Pm[[m, j]] = Pm[[j, m]]
        S = Pm @ S @ Pm
        perm[[m, j]] = perm[[j, m]]              # Q_m bookkeeping
        k11 = S[m, m]
        q = np.zeros(n)
        q[m:] = S[m:, m] / np.sqrt(k11)
        S = S - np.outer(q, q)
        L[perm, m] = q                         # back to original row order
        pivots.append(int(perm[m]))
    return L, pivots


def test_golden_diag_3_1_2(orc):
    g = json.load(open(os.path.join(GOLD, "closed_forms.json")))["pivchol_diag_3_1_2"]
    L, piv, ku, res = orc.pivchol_dense(np.array(g["K"], float), g["k"])
    assert list(piv) == g["pivots"]
    np.testing.assert_allclose(L @ L.T, np.array(g["LLt"], float), atol=1e-15)
    assert res == pytest.approx(g["resid_trace"])
    assert ku == 2


def test_rank_one_exact(orc):
    v = np.array([1.0, -2.0, 0.5, 3.0])
    L, piv, ku, res = orc.pivchol_dense(np.outer(v, v), 3)
    assert ku == 1          # numerical rank reached: early stop (reading R23)
    np.testing.assert_allclose(L[:, :1] @ L[:, :1].T, np.outer(v, v), atol=1e-12)
    assert abs(res) < 1e-12
    assert list(piv[1:]) == [-1, -1]


@pytest.mark.parametrize("k", [1, 3, 6])
def test_matches_brute_force_with_permutation_matrices(orc, k):
    rng = np.random.default_rng(0)
    X = rng.random((9, 1))
    K = ref.kernel_matrix(ref.RBF, X, X, np.log(0.4), 0.0)
    L, piv, ku, res = orc.pivchol_dense(K, k)
    Lb, pb = brute_force_pivchol(K, k)
    assert list(piv) == pb
    np.testing.assert_allclose(L, Lb, atol=1e-10)
    assert res == pytest.approx(np.trace(K - L @ L.T), abs=1e-10)


def test_schur_psd_monotone_and_full_rank_exact(orc):
    rng = np.random.default_rng(1)
    X = rng.standard_normal((40, 2))
    K = ref.kernel_matrix(ref.MATERN52, X, X, np.log(0.8), 0.0)
    prev = np.inf
    for k in range(0, 41, 4):
        L, piv, ku, res = orc.pivchol_dense(K, k)
        E = K - L @ L.T
        assert np.linalg.eigvalsh(E).min() > -1e-10      # E = K - LL^T PSD
        assert res <= prev + 1e-12                         # residual trace non-increasing
        assert len(set(int(p) for p in piv[:ku])) == ku    # distinct pivots
        prev = res
    L, piv, ku, res = orc.pivchol_dense(K, 40)
    np.testing.assert_allclose(L @ L.T, K, atol=1e-9)


@pytest.mark.parametrize("kind", [0, 1])
def test_kernel_pivchol_equals_dense_pivchol(orc, kind):
    rng = np.random.default_rng(2)
    X = rng.standard_normal((60, 3)).astype(np.float32)
    lls, ls_ = np.array([0.3, 0.5, 0.1]), 0.2
    L, piv, ku, res = orc.pivchol_kernel(kind, X, lls, ls_, 12)
    K = ref.kernel_matrix(kind, X.astype(np.float64), X.astype(np.float64), lls, ls_)
    Ld, pd, kd, rd = orc.pivchol_dense(K, 12)
    assert list(piv) == list(pd)
    np.testing.assert_allclose(L, Ld, atol=1e-10)
    assert res == pytest.approx(rd, rel=1e-9)
