"""ctypes binding of the fp64 CPU oracle (oracle/bbmm_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / `--impl reference` legs, never by the product
package paper_1809_11165_b200/.  Argument marshalling only -- all arithmetic
lives in bbmm_oracle.c, which cites the paper passage each step follows.

Layouts: row-major numpy arrays; X is float32 (the same values the GPU path
reads, upcast to fp64 inside), every other array fp64.  The pivoted-Cholesky
factor L is n x k row-major here (the CUDA path's own layout is its business).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bbmm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

RBF = 0
MATERN52 = 1

OK, ERR_ARG, ERR_NUMERIC = 0, 2, 4


class OracleError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain gcc, fp64, -ffp-contract=off, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-D_GNU_SOURCE", "-ffp-contract=off", "-fopenmp",
               "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_LIB)
        _declare(_lib)
    return _lib


_d = C.c_double
_i = C.c_int
_i64 = C.c_int64
_u64 = C.c_uint64
_p = C.c_void_p


def _declare(L):
    L.orc_kernel.restype = _d
    L.orc_kernel.argtypes = [_i, _i, _p, _p, _i, _p, _d]
    L.orc_kernel_grad.restype = None
    L.orc_kernel_grad.argtypes = [_i, _i, _p, _p, _i, _p, _d, _p]
    L.orc_kernel_matmul.restype = None
    L.orc_kernel_matmul.argtypes = [_i, _p, _i64, _i, _i, _p, _d, _d, _p, _i, _p, _i64, _p]
    L.orc_dkernel_matmul.restype = None
    L.orc_dkernel_matmul.argtypes = [_i, _p, _i64, _i, _i, _p, _d, _p, _i, _p, _i64, _p]
    L.orc_pivchol_dense.restype = _i
    L.orc_pivchol_dense.argtypes = [_p, _i64, _i, _p, _p, _p, _p]
    L.orc_pivchol_kernel.restype = _i
    L.orc_pivchol_kernel.argtypes = [_i, _p, _i64, _i, _i, _p, _d, _i, _p, _p, _p, _p]
    L.orc_precond_setup.restype = _i
    L.orc_precond_setup.argtypes = [_p, _i64, _i, _i, _d, _p, _p]
    L.orc_precond_solve.restype = None
    L.orc_precond_solve.argtypes = [_p, _i64, _i, _i, _d, _p, _p, _i, _p]
    L.orc_splitmix64_mix.restype = _u64
    L.orc_splitmix64_mix.argtypes = [_u64]
    L.orc_rademacher.restype = None
    L.orc_rademacher.argtypes = [_u64, _i64, _i, _i, _p]
    L.orc_probes.restype = None
    L.orc_probes.argtypes = [_p, _i64, _i, _i, _p, _i, _i, _d, _p]
    L.orc_mbcg_dense.restype = _i
    L.orc_mbcg_dense.argtypes = [_p, _i64, _p, _i, _d, _p, _i, _i, _d, _p, _p, _p, _p, _p, _p, _p]
    L.orc_mbcg_kernel.restype = _i
    L.orc_mbcg_kernel.argtypes = [_i, _p, _i64, _i, _i, _p, _d, _d, _p, _i, _p, _i, _i, _d,
                                  _p, _p, _p, _p, _p, _p, _p]
    L.orc_tridiag_from_cg.restype = None
    L.orc_tridiag_from_cg.argtypes = [_i, _p, _p, _i, _p, _p]
    L.orc_tridiag_eig.restype = _i
    L.orc_tridiag_eig.argtypes = [_i, _p, _p, _p, _p]
    L.orc_slq_logdet.restype = _i
    L.orc_slq_logdet.argtypes = [_i, _i, _i, _i, _p, _p, _p, _p, _p, _p]
    L.orc_mll_and_grad.restype = _i
    L.orc_mll_and_grad.argtypes = [_i, _p, _p, _i64, _i, _i, _p, _d, _d, _i, _i, _i, _d, _u64,
                                   _p, _p, _p, _p, _p, _p, _p, _p, _p]
    L.orc_num_threads.restype = _i
    L.orc_predict.argtypes = [_i, _p, _p, _i64, _i, _p, _i64, _i, _p, _d, _d, _i, _i, _d, _p, _p]
    L.orc_predict.restype = _i
    L.orc_predict_cov.argtypes = [_i, _p, _p, _i64, _i, _p, _i64, _i, _p, _d, _d, _i, _i, _d, _p, _p]
    L.orc_predict_cov.restype = _i
    L.orc_train_adam.argtypes = [_i, _p, _p, _i64, _i, _i, _p, _i, _i, _i, _d, _u64, _i, _d, _d,
                                 _d, _d, _p, _p]
    L.orc_train_adam.restype = _i
    L.orc_sor_matmul.argtypes = [_i, _p, _i64, _i, _p, _i64, _i, _p, _d, _d, _p, _i, _i, _p]
    L.orc_sor_matmul.restype = _i
    L.orc_pivchol_sor.argtypes = [_i, _p, _i64, _i, _p, _i64, _i, _p, _d, _i, _p, _p, _p, _p]
    L.orc_pivchol_sor.restype = _i
    L.orc_mbcg_sor.argtypes = [_i, _p, _i64, _i, _p, _i64, _i, _p, _d, _d, _p, _i, _p, _i, _i, _d,
                               _p, _p, _p, _p, _p, _p, _p]
    L.orc_mbcg_sor.restype = _i
    L.orc_num_threads.argtypes = []


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _check(st, what):
    if st != OK:
        raise OracleError(f"{what}: status {st}")


def num_threads() -> int:
    return lib().orc_num_threads()


# ---------------------------------------------------------------- kernels
def kernel(kind, xi, xj, log_ls, log_s):
    xi, xj = _f64(xi), _f64(xj)
    ls = np.exp(_f64(np.atleast_1d(log_ls)))
    return lib().orc_kernel(kind, xi.size, _ptr(xi), _ptr(xj), ls.size, _ptr(ls), float(np.exp(log_s)))


def kernel_grad(kind, xa, xb, log_ls, log_s):
    xa, xb = _f64(xa), _f64(xb)
    ls = np.exp(_f64(np.atleast_1d(log_ls)))
    out = np.zeros(ls.size + 1)
    lib().orc_kernel_grad(kind, xa.size, _ptr(xa), _ptr(xb), ls.size, _ptr(ls),
                          float(np.exp(log_s)), _ptr(out))
    return out


def kernel_matmul(kind, X, log_ls, log_s, log_noise, M, rows=None):
    """(K_XX + sigma^2 I)[rows, :] @ M in fp64 (matrix-free)."""
    X = _f32(X)
    n, d = X.shape
    M = _f64(M).reshape(n, -1)
    c = M.shape[1]
    lls = _f64(np.atleast_1d(log_ls))
    r = None if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
    nr = n if r is None else r.size
    out = np.zeros((nr, c))
    lib().orc_kernel_matmul(kind, _ptr(X), n, d, lls.size, _ptr(lls), float(log_s), float(log_noise),
                            _ptr(M), c, _ptr(r), nr, _ptr(out))
    return out


def dkernel_matmul(kind, X, log_ls, log_s, M, rows=None):
    """[dK/dlog l_q . M]_q and dK/dlog s . M -> (n_ls + 1, nrows, c)."""
    X = _f32(X)
    n, d = X.shape
    M = _f64(M).reshape(n, -1)
    c = M.shape[1]
    lls = _f64(np.atleast_1d(log_ls))
    r = None if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
    nr = n if r is None else r.size
    out = np.zeros((lls.size + 1, nr, c))
    lib().orc_dkernel_matmul(kind, _ptr(X), n, d, lls.size, _ptr(lls), float(log_s), _ptr(M), c,
                             _ptr(r), nr, _ptr(out))
    return out


# ----------------------------------------------------- pivoted Cholesky
def pivchol_dense(K, k):
    K = _f64(K)
    n = K.shape[0]
    L = np.zeros((n, max(k, 1)))
    piv = np.full(max(k, 1), -1, np.int64)
    ku = C.c_int(0)
    res = C.c_double(0)
    _check(lib().orc_pivchol_dense(_ptr(K), n, k, _ptr(L), _ptr(piv), C.byref(ku), C.byref(res)),
           "pivchol_dense")
    return L[:, :k], piv[:k], ku.value, res.value


def pivchol_kernel(kind, X, log_ls, log_s, k):
    X = _f32(X)
    n, d = X.shape
    lls = _f64(np.atleast_1d(log_ls))
    L = np.zeros((n, max(k, 1)))
    piv = np.full(max(k, 1), -1, np.int64)
    ku = C.c_int(0)
    res = C.c_double(0)
    _check(lib().orc_pivchol_kernel(kind, _ptr(X), n, d, lls.size, _ptr(lls), float(log_s), k,
                                    _ptr(L), _ptr(piv), C.byref(ku), C.byref(res)),
           "pivchol_kernel")
    return L[:, :k], piv[:k], ku.value, res.value


# ------------------------------------------------------ preconditioner
def precond_setup(L, noise_var):
    """Cholesky of C = sigma^2 I + L^T L and log|L L^T + sigma^2 I|."""
    L = _f64(L)
    n, k = L.shape
    ch = np.zeros((max(k, 1), max(k, 1)))
    ld = C.c_double(0)
    _check(lib().orc_precond_setup(_ptr(L), n, max(k, 1), k, float(noise_var), _ptr(ch),
                                   C.byref(ld)), "precond_setup")
    return ch[:k, :k], ld.value


def precond_solve(L, noise_var, R):
    L = _f64(L)
    n, k = L.shape
    ch, _ = precond_setup(L, noise_var)
    ch = _f64(ch) if k > 0 else np.zeros((1, 1))
    R = _f64(R).reshape(n, -1)
    Z = np.zeros_like(R)
    lib().orc_precond_solve(_ptr(L), n, max(k, 1), k, float(noise_var), _ptr(ch), _ptr(R),
                            R.shape[1], _ptr(Z))
    return Z


# -------------------------------------------------------------- probes
def splitmix64_mix(z: int) -> int:
    return lib().orc_splitmix64_mix(z & 0xFFFFFFFFFFFFFFFF)


def rademacher(seed, n, k, t):
    eps = np.zeros((n + k, t), np.int8)
    lib().orc_rademacher(seed & 0xFFFFFFFFFFFFFFFF, n, k, t, _ptr(eps))
    return eps


def probes(eps, L, sigma):
    L = _f64(L)
    n, k = L.shape
    eps = np.ascontiguousarray(eps, dtype=np.int8)
    t = eps.shape[1]
    Z = np.zeros((n, t))
    lib().orc_probes(_ptr(eps), n, k, t, _ptr(L) if k > 0 else _ptr(np.zeros(1)), max(k, 1), k,
                     float(sigma), _ptr(Z))
    return Z


# ---------------------------------------------------------------- mBCG
def _mbcg_out(n, c, p):
    return (np.zeros((n, c)), np.zeros((p, c)), np.zeros((p, c)), np.zeros(c, np.int32),
            np.zeros(c), np.zeros(c), np.zeros((p, c)))


def mbcg_dense(A, B, p, tol=0.0, L=None, noise_var=1.0):
    """mBCG on an explicit SPD matrix A; L=None means no preconditioner."""
    A = _f64(A)
    n = A.shape[0]
    B = _f64(B).reshape(n, -1)
    c = B.shape[1]
    k = 0 if L is None else L.shape[1]
    Lp = np.zeros((n, 1)) if L is None else _f64(L)
    U, al, be, it, rr, r0, rh = _mbcg_out(n, c, p)
    _check(lib().orc_mbcg_dense(_ptr(A), n, _ptr(Lp), k, float(noise_var), _ptr(B), c, p, float(tol),
                                _ptr(U), _ptr(al), _ptr(be), _ptr(it), _ptr(rr), _ptr(r0), _ptr(rh)),
           "mbcg_dense")
    return dict(U=U, alpha=al, beta=be, iters=it, relres=rr, rho0=r0, relres_hist=rh)


def mbcg_kernel(kind, X, log_ls, log_s, log_noise, B, p, tol=0.0, L=None):
    X = _f32(X)
    n, d = X.shape
    B = _f64(B).reshape(n, -1)
    c = B.shape[1]
    lls = _f64(np.atleast_1d(log_ls))
    k = 0 if L is None else L.shape[1]
    Lp = np.zeros((n, 1)) if L is None else _f64(L)
    U, al, be, it, rr, r0, rh = _mbcg_out(n, c, p)
    _check(lib().orc_mbcg_kernel(kind, _ptr(X), n, d, lls.size, _ptr(lls), float(log_s),
                                 float(log_noise), _ptr(Lp), k, _ptr(B), c, p, float(tol), _ptr(U),
                                 _ptr(al), _ptr(be), _ptr(it), _ptr(rr), _ptr(r0), _ptr(rh)),
           "mbcg_kernel")
    return dict(U=U, alpha=al, beta=be, iters=it, relres=rr, rho0=r0, relres_hist=rh)


def tridiag_from_cg(alpha, beta):
    alpha, beta = _f64(alpha), _f64(beta)
    m = alpha.size
    dg, of = np.zeros(m), np.zeros(max(m - 1, 1))
    lib().orc_tridiag_from_cg(m, _ptr(alpha), _ptr(np.append(beta, 0.0)), 1, _ptr(dg), _ptr(of))
    return dg, of[:m - 1]


def tridiag_eig(diag, off):
    diag = _f64(diag)
    m = diag.size
    off = _f64(np.append(off, 0.0))
    ev, v0 = np.zeros(m), np.zeros(m)
    _check(lib().orc_tridiag_eig(m, _ptr(diag), _ptr(off), _ptr(ev), _ptr(v0)), "tridiag_eig")
    return ev, v0


def slq_logdet(res, col0=1):
    """SLQ estimate of log|P^{-1} Khat| from an mbcg_* result dict."""
    al, be = _f64(res["alpha"]), _f64(res["beta"])
    p, c = al.shape
    t = c - col0
    it = np.ascontiguousarray(res["iters"], dtype=np.int32)
    om = _f64(res["rho0"])
    out = C.c_double(0)
    per = np.zeros(t)
    _check(lib().orc_slq_logdet(p, c, col0, t, _ptr(it), _ptr(al), _ptr(be), _ptr(om), C.byref(out),
                                _ptr(per)), "slq_logdet")
    return out.value, per


# ------------------------------------------------------- MLL + gradient
STAT_KEYS = ("logdet_precond", "logdet_ratio", "quad_y", "resid_trace", "k_used", "iters",
             "logdet", "omega_sum")


def mll_and_grad(kind, X, y, log_ls, log_s, log_noise, t, k, p, tol=0.0, seed=1, eps=None):
    """One-call exact-GP MLL + gradient (the oracle of bbmm_mll_and_grad)."""
    X = _f32(X)
    n, d = X.shape
    y = _f32(y)
    lls = _f64(np.atleast_1d(log_ls))
    c = t + 1
    mll = C.c_double(0)
    grad = np.zeros(lls.size + 2)
    stats = np.zeros(8)
    U = np.zeros((n, c))
    piv = np.full(max(k, 1), -1, np.int64)
    al, be = np.zeros((p, c)), np.zeros((p, c))
    it = np.zeros(c, np.int32)
    e = None if eps is None else np.ascontiguousarray(eps, dtype=np.int8)
    _check(lib().orc_mll_and_grad(kind, _ptr(X), _ptr(y), n, d, lls.size, _ptr(lls), float(log_s),
                                  float(log_noise), t, k, p, float(tol), seed & 0xFFFFFFFFFFFFFFFF,
                                  _ptr(e), C.byref(mll), _ptr(grad), _ptr(stats), _ptr(U),
                                  _ptr(piv), _ptr(al), _ptr(be), _ptr(it)), "mll_and_grad")
    out = dict(mll=mll.value, grad=grad, U=U, pivots=piv[:k], alpha=al, beta=be, iters=it)
    out.update({kk: stats[i] for i, kk in enumerate(STAT_KEYS)})
    return out


# ------------------------------------------------------------ predictions
def predict(kind, X, y, Xstar, log_ls, log_s, log_noise, k, p, tol=0.0):
    """Predictive mean and pointwise latent variance, Eq. 1: one mBCG call on
    [y | k_{X x*}] with the rank-k pivoted-Cholesky preconditioner (the oracle of bbmm_predict)."""
    X = _f32(X)
    n, d = X.shape
    y = _f32(y)
    Xs = _f32(np.asarray(Xstar).reshape(-1, d))
    ns = Xs.shape[0]
    lls = _f64(np.atleast_1d(log_ls))
    mean, var = np.zeros(ns), np.zeros(ns)
    _check(lib().orc_predict(kind, _ptr(X), _ptr(y), n, d, _ptr(Xs), ns, lls.size, _ptr(lls),
                             float(log_s), float(log_noise), k, p, float(tol), _ptr(mean),
                             _ptr(var)), "predict")
    return mean, var


def predict_cov(kind, X, y, Xstar, log_ls, log_s, log_noise, k, p, tol=0.0):
    """Predictive mean and the full latent covariance between the test points (Eq. 1,
    PAPER.md:617-620; the oracle of bbmm_predict_cov).  Returns (mean (ns,), cov (ns, ns))."""
    X = _f32(X)
    n, d = X.shape
    y = _f32(y)
    Xs = _f32(np.asarray(Xstar).reshape(-1, d))
    ns = Xs.shape[0]
    lls = _f64(np.atleast_1d(log_ls))
    mean, cov = np.zeros(ns), np.zeros((ns, ns))
    _check(lib().orc_predict_cov(kind, _ptr(X), _ptr(y), n, d, _ptr(Xs), ns, lls.size, _ptr(lls),
                                 float(log_s), float(log_noise), k, p, float(tol), _ptr(mean),
                                 _ptr(cov)), "predict_cov")
    return mean, cov


# ------------------------------------------------------------ training
def train_adam(kind, X, y, log_ls, log_s, log_noise, t, k, p, steps, lr=0.1, b1=0.9, b2=0.999,
               eps=1e-8, tol=0.0, seed=1):
    """Adam on theta = (log l.., log s, log sigma) with the BBMM gradient (reading R26).
    Returns (theta_final, trace) with trace rows [mll(theta_s), theta_s...]."""
    X = _f32(X)
    n, d = X.shape
    y = _f32(y)
    th0 = _f64(np.concatenate([np.atleast_1d(log_ls), [log_s, log_noise]]))
    nls = th0.size - 2
    out = np.zeros_like(th0)
    trace = np.zeros((max(steps, 1), 1 + th0.size))
    _check(lib().orc_train_adam(kind, _ptr(X), _ptr(y), n, d, nls, _ptr(th0), t, k, p, float(tol),
                                int(seed) & (2**64 - 1), steps, float(lr), float(b1), float(b2),
                                float(eps), _ptr(out), _ptr(trace)), "train_adam")
    return out, trace[:steps]


# ------------------------------------------------------- SoR operator (row f4)
def sor_matmul(kind, X, Xu, log_ls, log_s, log_noise, M, with_noise=True):
    """K_SoR M (+ sigma^2 M): K_SoR = K_XU (K_UU + 1e-6 s I)^{-1} K_UX (reading R28)."""
    X, Xu = _f32(X), _f32(Xu)
    n, d = X.shape
    m = Xu.shape[0]
    M = _f64(M).reshape(n, -1)
    c = M.shape[1]
    lls = _f64(np.atleast_1d(log_ls))
    out = np.zeros((n, c))
    _check(lib().orc_sor_matmul(kind, _ptr(X), n, d, _ptr(Xu), m, lls.size, _ptr(lls), float(log_s),
                                float(log_noise), _ptr(M), c, int(with_noise), _ptr(out)),
           "sor_matmul")
    return out


def pivchol_sor(kind, X, Xu, log_ls, log_s, k):
    X, Xu = _f32(X), _f32(Xu)
    n, d = X.shape
    lls = _f64(np.atleast_1d(log_ls))
    L = np.zeros((n, max(k, 1)))
    piv = np.full(max(k, 1), -1, np.int64)
    ku, res = C.c_int(0), C.c_double(0)
    _check(lib().orc_pivchol_sor(kind, _ptr(X), n, d, _ptr(Xu), Xu.shape[0], lls.size, _ptr(lls),
                                 float(log_s), k, _ptr(L), _ptr(piv), C.byref(ku), C.byref(res)),
           "pivchol_sor")
    return L[:, :k], piv[:k], ku.value, res.value


def mbcg_sor(kind, X, Xu, log_ls, log_s, log_noise, B, p, tol=0.0, L=None):
    X, Xu = _f32(X), _f32(Xu)
    n, d = X.shape
    B = _f64(B).reshape(n, -1)
    c = B.shape[1]
    lls = _f64(np.atleast_1d(log_ls))
    k = 0 if L is None else L.shape[1]
    Lp = np.zeros((n, 1)) if L is None else _f64(L)
    U, al, be, it, rr, r0, rh = _mbcg_out(n, c, p)
    _check(lib().orc_mbcg_sor(kind, _ptr(X), n, d, _ptr(Xu), Xu.shape[0], lls.size, _ptr(lls),
                              float(log_s), float(log_noise), _ptr(Lp), k, _ptr(B), c, p, float(tol),
                              _ptr(U), _ptr(al), _ptr(be), _ptr(it), _ptr(rr), _ptr(r0), _ptr(rh)),
           "mbcg_sor")
    return dict(U=U, alpha=al, beta=be, iters=it, relres=rr, rho0=r0, relres_hist=rh)
