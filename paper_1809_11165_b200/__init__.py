"""Python binding of libbbmm.so -- the B200-native BBMM mBCG hot path.

Thin ctypes marshalling over the C-ABI declared in include/bbmm.h (same
function names without the ``bbmm_`` prefix).  Every step of the method runs
inside the CUDA library; this module only checks tensor placement / dtype,
passes device pointers and the current CUDA stream, and wraps results.

PyTorch is used for device memory, streams and (multi-GPU) the process group
that distributes the NCCL unique id.  There is NO fallback: if the compiled
library is missing or fails to load, importing this package raises.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libbbmm.so")

RBF = 0
MATERN52 = 1
ONTHEFLY = 0
STORED = 1
FP64ACC = 0     # matmul precision: fp64 D, fp64 products and sums (FFMA/DFMA path)
FP32ACC = 1     # fp32 D, 16-term fp32 chunks folded into fp64 (regime A only)
INT8EXACT = 2   # default: tcgen05 int8 tensor cores, exact integer contraction (else FP64ACC)
INT8EXACT31 = 3  # INT8EXACT with the on-the-fly RBF kernel values forced to the 31-bit grid
INT8EXACT23 = 4  # INT8EXACT with the on-the-fly RBF kernel values forced to the 23-bit grid

_STATUS = {0: "OK", 2: "ERR_ARG", 3: "ERR_DATA", 4: "ERR_NUMERIC", 5: "ERR_CUDA",
           6: "ERR_NCCL", 7: "ERR_OOM"}


class BBMMError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} not found: the CUDA library is not built (run __graft_entry__.build()); "
        "there is no CPU fallback")
_lib = C.CDLL(LIB_PATH)


class _Hyper(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_ls", C.c_int32), ("log_ls_h", C.POINTER(C.c_double)),
                ("log_outputscale", C.c_double), ("log_noise", C.c_double)]


class Stats(C.Structure):
    _fields_ = [("iters", C.c_int32), ("k_used", C.c_int32), ("logdet_precond", C.c_double),
                ("logdet_ratio", C.c_double), ("logdet", C.c_double), ("quad_y", C.c_double),
                ("resid_trace", C.c_double), ("relres_y", C.c_double), ("ms_total", C.c_double),
                ("ms_pivchol", C.c_double), ("ms_mbcg", C.c_double), ("ms_matmul", C.c_double),
                ("ms_slq", C.c_double), ("ms_deriv", C.c_double),
                ("matmul_launches", C.c_int32), ("gpu_launches", C.c_int32),
                ("matmul_path", C.c_int32), ("unconverged", C.c_int32),
                ("relres_max", C.c_double), ("ms_comm", C.c_double), ("kgrid_bits", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_p, _i32, _i64, _d, _u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_uint64
_HP = C.POINTER(_Hyper)

_lib.bbmm_version.restype = C.c_char_p
_lib.bbmm_last_error.restype = C.c_char_p
_lib.bbmm_last_error.argtypes = [_p]
_lib.bbmm_ctx_create.argtypes = [C.c_int, _p, C.POINTER(_p)]
_lib.bbmm_ctx_destroy.argtypes = [_p]
_lib.bbmm_nccl_unique_id.argtypes = [_p]
_lib.bbmm_ctx_set_comm.argtypes = [_p, C.c_int, C.c_int, _p]
_lib.bbmm_ctx_set_matmul_precision.argtypes = [_p, C.c_int]
_lib.bbmm_local_rows.argtypes = [_p, _i64, C.POINTER(_i64), C.POINTER(_i64)]
_lib.bbmm_kernel_matmul.argtypes = [_p, _p, _i64, _i32, _HP, C.c_int, _p, _i32, _i64, _p, _i64]
_lib.bbmm_pivchol.argtypes = [_p, _p, _i64, _i32, _HP, _i32, _p, _p, C.POINTER(_i32),
                              C.POINTER(_d)]
_lib.bbmm_mbcg.argtypes = [_p, _p, _i64, _i32, _HP, C.c_int, _p, _i32, _p, _i32, _i64, _i32, _d,
                           _p, _i64, _p, _p, _p, _p, _p, _p]
_lib.bbmm_mll_and_grad.argtypes = [_p, _p, _p, _i64, _i32, _HP, C.c_int, _i32, _i32, _i32, _d,
                                   _u64, _p, C.POINTER(_d), _p, C.POINTER(Stats), _p, _p]
_lib.bbmm_predict.argtypes = [_p, _p, _p, _i64, _i32, _p, _i64, _HP, C.c_int, _i32, _i32, _d, _p, _p]
_lib.bbmm_predict_cov.argtypes = [_p, _p, _p, _i64, _i32, _p, _i64, _HP, C.c_int, _i32, _i32, _d,
                                  _p, _p]
_lib.bbmm_train_adam.argtypes = [_p, _p, _p, _i64, _i32, _HP, C.c_int, _i32, _i32, _i32, _d, _u64,
                                 _i32, _d, _d, _d, _d, _p, _p]
_lib.bbmm_sor_mbcg.argtypes = [_p, _p, _i64, _i32, _p, _i32, _HP, _i32, _p, _i32, _i64, _i32, _d,
                               _p, _i64, _p, _p, _p, _p]
_lib.bbmm_local_group_create.argtypes = [_i32, C.POINTER(_p)]
_lib.bbmm_local_group_destroy.argtypes = [_p]
_lib.bbmm_ctx_set_local_comm.argtypes = [_p, _p, _i32]
for _f in ("bbmm_local_group_create", "bbmm_local_group_destroy", "bbmm_ctx_set_local_comm",
           "bbmm_ctx_create", "bbmm_ctx_destroy", "bbmm_nccl_unique_id", "bbmm_ctx_set_comm",
           "bbmm_local_rows", "bbmm_ctx_set_matmul_precision", "bbmm_kernel_matmul", "bbmm_pivchol", "bbmm_mbcg",
           "bbmm_mll_and_grad", "bbmm_predict", "bbmm_predict_cov", "bbmm_train_adam",
           "bbmm_sor_mbcg"):
    getattr(_lib, _f).restype = C.c_int


def row_partition(n: int, nranks: int, rank: int):
    """Rows [r0, r1) owned by `rank` (mirrors bbmm_local_rows): blocks of
    nb = ceil(ceil(n / nranks) / 128) * 128 rows, so rank boundaries align with
    the 128-point j-tiles of the tensor-core operand and the all-gathers."""
    nb = -(-(-(-n // nranks)) // 128) * 128
    r0 = min(n, rank * nb)
    return r0, min(n, r0 + nb), nb


def version() -> str:
    return _lib.bbmm_version().decode()


@dataclasses.dataclass
class Hyper:
    """theta = (log lengthscale(s), log outputscale, log noise std); kind RBF/MATERN52."""
    kind: int
    log_ls: np.ndarray
    log_s: float
    log_noise: float

    def _c(self):
        ls = np.ascontiguousarray(np.atleast_1d(self.log_ls), dtype=np.float64)
        h = _Hyper(int(self.kind), ls.size, ls.ctypes.data_as(C.POINTER(C.c_double)),
                   float(self.log_s), float(self.log_noise))
        h._keep = ls
        return h


def _torch():
    import torch
    return torch


class Context:
    """A library context bound to a CUDA device and stream (default: current)."""

    def __init__(self, device=None, stream=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise BBMMError(5, "no CUDA device available (the library has no CPU path)")
        dev = torch.cuda.current_device() if device is None else int(device)
        self.device = dev
        self._stream = stream if stream is not None else torch.cuda.current_stream(dev)
        h = _p()
        self._check_raw(_lib.bbmm_ctx_create(dev, _p(self._stream.cuda_stream), C.byref(h)),
                        "ctx_create")
        self._h = h
        self.nranks, self.rank = 1, 0

    def _check_raw(self, st, what):
        if st != 0:
            msg = _lib.bbmm_last_error(self._h).decode() if getattr(self, "_h", None) else what
            raise BBMMError(st, msg)

    def check(self, st):
        if st != 0:
            raise BBMMError(st, _lib.bbmm_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            _lib.bbmm_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self):
        return self._stream

    def set_comm(self, group=None):
        """Create the NCCL communicator over torch.distributed's world (or `group`).  Without an
        initialised process group: a 1-rank communicator (every collective is still issued)."""
        torch = _torch()
        import torch.distributed as dist
        if group is None and not dist.is_initialized():
            buf = (C.c_char * 128)()
            self.check(_lib.bbmm_nccl_unique_id(C.cast(buf, _p)))
            self.check(_lib.bbmm_ctx_set_comm(self._h, 1, 0, C.cast(buf, _p)))
            self.nranks, self.rank = 1, 0
            return self
        ws, rk = dist.get_world_size(group), dist.get_rank(group)
        buf = (C.c_char * 128)()
        if rk == 0:
            self.check(_lib.bbmm_nccl_unique_id(C.cast(buf, _p)))
        obj = [bytes(buf)]
        dist.broadcast_object_list(obj, src=0, group=group)
        raw = (C.c_char * 128).from_buffer_copy(obj[0])
        self.check(_lib.bbmm_ctx_set_comm(self._h, ws, rk, C.cast(raw, _p)))
        self.nranks, self.rank = ws, rk
        return self

    def set_local_comm(self, group: "LocalGroup", rank: int):
        """Join an in-process rank group (bbmm_ctx_set_local_comm): this context becomes
        rank `rank`; drive each rank's calls from its own thread."""
        self.check(_lib.bbmm_ctx_set_local_comm(self._h, group._h, int(rank)))
        self.nranks, self.rank = group.nranks, int(rank)
        return self

    def set_matmul_precision(self, prec: int):
        self.check(_lib.bbmm_ctx_set_matmul_precision(self._h, int(prec)))
        return self

    def local_rows(self, n):
        r0, r1 = _i64(), _i64()
        self.check(_lib.bbmm_local_rows(self._h, int(n), C.byref(r0), C.byref(r1)))
        return r0.value, r1.value


class LocalGroup:
    """In-process rank group (include/bbmm.h bbmm_local_group_create): the row-partitioned
    multi-rank path with host-staged collectives, e.g. several contexts on one GPU."""

    def __init__(self, nranks: int):
        h = _p()
        st = _lib.bbmm_local_group_create(int(nranks), C.byref(h))
        if st != 0:
            raise BBMMError(st, "local_group_create")
        self._h, self.nranks = h, int(nranks)

    def close(self):
        if getattr(self, "_h", None):
            _lib.bbmm_local_group_destroy(self._h)
            self._h = None


def _dev(t, dtype, name, ctx):
    torch = _torch()
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor on cuda:{ctx.device}")
    if t.device.type != "cuda" or t.device.index != ctx.device:
        raise ValueError(f"{name} must live on cuda:{ctx.device}")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return _p(t.data_ptr())


def _shape(t, shape, name):
    """Sizes the C-ABI cannot check (it receives raw pointers): a wrong-sized array would make
    the kernels read or write past the end of a device buffer.  None in `shape` = any size."""
    got = tuple(t.shape)
    if len(got) != len(shape) or any(w is not None and g != w for g, w in zip(got, shape)):
        want = "x".join("*" if w is None else str(w) for w in shape)
        raise ValueError(f"{name} must be {want}, got {'x'.join(map(str, got)) or 'scalar'}")


def _X_shape(X, name="X"):
    if X.dim() != 2:
        raise ValueError(f"{name} must be n x d, got {tuple(X.shape)}")
    return X.shape


def kernel_matmul(ctx: Context, X, D, hyper: Hyper, kmode: int = ONTHEFLY):
    """V = (K(X,X) + sigma^2 I)[local rows] @ D.  X: n x d fp32, D: n x c fp64."""
    torch = _torch()
    n, d = _X_shape(X)
    _shape(D, (n, None), "D")
    c = D.shape[1]
    r0, r1 = ctx.local_rows(n)
    V = torch.empty((r1 - r0, c), dtype=torch.float64, device=X.device)
    hp = hyper._c()
    ctx.check(_lib.bbmm_kernel_matmul(ctx._h, _dev(X, torch.float32, "X", ctx), n, d,
                                      C.byref(hp), kmode, _dev(D, torch.float64, "D", ctx), c, c,
                                      _p(V.data_ptr()), c))
    return V


def pivchol(ctx: Context, X, hyper: Hyper, k: int):
    """Rank-k pivoted Cholesky of K_XX: (L [k x n fp64], pivots, k_used, resid_trace)."""
    torch = _torch()
    n, d = _X_shape(X)
    L = torch.zeros((max(k, 1), n), dtype=torch.float64, device=X.device)
    piv = np.full(max(k, 1), -1, np.int64)
    ku, res = _i32(), _d()
    hp = hyper._c()
    ctx.check(_lib.bbmm_pivchol(ctx._h, _dev(X, torch.float32, "X", ctx), n, d, C.byref(hp), k,
                                _p(L.data_ptr()), piv.ctypes.data_as(_p), C.byref(ku),
                                C.byref(res)))
    return L[:k], piv[:k], ku.value, res.value


def mbcg(ctx: Context, X, hyper: Hyper, B, L=None, max_iter: int = 20, tol: float = 0.0,
         kmode: int = ONTHEFLY):
    """mBCG (Alg. S2) on Khat with preconditioner L L^T + sigma^2 I (L: k x n) or none."""
    torch = _torch()
    n, d = _X_shape(X)
    r0, r1 = ctx.local_rows(n)
    _shape(B, (r1 - r0, None), "B (local rows x ncols)")
    nl, c = B.shape
    k = 0 if L is None else int(L.shape[0])
    if L is not None:
        _shape(L, (k, n), "L")
    U = torch.empty_like(B)
    al = np.zeros((max_iter, c))
    be = np.zeros((max_iter, c))
    it = np.zeros(c, np.int32)
    rr = np.zeros(c)
    r0 = np.zeros(c)
    rh = np.zeros((max_iter, c))
    hp = hyper._c()
    Lp = _dev(L, torch.float64, "L", ctx) if k > 0 else None
    ctx.check(_lib.bbmm_mbcg(ctx._h, _dev(X, torch.float32, "X", ctx), n, d, C.byref(hp), kmode,
                             Lp, k, _dev(B, torch.float64, "B", ctx), c, c, max_iter, float(tol),
                             _p(U.data_ptr()), c, al.ctypes.data_as(_p), be.ctypes.data_as(_p),
                             it.ctypes.data_as(_p), rr.ctypes.data_as(_p), r0.ctypes.data_as(_p),
                             rh.ctypes.data_as(_p)))
    return dict(U=U, alpha=al, beta=be, iters=it, relres=rr, rho0=r0, relres_hist=rh)


def mll_and_grad(ctx: Context, X, y, hyper: Hyper, t: int, k: int, max_iter: int = 20,
                 tol: float = 0.0, seed: int = 1, eps=None, kmode: int = ONTHEFLY,
                 return_solves: bool = False):
    """One-call exact-GP marginal log likelihood and gradient (north-star entry)."""
    torch = _torch()
    n, d = _X_shape(X)
    _shape(y, (n,), "y")
    if eps is not None:
        _shape(eps, (n + k, t), "eps")
    nls = int(np.atleast_1d(hyper.log_ls).size)
    mll = _d()
    grad = np.zeros(nls + 2)
    st = Stats()
    piv = np.full(max(k, 1), -1, np.int64)
    U = None
    if return_solves:
        r0, r1 = ctx.local_rows(n)
        U = torch.empty((r1 - r0, t + 1), dtype=torch.float64, device=X.device)
    hp = hyper._c()
    ep = _dev(eps, torch.int8, "eps", ctx) if eps is not None else None
    ctx.check(_lib.bbmm_mll_and_grad(ctx._h, _dev(X, torch.float32, "X", ctx),
                                     _dev(y, torch.float32, "y", ctx), n, d, C.byref(hp), kmode,
                                     t, k, max_iter, float(tol), int(seed) & (2**64 - 1), ep,
                                     C.byref(mll), grad.ctypes.data_as(_p), C.byref(st),
                                     _p(U.data_ptr()) if U is not None else None,
                                     piv.ctypes.data_as(_p)))
    out = dict(mll=mll.value, grad=grad, pivots=piv[:k], stats=st.as_dict())
    if U is not None:
        out["U"] = U
    return out


def predict(ctx: Context, X, y, Xstar, hyper: Hyper, k: int, max_iter: int = 20, tol: float = 0.0,
            kmode: int = ONTHEFLY, variance: bool = True):
    """GP predictive mean and pointwise latent variance, Eq. 1 (bbmm_predict).
    Returns (mean, var) as fp64 cuda tensors of length nstar (var is None if variance=False)."""
    torch = _torch()
    n, d = _X_shape(X)
    _shape(y, (n,), "y")
    _shape(Xstar, (None, d), "Xstar")
    ns = Xstar.shape[0]
    mean = torch.empty(ns, dtype=torch.float64, device=X.device)
    var = torch.empty(ns, dtype=torch.float64, device=X.device) if variance else None
    hp = hyper._c()
    ctx.check(_lib.bbmm_predict(ctx._h, _dev(X, torch.float32, "X", ctx),
                                _dev(y, torch.float32, "y", ctx), n, d,
                                _dev(Xstar, torch.float32, "Xstar", ctx), ns, C.byref(hp), kmode, k,
                                max_iter, float(tol), _p(mean.data_ptr()),
                                _p(var.data_ptr()) if var is not None else None))
    return mean, var


def predict_cov(ctx: Context, X, y, Xstar, hyper: Hyper, k: int, max_iter: int = 20,
                tol: float = 0.0, kmode: int = ONTHEFLY):
    """GP predictive mean and the full latent covariance between the test points, Eq. 1
    (bbmm_predict_cov).  Returns (mean (nstar,), cov (nstar, nstar)) as fp64 cuda tensors."""
    torch = _torch()
    n, d = _X_shape(X)
    _shape(y, (n,), "y")
    _shape(Xstar, (None, d), "Xstar")
    ns = Xstar.shape[0]
    mean = torch.empty(ns, dtype=torch.float64, device=X.device)
    cov = torch.empty((ns, ns), dtype=torch.float64, device=X.device)
    hp = hyper._c()
    ctx.check(_lib.bbmm_predict_cov(ctx._h, _dev(X, torch.float32, "X", ctx),
                                    _dev(y, torch.float32, "y", ctx), n, d,
                                    _dev(Xstar, torch.float32, "Xstar", ctx), ns, C.byref(hp),
                                    kmode, k, max_iter, float(tol), _p(mean.data_ptr()),
                                    _p(cov.data_ptr())))
    return mean, cov


def train_adam(ctx: Context, X, y, hyper: Hyper, t: int, k: int, max_iter: int = 20,
               steps: int = 100, lr: float = 0.1, beta1: float = 0.9, beta2: float = 0.999,
               eps: float = 1e-8, tol: float = 0.0, seed: int = 1, kmode: int = ONTHEFLY):
    """Adam hyperparameter training (bbmm_train_adam).
    Returns (trained Hyper, trace) with trace rows [mll(theta_s), theta_s...]."""
    torch = _torch()
    n, d = _X_shape(X)
    _shape(y, (n,), "y")
    nls = int(np.atleast_1d(hyper.log_ls).size)
    th = np.zeros(nls + 2)
    trace = np.zeros((max(steps, 1), nls + 3))
    hp = hyper._c()
    ctx.check(_lib.bbmm_train_adam(ctx._h, _dev(X, torch.float32, "X", ctx),
                                   _dev(y, torch.float32, "y", ctx), n, d, C.byref(hp), kmode, t, k,
                                   max_iter, float(tol), int(seed) & (2**64 - 1), steps, float(lr),
                                   float(beta1), float(beta2), float(eps), th.ctypes.data_as(_p),
                                   trace.ctypes.data_as(_p)))
    return Hyper(hyper.kind, th[:nls], th[nls], th[nls + 1]), trace[:steps]


def sor_mbcg(ctx: Context, X, Xu, hyper: Hyper, B, k: int = 0, max_iter: int = 20,
             tol: float = 0.0):
    """mBCG on the SoR / SGPR operator K_XU (K_UU + 1e-6 s I)^{-1} K_UX + sigma^2 I with a
    rank-k pivoted-Cholesky preconditioner of K_SoR (bbmm_sor_mbcg)."""
    torch = _torch()
    n, d = _X_shape(X)
    _shape(Xu, (None, d), "Xu")
    r0, r1 = ctx.local_rows(n)
    _shape(B, (r1 - r0, None), "B (local rows x ncols)")
    m = Xu.shape[0]
    nl, c = B.shape
    U = torch.empty_like(B)
    piv = np.full(max(k, 1), -1, np.int64)
    it = np.zeros(c, np.int32)
    rr = np.zeros(c)
    rh = np.zeros((max_iter, c))
    hp = hyper._c()
    ctx.check(_lib.bbmm_sor_mbcg(ctx._h, _dev(X, torch.float32, "X", ctx), n, d,
                                 _dev(Xu, torch.float32, "Xu", ctx), m, C.byref(hp), k,
                                 _dev(B, torch.float64, "B", ctx), c, c, max_iter, float(tol),
                                 _p(U.data_ptr()), c, piv.ctypes.data_as(_p), it.ctypes.data_as(_p),
                                 rr.ctypes.data_as(_p), rh.ctypes.data_as(_p)))
    return dict(U=U, pivots=piv[:k], iters=it, relres=rr, relres_hist=rh)
