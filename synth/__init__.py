"""Seeded synthetic inputs shared by the CUDA path, the oracle and the bench.

This module holds NO arithmetic of the BBMM method (no kernel evaluation, no
solves, no preconditioning): it only draws the problem instances (X, y, theta)
the paper's exact-GP experiments run on, shaped like BASELINE.json's configs.
The paper's workloads are UCI datasets, which are not
shipped; the recipe below gives data
of the same shape and hyperparameters in the regime where an fp32 GPU path and
an fp64 oracle can be compared (SURVEY.md §8c "regime A").

Probe signs are NOT drawn here: both sides implement the same counter-based
splitmix64 generator.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

RBF = 0
MATERN52 = 1


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    kind: int          # RBF / MATERN52
    n: int
    d: int
    t: int             # probes
    k: int             # pivoted-Cholesky rank
    p: int             # max mBCG iterations
    ard: bool
    stored: bool       # default K-mode of the config (stored K vs on-the-fly)
    x_dist: str        # "normal" or "uniform01"
    c_ell: float       # lengthscale = c_ell * sqrt(d)  (C0: lengthscale = c_ell)
    noise_var: float   # sigma^2
    outputscale: float = 1.0


# BASELINE.json "configs" (C0..C4); p = 20 everywhere.
CONFIGS = {
    "C0": Config("C0", RBF, 256, 1, 10, 5, 20, False, False, "uniform01", 0.1, 0.1),
    "C1": Config("C1", RBF, 3338, 19, 10, 5, 20, False, True, "normal", 2.0, 0.3),
    "C2": Config("C2", MATERN52, 45730, 9, 16, 20, 20, True, True, "normal", 2.0, 0.3),
    "C3": Config("C3", RBF, 200_000, 26, 32, 50, 20, True, False, "normal", 2.0, 0.3),
    "C4": Config("C4", RBF, 1_000_000, 3, 16, 100, 20, False, False, "normal", 2.0, 0.3),
}


def scaled(cfg: Config, n: int) -> Config:
    """Same recipe at a different n (parity tests at oracle-friendly sizes)."""
    return dataclasses.replace(cfg, n=int(n))


@dataclasses.dataclass
class Problem:
    cfg: Config
    X: np.ndarray          # (n, d) float32, row-major
    y: np.ndarray          # (n,) float32
    log_ls: np.ndarray     # (1,) or (d,) float64
    log_s: float
    log_noise: float       # sigma = exp(log_noise), sigma^2 = exp(2 log_noise)

    @property
    def n(self):
        return self.X.shape[0]

    @property
    def d(self):
        return self.X.shape[1]


def make_problem(cfg: Config, seed: int = 0) -> Problem:
    """Draw X, y and theta for `cfg` (seeded, deterministic).

    X ~ N(0,1)^d (C0: U[0,1], the 1-D setting of the paper's theory,
    PAPER.md:1179); y = standardise(sum_{r<64} sin(w_r.x + b_r)) + N(0, sigma^2)
    with w_r ~ N(0, diag(1/l^2)); theta: s = 1, sigma^2 and l = c_ell*sqrt(d)
    (ARD: l_q = c_ell*sqrt(d)*exp(u_q), u_q ~ U[-1/2, 1/2]).
    """
    rng = np.random.default_rng(seed)
    n, d = cfg.n, cfg.d
    if cfg.x_dist == "uniform01":
        X = rng.random((n, d))
    else:
        X = rng.standard_normal((n, d))
    X = X.astype(np.float32)

    base = cfg.c_ell if cfg.name == "C0" else cfg.c_ell * math.sqrt(d)
    if cfg.ard:
        u = np.random.default_rng(seed + 2).uniform(-0.5, 0.5, size=d)
        ls = base * np.exp(u)
    else:
        ls = np.array([base])
    log_ls = np.log(ls).astype(np.float64)

    rr = np.random.default_rng(seed + 1)
    w = rr.standard_normal((64, d)) / (ls if cfg.ard else ls[0])
    b = rr.uniform(0.0, 2.0 * math.pi, size=64)
    f = np.zeros(n)
    chunk = 1 << 16
    for i0 in range(0, n, chunk):
        f[i0:i0 + chunk] = np.sin(X[i0:i0 + chunk].astype(np.float64) @ w.T + b).sum(1)
    f = (f - f.mean()) / (f.std() + 1e-300)
    y = f + math.sqrt(cfg.noise_var) * rr.standard_normal(n)
    y = y.astype(np.float32)
    return Problem(cfg, X, y, log_ls, math.log(cfg.outputscale), 0.5 * math.log(cfg.noise_var))


def test_points(cfg: Config, ns: int, seed: int = 7) -> np.ndarray:
    """ns x d float32 test inputs x* from the same distribution as X (predictions, row f1)."""
    rng = np.random.default_rng(seed)
    Xs = rng.random((ns, cfg.d)) if cfg.x_dist == "uniform01" else rng.standard_normal((ns, cfg.d))
    return Xs.astype(np.float32)


def random_block(n: int, c: int, seed: int) -> np.ndarray:
    """A dense n x c float32 block [N(0,1) | Rademacher] used as a matmul RHS."""
    rng = np.random.default_rng(seed)
    M = np.empty((n, c), np.float32)
    M[:, 0] = rng.standard_normal(n)
    if c > 1:
        M[:, 1:] = rng.choice(np.array([-1.0, 1.0], np.float32), size=(n, c - 1))
    return M
