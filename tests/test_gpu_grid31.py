"""GPU parity of the INT8EXACT31 precision (on-the-fly RBF kernel values on a 31-bit grid).

BBMM_MATMUL_INT8EXACT31 keeps the MUFU's fp32 kernel values k~ = 2^S on a 31-bit fixed-point grid
(the 23-bit truncation in three u8 slices plus a residual u8 slice, csrc/k1tc2.cu MODE 3) instead
of INT8EXACT's 23-bit grid, so the only per-entry error left is the MUFU's own.
Checked here: (1) the kernel-matmul against the fp64 oracle at the element-wise bound, over tile
edges and at the full C4 size on sampled rows (many uint32 drain windows); (2) the per-entry
kernel values against the fp64 definition (reading R1): the rms error falls below INT8EXACT's by
the removed grid rounding; (3) MLL + gradient parity at the north-star bars.
"""
import math

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)

import paper_1809_11165_b200 as bb  # noqa: E402

from .test_gpu_parity import colwise_rel, dev, hyper_of, matmul_bound, run_both  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    c = bb.Context(0)
    yield c
    c.close()


def _matmul(ctx, pr, D, prec):
    ctx.set_matmul_precision(prec)
    try:
        return bb.kernel_matmul(ctx, dev(pr.X), dev(D, torch.float64), hyper_of(pr)).cpu().numpy()
    finally:
        ctx.set_matmul_precision(bb.INT8EXACT)


@pytest.mark.parametrize("name,n,c", [("C4", 4099, 17), ("C4", 129, 3), ("C4", 70, 1), ("C3", 3001, 33),
                                      ("C4", 2100, 13), ("C3", 1000, 8)])
def test_grid31_kernel_matmul_matches_oracle(ctx, orc, name, n, c):
    pr = synth.make_problem(synth.scaled(synth.CONFIGS[name], n), seed=3)
    D = synth.random_block(n, c, seed=4).astype(np.float64)
    V = _matmul(ctx, pr, D, bb.INT8EXACT31)
    ref = orc.kernel_matmul(pr.cfg.kind, pr.X, pr.log_ls, pr.log_s, pr.log_noise, D)
    err = np.abs(V - ref)
    bound = matmul_bound(orc, pr, D)
    assert np.all(err <= bound), float((err / bound).max())
    assert colwise_rel(V, ref).max() < 2e-5


def test_grid31_kernel_values_are_finer(ctx):
    """Unit columns D = [e_j1 .. e_jm] expose the kernel values each operator computed (V = s K e_j
    + sigma^2 e_j): against the fp64 kernel (reading R1: s exp(-r^2/2)) the 31-bit grid's rms error
    is the MUFU's alone (~3.3e-8 at C4 shapes, scripts/microbench/prec_bench.cu), well under the
    23-bit grid's (~5.3e-8)."""
    cfg = synth.scaled(synth.CONFIGS["C4"], 60000)     # > 2 drain windows of MODE 3
    pr = synth.make_problem(cfg, seed=0)
    n, m = cfg.n, 24
    cols = np.random.default_rng(5).choice(n, m, replace=False)
    D = np.zeros((n, m))
    D[cols, np.arange(m)] = 1.0
    ls = math.exp(float(pr.log_ls[0]))
    Xs = pr.X.astype(np.float64) / ls
    s = math.exp(pr.log_s)
    noise = math.exp(2 * pr.log_noise)
    Kref = np.stack([s * np.exp(-0.5 * ((Xs - Xs[j]) ** 2).sum(1)) for j in cols], 1)
    rms = {}
    for prec in (bb.INT8EXACT23, bb.INT8EXACT31):
        V = _matmul(ctx, pr, D, prec)
        V[cols, np.arange(m)] -= noise
        rms[prec] = float(np.sqrt(((V - Kref) ** 2).mean()) / s)
    assert rms[bb.INT8EXACT31] < 4.0e-8, rms
    assert rms[bb.INT8EXACT31] < 0.8 * rms[bb.INT8EXACT23], rms


@pytest.mark.parametrize("name,n", [("C4", 4000), ("C4", 1001), ("C3", 2500)])
def test_grid31_mll_and_grad_matches_oracle(ctx, orc, name, n):
    cfg = synth.scaled(synth.CONFIGS[name], n)
    pr, g, o = run_both(ctx, orc, cfg, prec=bb.INT8EXACT31)
    st = g["stats"]
    assert st["matmul_path"] == 2
    np.testing.assert_array_equal(g["pivots"], o["pivots"])
    assert colwise_rel(g["U"].cpu().numpy(), o["U"]).max() < 1e-4
    assert abs(st["logdet"] - o["logdet"]) <= 1e-3 * abs(o["logdet"])
    assert abs(g["mll"] - o["mll"]) <= 1e-3 * abs(o["mll"])
    assert np.linalg.norm(g["grad"] - o["grad"]) <= 1e-3 * np.linalg.norm(o["grad"])


def test_grid31_full_size_matmul_sampled_rows(ctx, orc):
    """C4 at its BASELINE size (n = 1M: 46 uint32 drain windows of MODE 3), the bench's launch
    configuration: sampled rows vs the oracle at the element-wise bound."""
    cfg = synth.CONFIGS["C4"]
    pr = synth.make_problem(cfg, seed=0)
    D = synth.random_block(cfg.n, cfg.t + 1, seed=4).astype(np.float64)
    V = _matmul(ctx, pr, D, bb.INT8EXACT31)
    rows = np.unique(np.concatenate([[0, 1, cfg.n - 1], np.random.default_rng(0).integers(0, cfg.n, 29)]))
    ref = orc.kernel_matmul(cfg.kind, pr.X, pr.log_ls, pr.log_s, pr.log_noise, D, rows=rows)
    absb = orc.kernel_matmul(cfg.kind, pr.X, pr.log_ls, pr.log_s, pr.log_noise, np.abs(D), rows=rows)
    err = np.abs(V[rows] - ref)
    assert np.all(err <= 2e-6 * absb + 1e-12), float((err / absb).max())


@pytest.mark.parametrize("n,bits", [(4000, 23), (131072, 23), (262144, 31), (1000000, 31)])
def test_default_grid_follows_the_error_model(ctx, n, bits):
    """INT8EXACT picks the k~ grid per call: 31 bits where sqrt(n) 5.3e-8 s / sigma^2 > 0.8e-4
    (C4 recipe: s = 1, sigma^2 = 0.3 -> the switch at n ~ 205k); stats report it."""
    cfg = synth.scaled(synth.CONFIGS["C4"], n)
    pr = synth.make_problem(cfg, seed=0)
    g = bb.mll_and_grad(ctx, dev(pr.X), dev(pr.y), hyper_of(pr), 1, 5, 2, seed=7)
    assert g["stats"]["matmul_path"] == 2 and g["stats"]["kgrid_bits"] == bits
    ctx.set_matmul_precision(bb.INT8EXACT23)
    try:
        g = bb.mll_and_grad(ctx, dev(pr.X), dev(pr.y), hyper_of(pr), 1, 5, 2, seed=7)
    finally:
        ctx.set_matmul_precision(bb.INT8EXACT)
    assert g["stats"]["kgrid_bits"] == 23


def test_default_grid_with_column_chunks_sampled_rows(ctx, orc):
    """n = 300 000 (the default operator on the 31-bit grid) with 41 columns (two column chunks of
    33): sampled rows vs the oracle at the element-wise bound."""
    cfg = synth.scaled(synth.CONFIGS["C4"], 300000)
    pr = synth.make_problem(cfg, seed=0)
    D = synth.random_block(cfg.n, 41, seed=4).astype(np.float64)
    V = bb.kernel_matmul(ctx, dev(pr.X), dev(D, torch.float64), hyper_of(pr)).cpu().numpy()
    rows = np.unique(np.concatenate([[0, cfg.n - 1], np.random.default_rng(1).integers(0, cfg.n, 30)]))
    ref = orc.kernel_matmul(cfg.kind, pr.X, pr.log_ls, pr.log_s, pr.log_noise, D, rows=rows)
    absb = orc.kernel_matmul(cfg.kind, pr.X, pr.log_ls, pr.log_s, pr.log_noise, np.abs(D), rows=rows)
    err = np.abs(V[rows] - ref)
    assert np.all(err <= 2e-6 * absb + 1e-12), float((err / absb).max())
