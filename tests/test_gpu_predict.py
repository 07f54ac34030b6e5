"""GPU parity for predictions (Eq. 1): bbmm_predict
through the C-ABI vs the fp64 oracle's predict on the same seeded inputs.

Bar: the solves carry the blackbox matmul's precision (DESIGN.md "Parity bar":
1e-4 per solve column), so mean and variance are held to 1e-4 relative to
max(|mean|) and to 1e-4 s respectively; the mean-only call must agree with the
mean of the full call (column independence of mBCG)."""
import math

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)

import paper_1809_11165_b200 as bb  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    c = bb.Context(0)
    yield c
    c.close()


def dev(a, dtype=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


# (config, n, n*, kmode): n* = 1, 7 (one batch), 40 (16 + 17 + 7: ragged last batch)
CASES = [("C0", 256, 7, bb.ONTHEFLY), ("C1", 3338, 1, bb.STORED), ("C1", 2000, 40, bb.ONTHEFLY),
         ("C2", 1500, 7, bb.STORED), ("C3", 1200, 20, bb.ONTHEFLY), ("C4", 5000, 40, bb.ONTHEFLY),
         ("C4", 300, 1, bb.ONTHEFLY)]


@pytest.mark.parametrize("name,n,ns,kmode", CASES)
def test_predict_matches_oracle(ctx, orc, name, n, ns, kmode):
    cfg = synth.scaled(synth.CONFIGS[name], n)
    pr = synth.make_problem(cfg, seed=5)
    Xs = synth.test_points(cfg, ns, seed=9)
    h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
    k = min(cfg.k, n)
    m, v = bb.predict(ctx, dev(pr.X), dev(pr.y), dev(Xs), h, k, max_iter=cfg.p, kmode=kmode)
    m, v = m.cpu().numpy(), v.cpu().numpy()
    mo, vo = orc.predict(cfg.kind, pr.X, pr.y, Xs, pr.log_ls, pr.log_s, pr.log_noise, k, cfg.p)
    s = math.exp(pr.log_s)
    assert np.abs(m - mo).max() <= 1e-4 * max(np.abs(mo).max(), 1e-3), (m, mo)
    assert np.abs(v - vo).max() <= 1e-4 * s, (v, vo)
    assert np.all(v > -1e-6 * s) and np.all(v <= s * (1 + 1e-9))
    # mean-only path: one solve of y, then k_{X x*}^T alpha
    m2, v2 = bb.predict(ctx, dev(pr.X), dev(pr.y), dev(Xs), h, k, max_iter=cfg.p, kmode=kmode,
                        variance=False)
    assert v2 is None
    np.testing.assert_allclose(m2.cpu().numpy(), m, rtol=0, atol=1e-10 * max(np.abs(m).max(), 1.0))


def test_predict_far_field_and_interpolation(ctx, orc):
    cfg = synth.scaled(synth.CONFIGS["C4"], 2000)
    pr = synth.make_problem(cfg, seed=2)
    h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
    Xs = np.concatenate([np.full((1, cfg.d), 1e3, np.float32), pr.X[[5, 17]]])
    m, v = bb.predict(ctx, dev(pr.X), dev(pr.y), dev(Xs), h, cfg.k, max_iter=cfg.p)
    m, v = m.cpu().numpy(), v.cpu().numpy()
    s = math.exp(pr.log_s)
    assert m[0] == 0.0 and v[0] == s                      # k_{X x*} = 0 exactly: prior
    mo, vo = orc.predict(cfg.kind, pr.X, pr.y, Xs[1:], pr.log_ls, pr.log_s, pr.log_noise, cfg.k,
                         cfg.p)
    np.testing.assert_allclose(m[1:], mo, atol=1e-4 * np.abs(mo).max())
    np.testing.assert_allclose(v[1:], vo, atol=1e-4 * s)


def test_predict_bad_args(ctx):
    X = dev(np.zeros((10, 2), np.float32))
    y = dev(np.zeros(10, np.float32))
    h = bb.Hyper(bb.RBF, [0.0], 0.0, math.log(0.3))
    with pytest.raises(ValueError):
        bb.predict(ctx, X, y, dev(np.zeros((3, 3), np.float32)), h, 2)
    with pytest.raises(bb.BBMMError):
        bb.predict(ctx, X, y, dev(np.full((2, 2), np.nan, np.float32)), h, 2)


@pytest.mark.parametrize("name,n,ns,kmode", [("C4", 3000, 40, bb.ONTHEFLY), ("C1", 2000, 17, bb.STORED),
                                             ("C2", 1500, 5, bb.ONTHEFLY), ("C0", 256, 1, bb.ONTHEFLY)])
def test_predict_cov_matches_oracle(ctx, orc, name, n, ns, kmode):
    """Full predictive covariance between the test points (Eq. 1, bbmm_predict_cov) vs the
    oracle's: element-wise 1e-4 s; its diagonal equals bbmm_predict's variance."""
    cfg = synth.scaled(synth.CONFIGS[name], n)
    pr = synth.make_problem(cfg, seed=5)
    Xs = synth.test_points(cfg, ns, seed=9)
    h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
    k = min(cfg.k, n)
    m, C = bb.predict_cov(ctx, dev(pr.X), dev(pr.y), dev(Xs), h, k, max_iter=cfg.p, kmode=kmode)
    m, C = m.cpu().numpy(), C.cpu().numpy()
    mo, Co = orc.predict_cov(cfg.kind, pr.X, pr.y, Xs, pr.log_ls, pr.log_s, pr.log_noise, k, cfg.p)
    s = math.exp(pr.log_s)
    assert np.abs(m - mo).max() <= 1e-4 * max(np.abs(mo).max(), 1e-3)
    assert np.abs(C - Co).max() <= 1e-4 * s, float(np.abs(C - Co).max())
    _, v = bb.predict(ctx, dev(pr.X), dev(pr.y), dev(Xs), h, k, max_iter=cfg.p, kmode=kmode)
    np.testing.assert_allclose(np.diag(C), v.cpu().numpy(), rtol=0, atol=1e-12 * s)
