"""Multi-rank row partition on ONE GPU.

G contexts on cuda:0, each driven by its own thread, joined in an in-process rank group
(bbmm_local_group_create / bbmm_ctx_set_local_comm: host-staged all-gather / all-reduce in
rank order).  Every rank runs the same library code as an NCCL rank -- its row range of K-hat,
U, R, Z, D, V, the all-gather of the packed search directions and the all-reduces of the dots
-- so these tests check the partitioned data flow on the real kernels: the G-rank results
must match the single-rank call (reduction order is the only difference) and the oracle.
Covers the tensor-core on-the-fly path (RBF and Matern), the stored int8 path, the FP64ACC
path, ranks with no rows, and the kernel-matmul / mBCG entry points."""
import threading

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)

import paper_1809_11165_b200 as bb  # noqa: E402


def dev(a, dtype=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


def hyper_of(pr):
    return bb.Hyper(pr.cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)


def colwise_rel(a, b):
    return np.linalg.norm(a - b, axis=0) / np.maximum(np.linalg.norm(b, axis=0), 1e-300)


def run_ranks(nranks, fn, prec=bb.INT8EXACT):
    """fn(ctx) on every rank of an in-process group, one thread per rank; results by rank."""
    group = bb.LocalGroup(nranks)
    ctxs = [bb.Context(0, stream=torch.cuda.Stream()) for _ in range(nranks)]
    for r, c in enumerate(ctxs):
        c.set_local_comm(group, r).set_matmul_precision(prec)
    torch.cuda.synchronize()
    out, errs = [None] * nranks, []

    def work(r):
        try:
            out[r] = fn(ctxs[r])
        except Exception as e:          # noqa: BLE001  (re-raised below)
            errs.append(e)

    th = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for c in ctxs:
        c.close()
    group.close()
    if errs:
        raise errs[0]
    return out


def single(fn, prec=bb.INT8EXACT):
    """The single-rank reference call, on the same per-step kernels as the ranks (the fused
    single-rank iteration uses an explicit C^-1 in the Woodbury solve: other rounding)."""
    import os
    ctx = bb.Context(0).set_matmul_precision(prec)
    os.environ["BBMM_NO_FUSED_MBCG"] = "1"
    try:
        return fn(ctx)
    finally:
        os.environ.pop("BBMM_NO_FUSED_MBCG", None)
        ctx.close()


CASES = [  # name, n, kmode, prec, nranks, expected matmul path
    ("C4", 3000, bb.ONTHEFLY, bb.INT8EXACT, 2, 2),
    ("C4", 3000, bb.ONTHEFLY, bb.INT8EXACT, 3, 2),
    ("C1", 3338, bb.STORED, bb.INT8EXACT, 2, 3),
    ("C2", 2500, bb.ONTHEFLY, bb.INT8EXACT, 2, 2),    # Matern on the fly on tcgen05 (MODE 2)
    ("C2", 2500, bb.ONTHEFLY, bb.FP64ACC, 2, 0),
    ("C3", 2000, bb.ONTHEFLY, bb.INT8EXACT, 2, 2),
    ("C4", 3000, bb.ONTHEFLY, bb.FP64ACC, 2, 0),
    ("C4", 300, bb.ONTHEFLY, bb.INT8EXACT, 4, 2),     # n = 300, nb = 128: rank 3 owns no rows
    ("C4", 3000, bb.ONTHEFLY, bb.INT8EXACT31, 3, 2),  # the 31-bit k~ grid (K1-TC MODE 3)
]


@pytest.mark.parametrize("name,n,kmode,prec,nranks,path", CASES)
def test_mll_and_grad_partitioned_matches_single_rank_and_oracle(orc, name, n, kmode, prec,
                                                                  nranks, path):
    cfg = synth.scaled(synth.CONFIGS[name], n)
    pr = synth.make_problem(cfg, seed=0)
    X, y, h = dev(pr.X), dev(pr.y), hyper_of(pr)

    def call(ctx):
        return bb.mll_and_grad(ctx, X, y, h, cfg.t, cfg.k, cfg.p, seed=7, kmode=kmode,
                               return_solves=True)

    parts = run_ranks(nranks, call, prec)
    one = single(call, prec)
    # identical scalars on every rank (rank-ordered reductions)
    for g in parts[1:]:
        assert g["mll"] == parts[0]["mll"]
        np.testing.assert_array_equal(g["grad"], parts[0]["grad"])
    for r, g in enumerate(parts):
        assert g["stats"]["matmul_path"] == path
        r0, r1, _ = bb.row_partition(n, nranks, r)
        assert g["U"].shape[0] == r1 - r0
    U = np.concatenate([g["U"].cpu().numpy() for g in parts], 0)
    g0 = parts[0]
    # vs the single-rank call: only the reduction order differs
    assert colwise_rel(U, one["U"].cpu().numpy()).max() < 1e-6
    assert abs(g0["mll"] - one["mll"]) <= 1e-8 * abs(one["mll"])
    # (the ARD / Matern derivative pass sums fp32 pair products in 16-term chunks per
    #  (row block, j chunk); the row partition changes those blocks -> ~1e-6-level differences)
    assert np.linalg.norm(g0["grad"] - one["grad"]) <= 2e-5 * np.linalg.norm(one["grad"])
    np.testing.assert_array_equal(g0["pivots"], one["pivots"])
    # vs the oracle at the parity bar
    o = orc.mll_and_grad(cfg.kind, pr.X, pr.y, pr.log_ls, pr.log_s, pr.log_noise, cfg.t, cfg.k,
                         cfg.p, seed=7)
    np.testing.assert_array_equal(g0["pivots"], o["pivots"])
    assert colwise_rel(U, o["U"]).max() < 1e-4
    assert abs(g0["mll"] - o["mll"]) <= 1e-3 * abs(o["mll"])
    assert np.linalg.norm(g0["grad"] - o["grad"]) <= 1e-3 * np.linalg.norm(o["grad"])


@pytest.mark.parametrize("kmode", [bb.ONTHEFLY, bb.STORED])
def test_kernel_matmul_partitioned_rows(orc, kmode):
    cfg = synth.scaled(synth.CONFIGS["C4"], 2500)
    pr = synth.make_problem(cfg, seed=3)
    X, h = dev(pr.X), hyper_of(pr)
    D = dev(synth.random_block(2500, 17, seed=4).astype(np.float64), torch.float64)
    parts = run_ranks(2, lambda ctx: bb.kernel_matmul(ctx, X, D, h, kmode).cpu().numpy())
    V = np.concatenate(parts, 0)
    Vs = single(lambda ctx: bb.kernel_matmul(ctx, X, D, h, kmode).cpu().numpy())
    np.testing.assert_allclose(V, Vs, rtol=0, atol=1e-12 * np.abs(Vs).max())


def test_mbcg_partitioned_rows(orc):
    cfg = synth.scaled(synth.CONFIGS["C4"], 3000)
    pr = synth.make_problem(cfg, seed=1)
    X, h = dev(pr.X), hyper_of(pr)
    B = synth.random_block(3000, 17, seed=5).astype(np.float64)
    Lo = orc.pivchol_kernel(cfg.kind, pr.X, pr.log_ls, pr.log_s, cfg.k)[0]
    Ld = dev(Lo.T, torch.float64)

    def call(ctx):
        r0, r1 = ctx.local_rows(3000)
        return bb.mbcg(ctx, X, h, dev(B[r0:r1], torch.float64), L=Ld, max_iter=cfg.p)

    parts = run_ranks(2, call)
    one = single(lambda ctx: bb.mbcg(ctx, X, h, dev(B, torch.float64), L=Ld, max_iter=cfg.p))
    U = np.concatenate([r["U"].cpu().numpy() for r in parts], 0)
    assert colwise_rel(U, one["U"].cpu().numpy()).max() < 1e-6
    np.testing.assert_allclose(parts[0]["alpha"][:5], one["alpha"][:5], rtol=1e-9)
    np.testing.assert_array_equal(parts[0]["alpha"], parts[1]["alpha"])


@pytest.mark.parametrize("name,n,kmode", [("C4", 3000, bb.ONTHEFLY), ("C1", 2000, bb.STORED)])
def test_predict_partitioned_matches_single_rank(orc, name, n, kmode):
    """Row f1 on the partitioned path: every rank returns the same mean / variance for all test
    points, equal to the single-rank call."""
    cfg = synth.scaled(synth.CONFIGS[name], n)
    pr = synth.make_problem(cfg, seed=5)
    Xs = dev(synth.test_points(cfg, 20, seed=9))
    X, y, h = dev(pr.X), dev(pr.y), hyper_of(pr)

    def call(ctx):
        m, v = bb.predict(ctx, X, y, Xs, h, cfg.k, max_iter=cfg.p, kmode=kmode)
        return m.cpu().numpy(), v.cpu().numpy()

    parts = run_ranks(2, call)
    ms, vs = single(call)
    for m, v in parts:
        np.testing.assert_array_equal(m, parts[0][0])
        np.testing.assert_array_equal(v, parts[0][1])
    s = np.exp(pr.log_s)
    assert np.abs(parts[0][0] - ms).max() <= 1e-6 * max(np.abs(ms).max(), 1e-3)
    assert np.abs(parts[0][1] - vs).max() <= 1e-6 * s


def test_train_adam_partitioned_matches_single_rank(orc):
    """Row f2 on the partitioned path: identical trained theta on every rank, equal to the
    single-rank trainer up to reduction order."""
    cfg = synth.scaled(synth.CONFIGS["C4"], 2000)
    pr = synth.make_problem(cfg, seed=6)
    X, y, h0 = dev(pr.X), dev(pr.y), hyper_of(pr)

    def call(ctx):
        h1, tr = bb.train_adam(ctx, X, y, h0, cfg.t, cfg.k, cfg.p, steps=3, seed=3)
        return np.concatenate([np.atleast_1d(h1.log_ls), [h1.log_s, h1.log_noise]]), tr

    parts = run_ranks(2, call)
    th1, tr1 = single(call)
    np.testing.assert_array_equal(parts[0][0], parts[1][0])
    np.testing.assert_allclose(parts[0][0], th1, rtol=0, atol=1e-8)
    np.testing.assert_allclose(parts[0][1][:, 0], tr1[:, 0], rtol=1e-8)


@pytest.mark.parametrize("name,n,kmode", [("C4", 3000, bb.ONTHEFLY), ("C1", 3338, bb.STORED),
                                          ("C3", 2000, bb.ONTHEFLY)])
def test_nccl_single_rank_communicator(orc, name, n, kmode):
    """The NCCL transport on real hardware: a 1-rank NCCL communicator (bbmm_ctx_set_comm with
    nranks = 1) makes the library issue every collective of the multi-GPU path -- all-reduces
    of the dots, the column-max all-reduce, the all-gathers of the packed search directions and
    of the derivative operands -- through NCCL, inside the captured CUDA graph of the mBCG
    iterations, with rho' from the Woodbury identity.  Results match the communicator-free call
    (per-step kernels) and the oracle; the stats attribute time to the collectives."""
    import os
    cfg = synth.scaled(synth.CONFIGS[name], n)
    pr = synth.make_problem(cfg, seed=0)
    X, y, h = dev(pr.X), dev(pr.y), hyper_of(pr)

    def call(ctx):
        return bb.mll_and_grad(ctx, X, y, h, cfg.t, cfg.k, cfg.p, seed=7, kmode=kmode,
                               return_solves=True)

    one = single(call)
    ctx = bb.Context(0).set_comm()
    try:
        g = call(ctx)
        g2 = call(ctx)                                   # the context is reusable
    finally:
        ctx.close()
    assert g["stats"]["ms_comm"] > 0.0
    assert g2["mll"] == g["mll"]
    assert colwise_rel(g["U"].cpu().numpy(), one["U"].cpu().numpy()).max() < 1e-8
    assert abs(g["mll"] - one["mll"]) <= 1e-10 * abs(one["mll"])
    assert np.linalg.norm(g["grad"] - one["grad"]) <= 1e-8 * np.linalg.norm(one["grad"])
    o = orc.mll_and_grad(cfg.kind, pr.X, pr.y, pr.log_ls, pr.log_s, pr.log_noise, cfg.t, cfg.k,
                         cfg.p, seed=7)
    assert colwise_rel(g["U"].cpu().numpy(), o["U"]).max() < 1e-4
    assert abs(g["mll"] - o["mll"]) <= 1e-3 * abs(o["mll"])


def test_graph_capture_matches_eager_iterations(orc):
    """The captured mBCG iterations (tol = 0, per-step kernels) against the same iterations
    launched one by one (BBMM_NO_GRAPH=1): bit-identical results."""
    import os
    cfg = synth.scaled(synth.CONFIGS["C4"], 3000)
    pr = synth.make_problem(cfg, seed=0)
    X, y, h = dev(pr.X), dev(pr.y), hyper_of(pr)

    def call(ctx):
        return bb.mll_and_grad(ctx, X, y, h, cfg.t, cfg.k, cfg.p, seed=7, return_solves=True)

    a = single(call)
    os.environ["BBMM_NO_GRAPH"] = "1"
    try:
        b = single(call)
    finally:
        os.environ.pop("BBMM_NO_GRAPH", None)
    assert a["mll"] == b["mll"]
    np.testing.assert_array_equal(a["grad"], b["grad"])
    np.testing.assert_array_equal(a["U"].cpu().numpy(), b["U"].cpu().numpy())
    assert a["stats"]["ms_matmul"] > 0 and a["stats"]["matmul_launches"] == cfg.p


def test_predict_cov_partitioned_matches_single_rank(orc):
    cfg = synth.scaled(synth.CONFIGS["C4"], 3000)
    pr = synth.make_problem(cfg, seed=0)
    Xs = dev(synth.test_points(cfg, 21, seed=3))
    X, y, h = dev(pr.X), dev(pr.y), hyper_of(pr)

    def call(ctx):
        m, C = bb.predict_cov(ctx, X, y, Xs, h, cfg.k, max_iter=cfg.p)
        return m.cpu().numpy(), C.cpu().numpy()

    parts = run_ranks(3, call)
    m1, C1 = single(call)
    for m, C in parts:
        np.testing.assert_array_equal(C, parts[0][1])
        assert np.abs(C - C1).max() <= 1e-8 and np.abs(m - m1).max() <= 1e-8


@pytest.mark.parametrize("name,t,nranks", [("C4", 39, 2), ("C2", 24, 3)])
def test_column_chunks_partitioned_matches_single_rank(orc, name, t, nranks):
    """K1-TC column chunks (t + 1 above the largest block) on a row partition: each chunk's packed
    operand is all-gathered on its own; results equal the single-rank call up to reduction order."""
    cfg = synth.dataclasses.replace(synth.scaled(synth.CONFIGS[name], 1500), t=t, k=20)
    pr = synth.make_problem(cfg, seed=0)
    X, y, h = dev(pr.X), dev(pr.y), hyper_of(pr)

    def call(ctx):
        return bb.mll_and_grad(ctx, X, y, h, cfg.t, cfg.k, cfg.p, seed=7, kmode=bb.ONTHEFLY,
                               return_solves=True)

    parts = run_ranks(nranks, call, bb.INT8EXACT)
    one = single(call)
    assert all(g["stats"]["matmul_path"] == 2 for g in parts)
    U = np.concatenate([g["U"].cpu().numpy() for g in parts], 0)
    assert colwise_rel(U, one["U"].cpu().numpy()).max() < 1e-6
    assert abs(parts[0]["mll"] - one["mll"]) <= 1e-8 * abs(one["mll"])
    assert np.linalg.norm(parts[0]["grad"] - one["grad"]) <= 2e-5 * np.linalg.norm(one["grad"])
