"""GPU parity at large n: bbmm_mll_and_grad against fp64 oracle results cached in tests/golden/large/.

The cache is written by scripts/make_oracle_cache.py, which calls only oracle/ and synth/ (the
oracle at these sizes costs minutes to an hour of host time, so it is not recomputed per run).
Each file carries a SHA-256 of its inputs; the test rebuilds X, y, theta with synth and refuses a
stale cache.  Sizes (VERDICT r1 "next" 1): C4 shape n = 131 072 (4.5 uint32 drain windows of the
on-the-fly tcgen05 kernel, per-step mBCG kernels, the MODE-1 derivative over many windows) and
n = 262 144 (where the default operator switches to the 31-bit kernel-value grid), C3
shape n = 80 000 (ARD, t = 32, tensor-core derivative pass), C2 at its full BASELINE size
n = 45 730 (stored K, Matern-5/2 ARD).

Bars (north_star): pivots bit-exact; solves <= 1e-4 per column (norm-wise);
log|Khat| and mll <= 1e-3 relative; gradient <= 1e-3 norm-wise.  Each case states the oracle's
relres of the y column at p (regime A: < 1e-3).  Where mBCG is far from converged at p
(regime B) the fp64 oracle's own iterate moves by more than the solve bar under a change of
summation order, so there the solve / gradient bars are those of DESIGN.md §6a.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)

import paper_1809_11165_b200 as bb  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
LARGE = os.path.join(HERE, "golden", "large")
OUT = os.path.join(os.path.dirname(HERE), "gpurun_out")

CASES = [("C4", 131072), ("C4", 262144), ("C3", 80000), ("C3", 131072), ("C2", 45730)]
# Regime B: the solve bar is twice the oracle's own rounding floor -- how far the
# fp64 oracle's solves move when its right-hand side moves by one ulp (<name>_n<n>_floor.json,
# scripts/oracle_rounding_floor.py) -- and at least the north-star 1e-4; the gradient bar is 5x the
# regime-A bar (the gradient contracts the same unconverged solves).
REGIME_B_GRAD = 5e-3


def _regime_b_solve_bar(name, n):
    path = os.path.join(LARGE, f"{name}_n{n}_floor.json")
    if not os.path.exists(path):       # no measured floor: the strict bar
        return 1e-4
    return max(1e-4, 2.0 * json.load(open(path))["solve_floor_max"])


def _load(name, n):
    path = os.path.join(LARGE, f"{name}_n{n}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not cached (scripts/make_oracle_cache.py {name}:{n})")
    z = np.load(path)
    return json.loads(str(z["meta"])), z


def _hash(pr):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(pr.X).tobytes())
    h.update(np.ascontiguousarray(pr.y).tobytes())
    h.update(np.asarray(pr.log_ls, np.float64).tobytes())
    h.update(np.asarray([pr.log_s, pr.log_noise], np.float64).tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def ctx():
    c = bb.Context(0)
    yield c
    c.close()


def _run(ctx, name, n, prec, kmode=None):
    meta, z = _load(name, n)
    cfg = synth.scaled(synth.CONFIGS[name], n)
    pr = synth.make_problem(cfg, seed=meta["seed_x"])
    assert _hash(pr) == meta["input_sha256"], "cached oracle results are stale (input recipe changed)"
    X = torch.from_numpy(pr.X).cuda()
    y = torch.from_numpy(pr.y).cuda()
    h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
    ctx.set_matmul_precision(prec)
    try:
        km = kmode if kmode is not None else (bb.STORED if cfg.stored else bb.ONTHEFLY)
        g = bb.mll_and_grad(ctx, X, y, h, cfg.t, cfg.k, cfg.p, seed=meta["seed_probes"],
                            kmode=km, return_solves=True)
    finally:
        ctx.set_matmul_precision(bb.INT8EXACT)
    U = g["U"].cpu().numpy()
    Uo = z["U"].astype(np.float64)
    cols = np.linalg.norm(U - Uo, axis=0) / z["Unorm"]
    err = dict(
        solve=float(cols.max()), solve_y=float(cols[0]), solve_probe_median=float(np.median(cols[1:])),
        logdet=float(abs(g["stats"]["logdet"] - float(z["logdet"])) / abs(float(z["logdet"]))),
        mll=float(abs(g["mll"] - float(z["mll"])) / abs(float(z["mll"]))),
        grad=float(np.linalg.norm(g["grad"] - z["grad"]) / np.linalg.norm(z["grad"])),
        pivots_equal=bool(np.array_equal(g["pivots"], z["pivots"])))
    rec = dict(case=f"{name} n={n}", precision={bb.INT8EXACT: "int8exact", bb.FP64ACC: "fp64acc",
                                               bb.INT8EXACT31: "int8exact31",
                                               bb.INT8EXACT23: "int8exact23"}[prec],
               matmul_path=g["stats"]["matmul_path"], oracle_relres_y=meta["relres_y"],
               regime=meta["regime"], gpu_relres_y=g["stats"]["relres_y"],
               unconverged=g["stats"]["unconverged"], ms_total=g["stats"]["ms_total"], **err)
    print(json.dumps(rec))
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, "fullsize_parity.jsonl"), "a") as f:
        f.write(json.dumps(rec) + "\n")
    return meta, g, err


@pytest.mark.parametrize("name,n", CASES)
def test_fullsize_mll_and_grad_matches_cached_oracle(ctx, name, n):
    meta, g, err = _run(ctx, name, n, bb.INT8EXACT)
    assert err["pivots_equal"]
    assert g["stats"]["k_used"] == synth.CONFIGS[name].k
    assert err["logdet"] <= 1e-3 and err["mll"] <= 1e-3, err
    if meta["regime"] == "A":
        assert err["solve"] <= 1e-4, err
        assert err["grad"] <= 1e-3, err
        assert g["stats"]["unconverged"] == 0
    else:
        assert g["stats"]["unconverged"] == 1
        assert err["solve"] <= _regime_b_solve_bar(name, n), err
        assert err["grad"] <= REGIME_B_GRAD, err


@pytest.mark.parametrize("name,n", [c for c in CASES if c[0] == "C4"])
def test_fullsize_grid31_c4(ctx, name, n):
    """INT8EXACT31 (31-bit kernel-value grid) at the C4 shape: the solve error falls with the
    per-entry kernel-value error (||du||/||u|| ~ sqrt(n) eps / sigma^2)."""
    meta, g, err = _run(ctx, name, n, bb.INT8EXACT31)
    assert err["pivots_equal"] and g["stats"]["matmul_path"] == 2
    assert err["logdet"] <= 1e-3 and err["mll"] <= 1e-3, err
    assert err["solve"] <= 1e-4 and err["grad"] <= 1e-3, err


def test_fullsize_23bit_grid_at_the_switch_point(ctx):
    """The 23-bit k~ grid forced (INT8EXACT23) at the C4 shape, n = 262 144 -- just above the size
    where the default switches to the 31-bit grid (sqrt(n) 5.3e-8 s / sigma^2 = 9.0e-5 > 0.8e-4):
    the solve error there is the model's (residual estimate 8.7e-5), still inside the 1e-4 bar but
    without the 20 % margin the switch keeps."""
    meta, g, err = _run(ctx, "C4", 262144, bb.INT8EXACT23)
    assert g["stats"]["kgrid_bits"] == 23 and err["pivots_equal"]
    assert 0.6e-4 <= err["solve"] <= 1e-4, err
    assert err["logdet"] <= 1e-3 and err["mll"] <= 1e-3 and err["grad"] <= 1e-3, err


@pytest.mark.parametrize("prec", [bb.INT8EXACT, bb.FP64ACC])
def test_fullsize_c2_matern_on_the_fly(ctx, prec):
    """C2 at its full size through the on-the-fly Matern-5/2 operator (K1-TC MODE 2, 39-bit D)
    instead of the stored one, against the same cached oracle run: regime B, so the bars of
    DESIGN.md §6a."""
    meta, g, err = _run(ctx, "C2", 45730, prec, kmode=bb.ONTHEFLY)
    assert err["pivots_equal"]
    assert err["logdet"] <= 1e-3 and err["mll"] <= 1e-3, err
    assert err["solve"] <= _regime_b_solve_bar("C2", 45730), err
    assert err["grad"] <= REGIME_B_GRAD, err


@pytest.mark.parametrize("name,n", CASES)
def test_fullsize_fp64acc_reference_point(ctx, name, n):
    """The CUDA-core fp64-accumulating operator on the same cached cases: the floor an fp32
    kernel value with fp64 D reaches (DESIGN.md §6a compares the default path against it)."""
    meta, g, err = _run(ctx, name, n, bb.FP64ACC)
    assert err["pivots_equal"]
    assert err["logdet"] <= 1e-3 and err["mll"] <= 1e-3, err


# ------------------------------------------------ n = 1M: the north-star solve bar without a 1M oracle
def _residual_estimate(ctx, orc, n, prec, m=512):
    """||y - Khat u|| / (sigma^2 ||u||) for the GPU's y-solve u, the residual evaluated with the fp64
    oracle's Khat on m fixed sampled rows (||r||^2 ~ (n/m) sum r_i^2).  Since lambda_min(Khat) >=
    sigma^2, ||u - Khat^-1 y|| <= ||r|| / sigma^2 (scripts/solve_residual_bound.py)."""
    cfg = synth.scaled(synth.CONFIGS["C4"], n)
    pr = synth.make_problem(cfg, seed=0)
    h = bb.Hyper(cfg.kind, pr.log_ls, pr.log_s, pr.log_noise)
    ctx.set_matmul_precision(prec)
    try:
        g = bb.mll_and_grad(ctx, torch.from_numpy(pr.X).cuda(), torch.from_numpy(pr.y).cuda(), h, cfg.t,
                            cfg.k, cfg.p, seed=7, return_solves=True)
    finally:
        ctx.set_matmul_precision(bb.INT8EXACT)
    u = g["U"][:, 0].cpu().numpy().astype(np.float64)
    rows = np.sort(np.random.default_rng(11).choice(n, m, replace=False))
    Ku = orc.kernel_matmul(cfg.kind, pr.X, pr.log_ls, pr.log_s, pr.log_noise, u[:, None].copy(), rows=rows)
    r = pr.y.astype(np.float64)[rows] - Ku[:, 0]
    rnorm = np.sqrt(n / m * float((r ** 2).sum()))
    return rnorm / (np.exp(2 * pr.log_noise) * np.linalg.norm(u)), u


def test_residual_estimate_tracks_the_oracle_distance(ctx, orc):
    """Calibration at n = 131 072 against the cached oracle solve: the residual estimate is within
    15 % of the measured distance (the kernel-value error lives in the sigma^2 eigenspace)."""
    meta, z = _load("C4", 131072)
    for prec in (bb.INT8EXACT23, bb.INT8EXACT31):
        est, u = _residual_estimate(ctx, orc, 131072, prec)
        true = float(np.linalg.norm(u - z["U"][:, 0].astype(np.float64)) / z["Unorm"][0])
        assert abs(est - true) <= 0.15 * true, (prec, est, true)


def test_north_star_c4_1m_solve(ctx, orc):
    """C4 at n = 1M (the north-star size), residual estimate on 4096 fixed oracle-evaluated rows
    (deterministic: exact integer contraction; ~1.5 % sampling accuracy, and an upper bound that
    exceeded the true distance by 0.3-3 % at n = 131 072): the default operator (INT8EXACT, the
    31-bit kernel-value grid there) puts the y-solve AT the 1e-4 bar -- 1.0009e-4, the floor of
    fp32 MUFU kernel values -- asserted within the estimate's accuracy (5 %);
    the 23-bit grid is at 1.7e-4 (recorded: asserted only to be worse)."""
    est31, _ = _residual_estimate(ctx, orc, 1000000, bb.INT8EXACT, m=4096)
    est23, _ = _residual_estimate(ctx, orc, 1000000, bb.INT8EXACT23, m=4096)
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, "fullsize_parity.jsonl"), "a") as f:
        f.write(json.dumps(dict(case="C4 n=1000000", kind="residual estimate ||y - Khat u||/(sigma^2 ||u||)",
                                int8exact_auto_31bit=est31, int8exact23=est23)) + "\n")
    assert est31 <= 1.05e-4, est31
    assert est23 > 1.5 * est31
