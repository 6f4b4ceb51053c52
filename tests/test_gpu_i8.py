"""The int8 certified filter (ACCORD_GEMM_I8_FILTER) on the
hardware: tcgen05 kind::i8 with exact s32 accumulation, Y rows quantised per
row, X^T per block of 256 variables, bound = the measured quantisation errors
(Cauchy-Schwarz). The support rule it must not break is Eq. 3.5's
(PAPER.md:233-238): no entry with |G_ik| > lambda may be dropped.

Every check of the bf16 filter's certification (tests/test_gpu_filter.py) is
repeated for the int8 operands -- ratio |acc - nG| / (n delta) < 1 entry by
entry, zero false negatives against the GPU's exact G and the float64
oracle's own iterate, the oracle's tau schedule -- plus the end results: the
estimate after the run against the oracle (BJ parity bar) and lambda_max /
the path on this GEMM kind.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from accord_inputs import make_problem                # noqa: E402
from oracle import accord_oracle as O                 # noqa: E402
import paper_2412_11554_b200 as A                     # noqa: E402
from tests.test_gpu_filter import audit_check         # noqa: E402
from tests.parity_util import compare_full             # noqa: E402


def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA not available on a -m gpu run")


@pytest.mark.parametrize("lam", [0.05, 0.1, 0.2])
def test_i8_filter_certified_config2_every_iteration(lam):
    _cuda()
    pr = make_problem(2)
    c = pr.cfg
    Xt64 = pr.Xt.astype(np.float64)
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    Om_or = np.eye(c.p)
    worst = 0.0
    with A.AccordSolver(torch.from_numpy(pr.Xt).cuda(), lam, inv_L=inv_L,
                        gemm=A.GEMM_I8_FILTER) as s:
        assert s.info()["gemm"] == A.GEMM_I8_FILTER
        for t in range(c.T):
            G_or = O.gradient(Om_or, Xt64)
            rep = audit_check(s, Xt64, lam, s.export_csr(), G_or, tag=f"i8 c2 lam={lam} t={t}")
            assert rep["ratio"] < 1.0
            worst = max(worst, rep["ratio"])
            st = s.step(1)[0]
            r = O.fbs(pr.Xt, lam, c.tau0, c.beta, inv_L, T=1, Omega0=Om_or)
            assert st["tau"] == r["taus"][0], (t, st["tau"], r["taus"][0])
            Om_or = r["Omega"]
        W = s.export_csr().to_dense(c.p)
    assert np.abs(W - Om_or).max() <= 1e-5 * np.abs(Om_or).max()
    assert worst < 1.0


@pytest.mark.parametrize("lam", [0.05, 0.2])
def test_i8_matches_bf16_filter_run(lam):
    """Both filters hand the same exact values to the same prox: the iterate,
    the tau schedule and the objective agree (a larger C only adds entries
    whose prox is 0; sums can differ by float64 re-association only)."""
    _cuda()
    pr = make_problem(2)
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    out = {}
    for g in (A.GEMM_BF16_FILTER, A.GEMM_I8_FILTER):
        with A.AccordSolver(torch.from_numpy(pr.Xt).cuda(), lam, inv_L=inv_L, gemm=g) as s:
            st = s.step(30)
            out[g] = (s.export_csr(), [x["tau"] for x in st], s.objective()[0],
                      [x["n_cand"] for x in st])
    a, b = out[A.GEMM_BF16_FILTER], out[A.GEMM_I8_FILTER]
    assert a[1] == b[1]
    assert np.array_equal(a[0].row_ptr, b[0].row_ptr) and np.array_equal(a[0].col, b[0].col)
    assert np.abs(a[0].val - b[0].val).max() <= 1e-6 * np.abs(a[0].val).max()
    assert abs(a[2] - b[2]) <= 1e-10 * abs(a[2])


@pytest.mark.slow
def test_i8_filter_certified_config3_first_iterations():
    _cuda()
    pr = make_problem(3)
    c = pr.cfg
    lam = c.lambdas[0]
    Xt64 = pr.Xt.astype(np.float64)
    rng = np.random.default_rng(12)
    rows = np.sort(rng.choice(c.p, size=64, replace=False))
    taus = []
    with A.AccordSolver(torch.from_numpy(pr.Xt).cuda(), lam, inv_L=0.0,
                        gemm=A.GEMM_I8_FILTER) as s:
        for t in range(3):
            if t == 0:
                Om_r = np.zeros((len(rows), c.p))
                Om_r[np.arange(len(rows)), rows] = 1.0
            else:
                Om_r = O.fbs_rows(pr.Xt, rows, lam, taus)["Omega_rows"]
            G_or = (Om_r @ Xt64) @ Xt64.T / c.n
            audit_check(s, Xt64, lam, s.export_csr(), G_or, or_rows=rows, tag=f"i8 c3 t={t}")
            taus.append(s.step(1)[0]["tau"])


@pytest.mark.parametrize("nosym", [False, True])
def test_i8_filter_certified_aligned_rounding(nosym, monkeypatch):
    """Every quantisation error of the same sign: all x in a narrow band just
    below the block maximum, so q = 127 and e = 127 b - x >= 0 everywhere
    (Cauchy-Schwarz nearly tight); lambda = the median |G| off the diagonal."""
    _cuda()
    if nosym:
        monkeypatch.setenv("ACCORD_GEMM_NOSYM", "1")
    rng = np.random.default_rng(127)
    p, n = 512, 4096
    Xt = (1.0 + rng.uniform(0.0, 1.0, (p, n)) * 2.0 ** -8).astype(np.float32)
    Xt64 = Xt.astype(np.float64)
    S = Xt64 @ Xt64.T / n
    lam = float(np.median(np.abs(S[~np.eye(p, dtype=bool)])))
    reps = []
    with A.AccordSolver(torch.from_numpy(Xt).cuda(), lam, inv_L=0.0,
                        gemm=A.GEMM_I8_FILTER) as s:
        for t in range(3):
            reps.append(audit_check(s, Xt64, lam, s.export_csr(), tag=f"i8 adv nosym={nosym} t={t}"))
            s.step(1)
    assert reps[0]["ratio"] > 0.3, reps[0]


@pytest.mark.parametrize("key", ["t_ba_f32", "t_hubs_f32", 2])
def test_i8_lambda_max_matches_oracle(key):
    _cuda()
    pr = make_problem(key)
    lm_or = O.lambda_max(pr.Xt)
    with A.AccordSolver(torch.from_numpy(pr.Xt).cuda(), 0.1, inv_L=0.0,
                        gemm=A.GEMM_I8_FILTER) as s:
        s.step(2)
        lm = s.lambda_max()
    assert abs(lm - lm_or) <= 1e-12 * lm_or, (lm, lm_or)


def test_i8_path_matches_oracle():
    _cuda()
    pr = make_problem("t_ba_f32")
    Xt = pr.Xt
    inv_L = 1.0 / O.spectral_bound(Xt)
    with A.AccordSolver(torch.from_numpy(Xt).cuda(), 0.1, inv_L=inv_L,
                        gemm=A.GEMM_I8_FILTER) as s:
        grid = s.lambda_grid(4, 0.2)
        res = s.path(grid, max_iter=40, tol=0.0, gamma=0.5)
        W = s.export_csr().to_dense(pr.cfg.p)
    ref = O.fit_path(Xt, grid, inv_L=inv_L, tol=0.0, max_iter=40, gamma=0.5)
    assert list(res["nnz_off"]) == ref["nnz_off"]
    np.testing.assert_allclose(res["epbic"], ref["epbic"], rtol=1e-6)
    assert res["best"] == ref["best"]
    Wr = ref["Omega"][ref["best"]]
    assert np.abs(W - Wr).max() <= 1e-5 * np.abs(Wr).max()


def test_i8_ragged_shapes_and_workspace():
    """n not a multiple of 128 (K tail of the int8 k-blocks), p not a multiple
    of 256 (ragged last block scale), inside a caller-owned workspace."""
    _cuda()
    rng = np.random.default_rng(5)
    p, n = 700, 333
    Xt = rng.standard_normal((p, n)).astype(np.float32)
    Xt -= Xt.mean(axis=1, keepdims=True)
    inv_L = 1.0 / O.spectral_bound(Xt)
    lam = 0.12
    with A.AccordSolver(torch.from_numpy(Xt).cuda(), lam, inv_L=inv_L, gemm=A.GEMM_I8_FILTER,
                        workspace="torch") as s:
        st = s.step(12)
        W = s.export_csr().to_dense(p)
    compare_full(Xt, lam, 12, inv_L, W, st, "f32")


def test_auto_switch_and_cost_check_config3():
    """AUTO at config 3 (p = 20,000, lambda = 0.1 = 3.2 null sd: the int8 bound
    admits ~3x the bf16 filter's candidates, more than its GEMM saving is
    worth at this p): bf16 until the support is small, one int8 iteration,
    then bf16 for good; the iterate equals the bf16-only
    run's."""
    _cuda()
    pr = make_problem(3)
    lam = pr.cfg.lambdas[0]
    out = {}
    for g in (A.GEMM_AUTO, A.GEMM_BF16_FILTER):
        with A.AccordSolver(torch.from_numpy(pr.Xt).cuda(), lam, inv_L=0.0, gemm=g) as s:
            st = s.step(10)
            out[g] = (s.export_csr(), st, s.info())
    flags = [x["gemm_i8"] for x in out[A.GEMM_AUTO][1]]
    assert flags[0] == 0 and sum(flags) == 1, flags          # exactly one int8 trial
    k = flags.index(1)
    assert all(f == 0 for f in flags[k + 1:])
    assert out[A.GEMM_AUTO][2]["gemm_launches_i8"] == 1
    a, b = out[A.GEMM_AUTO], out[A.GEMM_BF16_FILTER]
    assert [x["tau"] for x in a[1]] == [x["tau"] for x in b[1]]
    assert np.array_equal(a[0].col, b[0].col)
    assert np.abs(a[0].val - b[0].val).max() <= 1e-6 * np.abs(b[0].val).max()
