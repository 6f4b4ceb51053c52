"""Direct certification of the bf16 tensor-core filter on the hardware
(SURVEY.md:365-369).

The design rests on one claim: the epilogue of the single-pass bf16 GEMM never
drops an entry with |G_ik| > lambda (Eq. 3.5 support rule),
because n*delta_ik = (A_i + gamma (A_i + B_i)) s_k + B_i d_k bounds
|acc_ik - n G_ik| rigorously. accord_filter_audit runs the NEXT iteration's
GEMM + epilogue + finalize exactly as accord_step does and also dumps the raw
fp32 accumulator, so here every entry is checked:

  * ratio_ik = |acc_ik - n G_ik| / (n delta_ik) < 1, with G_ik computed in
    float64 from the f32 Y the GEMM's A operand was rounded from (the
    quantity the bound is about) and delta_ik the UN-inflated bound;
  * C contains diag U supp(Omega) U {|G_ik| > lambda (1 - 4e-6)} (G from the
    GPU's Y, float64) -- zero false negatives;
  * C contains {|G_oracle| > lambda (1 - 4e-6)} for the float64 oracle's own
    iterate (config 2: all rows, every iteration; config 3: sampled rows);
  * |C| / |C_exact| is reported (the filter's cost).

The adversarial case pushes the bound to its limit: n = 4096 (the largest K
of the filter) and same-sign data just above a bf16 half-ulp, so every
product's rounding error has the same sign (Cauchy-Schwarz is then nearly
tight) and the fp32 accumulation term gamma matters.
"""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from accord_inputs import make_problem, get_config   # noqa: E402
from oracle import accord_oracle as O                 # noqa: E402
import paper_2412_11554_b200 as A                     # noqa: E402

REPORT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "gpurun_out", "filter_audit.jsonl")


def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA not available on a -m gpu run")


def audit_check(s, Xt64, lam, om_csr, G_or=None, or_rows=None, tag="", block=1024):
    """One audited GEMM (in row blocks, to bound host memory at p = 20,000):
    returns a report dict, asserts the certificate."""
    a = s.filter_audit()
    p, n = Xt64.shape
    g = a["gamma"]
    s_k = a["col_s"].astype(np.float64)[None, :]
    d_k = a["col_d"].astype(np.float64)[None, :]
    rp, col = a["c_ptr"], a["c_col"]
    pk = len(rp) - 1
    r0 = s.row_begin
    ratio, err_max, fn, n_need = 0.0, 0.0, 0, 0
    rows_or = np.arange(pk) if or_rows is None else np.asarray(or_rows)
    fn_or, need_or_n, cand_or_n = 0, 0, 0
    for b0 in range(0, pk, block):
        b1 = min(pk, b0 + block)
        acc = a["acc"][b0:b1].double().cpu().numpy()
        assert not np.isnan(acc).any(), "audit: an accumulator entry was never written"
        Y = a["y"][b0:b1].double().cpu().numpy()
        G = (Y @ Xt64.T) / n                               # exact G of the GPU's Y (f64)
        Ai = a["row_A"][b0:b1].astype(np.float64)[:, None]
        Bi = a["row_B"][b0:b1].astype(np.float64)[:, None]
        nd = (Ai + g * (Ai + Bi)) * s_k + Bi * d_k       # n delta_ik, not inflated
        err = np.abs(acc - n * G)
        ratio = max(ratio, float((err / nd).max()))
        err_max = max(err_max, float(err.max()))
        C = np.zeros((b1 - b0, p), dtype=bool)
        rr = np.repeat(np.arange(b1 - b0), np.diff(rp[b0:b1 + 1]))
        C[rr, col[rp[b0]:rp[b1]]] = True
        need = np.abs(G) > lam * (1 - 4e-6)
        need[np.arange(b1 - b0), r0 + np.arange(b0, b1)] = True
        orr = np.repeat(np.arange(b1 - b0), np.diff(om_csr.row_ptr[b0:b1 + 1]))
        need[orr, om_csr.col[om_csr.row_ptr[b0]:om_csr.row_ptr[b1]]] = True
        fn += int((need & ~C).sum())
        n_need += int(need.sum())
        if G_or is not None:
            sel = np.nonzero((rows_or >= b0) & (rows_or < b1))[0]
            if len(sel):
                Go = G_or[sel]
                no = np.abs(Go) > lam * (1 - 4e-6)
                no[np.arange(len(sel)), r0 + rows_or[sel]] = True
                Cs = C[rows_or[sel] - b0]
                fn_or += int((no & ~Cs).sum())
                need_or_n += int(no.sum())
                cand_or_n += int(Cs.sum())
    rep = dict(tag=tag, ratio=ratio, err_max=err_max, n_cand=int(rp[-1]), n_need=n_need,
               false_neg=fn)
    if G_or is not None:
        rep["false_neg_oracle"] = fn_or
        rep["c_over_exact"] = cand_or_n / max(1, need_or_n)
    os.makedirs(os.path.dirname(REPORT), exist_ok=True)
    with open(REPORT, "a") as f:
        f.write(json.dumps(rep) + "\n")
    assert ratio < 1.0, rep
    assert fn == 0, rep
    if G_or is not None:
        assert rep["false_neg_oracle"] == 0, rep
    return rep


@pytest.mark.parametrize("lam", [0.05, 0.1, 0.2])
def test_filter_certified_config2_every_iteration(lam):
    """BASELINE config 2, all three lambdas, all 100 iterations: the audited
    candidate set against the GPU's exact G and the oracle's own iterate."""
    _cuda()
    pr = make_problem(2)
    c = pr.cfg
    Xt64 = pr.Xt.astype(np.float64)
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    Om_or = np.eye(c.p)
    worst = 0.0
    with A.AccordSolver(torch.from_numpy(pr.Xt).cuda(), lam, inv_L=inv_L) as s:
        assert s.info()["gemm"] == A.GEMM_BF16_FILTER
        for t in range(c.T):
            G_or = O.gradient(Om_or, Xt64)
            rep = audit_check(s, Xt64, lam, s.export_csr(), G_or, tag=f"c2 lam={lam} t={t}")
            worst = max(worst, rep["ratio"])
            st = s.step(1)[0]
            r = O.fbs(pr.Xt, lam, c.tau0, c.beta, inv_L, T=1, Omega0=Om_or)
            assert st["tau"] == r["taus"][0], (t, st["tau"], r["taus"][0])
            Om_or = r["Omega"]
    assert worst < 1.0


@pytest.mark.slow
def test_filter_certified_config3_first_iterations():
    """BASELINE config 3 (p = 20,000): every entry of the first 5 GEMMs
    against the GPU's exact G; 96 sampled rows against the oracle's rows
    (row replay with the same tau schedule, exact by PAPER.md:948-957)."""
    _cuda()
    pr = make_problem(3)
    c = pr.cfg
    lam = c.lambdas[0]
    Xt64 = pr.Xt.astype(np.float64)
    rng = np.random.default_rng(11)
    rows = np.sort(rng.choice(c.p, size=96, replace=False))
    taus = []
    with A.AccordSolver(torch.from_numpy(pr.Xt).cuda(), lam, inv_L=0.0) as s:
        for t in range(5):
            if t == 0:
                Om_r = np.zeros((len(rows), c.p))
                Om_r[np.arange(len(rows)), rows] = 1.0
            else:
                Om_r = O.fbs_rows(pr.Xt, rows, lam, taus)["Omega_rows"]
            G_or = (Om_r @ Xt64) @ Xt64.T / c.n
            audit_check(s, Xt64, lam, s.export_csr(), G_or, or_rows=rows, tag=f"c3 t={t}")
            taus.append(s.step(1)[0]["tau"])


@pytest.mark.parametrize("nosym", [False, True])
def test_filter_certified_adversarial_aligned_rounding(nosym, monkeypatch):
    """n = 4096, every x just above the bf16 half-ulp of 1 (x = 1 + 2^-8 +
    u 2^-9): all rounding errors positive, the products' errors aligned, the
    fp32 accumulator near 4096 (accumulation error largest). lambda = the
    median |G| off the diagonal, so half the entries sit near the threshold.
    The symmetric first GEMM (Omega = I) and the full schedule, then an
    iteration later (Omega != I)."""
    _cuda()
    if nosym:
        monkeypatch.setenv("ACCORD_GEMM_NOSYM", "1")
    rng = np.random.default_rng(4096)
    p, n = 512, 4096
    Xt = (1.0 + 2.0 ** -8 + rng.uniform(0.01, 0.99, (p, n)) * 2.0 ** -9).astype(np.float32)
    Xt64 = Xt.astype(np.float64)
    S = Xt64 @ Xt64.T / n
    off = S[~np.eye(p, dtype=bool)]
    lam = float(np.median(np.abs(off)))
    reps = []
    with A.AccordSolver(torch.from_numpy(Xt).cuda(), lam, inv_L=0.0) as s:
        assert s.info()["gemm"] == A.GEMM_BF16_FILTER
        for t in range(3):
            reps.append(audit_check(s, Xt64, lam, s.export_csr(), tag=f"adv nosym={nosym} t={t}"))
            s.step(1)
    # the aligned case really does stress the bound
    assert reps[0]["ratio"] > 0.5, reps[0]


@pytest.mark.parametrize("key,gemm", [("t_ba_f32", A.GEMM_AUTO), ("t_hubs_f32", A.GEMM_AUTO),
                                      (2, A.GEMM_AUTO), ("t_ba_f64", A.GEMM_SIMT),
                                      (1, A.GEMM_SIMT), ("t_ba_f32", A.GEMM_BF16X3)])
def test_lambda_max_and_grid_match_oracle(key, gemm):
    """lambda_max = max_{i != k} |S_ik| on the device (tensor-core max-reduce
    pass + candidate pass + exact refine; CUDA-core dots for SIMT / BF16X3)
    equals the oracle's to float64 rounding; the grid is its log-spaced
    descent."""
    _cuda()
    pr = make_problem(key)
    lm_or = O.lambda_max(pr.Xt)
    with A.AccordSolver(torch.from_numpy(pr.Xt).cuda(), 0.1, inv_L=0.0, gemm=gemm) as s:
        s.step(2)                               # the iterate is not I: lambda_max ignores it
        before = s.export_csr()
        lm = s.lambda_max()
        grid = s.lambda_grid(5, 0.1)
        after = s.export_csr()
        s.step(1)
    assert abs(lm - lm_or) <= 1e-12 * lm_or, (lm, lm_or)
    np.testing.assert_allclose(grid, O.lambda_grid(pr.Xt, 5, 0.1), rtol=1e-12)
    assert np.array_equal(before.col, after.col) and np.array_equal(before.val, after.val)


def test_lambda_max_nosym_and_zero_data(monkeypatch):
    _cuda()
    monkeypatch.setenv("ACCORD_GEMM_NOSYM", "1")
    pr = make_problem("t_mid_f32")
    with A.AccordSolver(torch.from_numpy(pr.Xt).cuda(), 0.1, inv_L=0.0) as s:
        assert abs(s.lambda_max() - O.lambda_max(pr.Xt)) <= 1e-12 * O.lambda_max(pr.Xt)
    Z = np.zeros((300, 64), dtype=np.float32)
    Z[:, 0] = 1.0
    Z[:, 1] = -1.0      # every variable identical up to scale: S_ik = 2/64 > 0
    with A.AccordSolver(torch.from_numpy(Z).cuda(), 0.1, inv_L=1.0) as s:
        assert abs(s.lambda_max() - 2.0 / 64) <= 1e-15


def test_path_on_the_tensor_core_filter_path():
    """accord_path on the default f32 BF16_FILTER path, grid from the device
    lambda_max, fixed iteration count per lambda (tol = 0): epBIC, off-diagonal
    nnz, selection and the selected estimate against oracle.fit_path (Eq. 3.7)."""
    _cuda()
    pr = make_problem("t_ba_f32")
    Xt = pr.Xt
    inv_L = 1.0 / O.spectral_bound(Xt)
    with A.AccordSolver(torch.from_numpy(Xt).cuda(), 0.1, inv_L=inv_L) as s:
        assert s.info()["gemm"] == A.GEMM_BF16_FILTER
        grid = s.lambda_grid(4, 0.2)
        res = s.path(grid, max_iter=40, tol=0.0, gamma=0.5)
        W = s.export_csr().to_dense(pr.cfg.p)
    ref = O.fit_path(Xt, grid, inv_L=inv_L, tol=0.0, max_iter=40, gamma=0.5)
    assert list(res["iters"]) == ref["iters"] == [40] * 4
    assert list(res["nnz_off"]) == ref["nnz_off"]
    np.testing.assert_allclose(res["epbic"], ref["epbic"], rtol=1e-6)
    assert res["best"] == ref["best"]
    Wr = ref["Omega"][ref["best"]]
    assert np.abs(W - Wr).max() <= 1e-5 * np.abs(Wr).max()
