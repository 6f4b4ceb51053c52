"""GPU parity of the NEXT rows against the float64 oracle:
KKT certificate (Eq. 3.3), solve-to-tolerance, bias-correction refit
(Eq. 3.8), warm-started lambda path with epBIC (Eq. 3.7), Theta-hat and
partial correlations."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from accord_inputs import make_problem   # noqa: E402
from oracle import accord_oracle as O     # noqa: E402
import paper_2412_11554_b200 as A         # noqa: E402


def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA not available on a -m gpu run")


def to_csr(W):
    rp = np.zeros(W.shape[0] + 1, dtype=np.int64)
    cols, vals = [], []
    for i in range(W.shape[0]):
        nz = np.nonzero(W[i])[0]
        cols.append(nz)
        vals.append(W[i, nz])
        rp[i + 1] = rp[i] + len(nz)
    return rp, np.concatenate(cols), np.concatenate(vals)


@pytest.mark.parametrize("key,gemm", [("t_ba_f64", A.GEMM_SIMT), ("t_ba_f32", A.GEMM_AUTO),
                                      ("t_hubs_f32", A.GEMM_AUTO)])
def test_kkt_certificate_matches_oracle(key, gemm):
    """Both sides certify the same iterate: the oracle's Omega after 6
    iterations, loaded into the GPU context with accord_set_omega_csr."""
    _cuda()
    pr = make_problem(key)
    c = pr.cfg
    lam = c.lambdas[0]
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    W = O.fbs(pr.Xt, lam, 0.5, 0.5, inv_L, T=6)["Omega"]
    if c.dtype == "f32":
        W = W.astype(np.float32).astype(np.float64)       # the GPU stores f32 values
    with A.AccordSolver(torch.from_numpy(pr.Xt).cuda(), lam, inv_L=inv_L, gemm=gemm) as s:
        s.set_omega_csr(*to_csr(W))
        k_gpu = s.kkt_residual()
        s.step(1)                       # the certificate does not disturb the iteration
    k_or = O.kkt_residual(W, pr.Xt, lam)
    tol = 1e-12 if pr.cfg.dtype == "f64" else 2e-6
    assert abs(k_gpu - k_or) <= tol * max(1.0, k_or), (k_gpu, k_or)


def test_solve_reaches_the_oracle_minimiser_f64():
    _cuda()
    pr = make_problem("t_ba_f64")
    lam = 0.1
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    with A.AccordSolver(torch.from_numpy(pr.Xt).cuda(), lam, inv_L=inv_L,
                        gemm=A.GEMM_SIMT) as s:
        it, last = s.solve(max_iter=3000, tol=1e-11)
        W = s.export_csr().to_dense(pr.cfg.p)
        kkt = s.kkt_residual()
    assert last["delta_fro"] < 1e-11 and it < 3000
    ref = O.fbs(pr.Xt, lam, 0.5, 0.5, inv_L, T=it)
    assert np.abs(W - ref["Omega"]).max() < 1e-10
    assert kkt < 1e-8 and O.kkt_residual(ref["Omega"], pr.Xt, lam) < 1e-8


@pytest.mark.parametrize("key,gemm,phi", [("t_ba_f64", A.GEMM_SIMT, 0.0),
                                          ("t_ba_f64", A.GEMM_SIMT, 0.5),
                                          ("t_hubs_f32", A.GEMM_AUTO, 0.0)])
def test_refit_matches_oracle(key, gemm, phi):
    _cuda()
    pr = make_problem(key)
    c = pr.cfg
    lam = c.lambdas[0]
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    T1, T2 = 40, 30
    with A.AccordSolver(torch.from_numpy(pr.Xt).cuda(), lam, inv_L=inv_L, gemm=gemm) as s:
        s.step(T1)
        s.refit(phi)
        st = s.step(T2)
        W = s.export_csr().to_dense(c.p)
        kkt = s.kkt_residual()
    base = O.fbs(pr.Xt, lam, 0.5, 0.5, inv_L, T=T1)
    mask = base["Omega"] != 0                                  # the oracle's own support
    Lm = O.penalty_matrix(c.p, lam, mask, phi)
    ref = O.fbs(pr.Xt, Lm, 0.5, 0.5, inv_L, T=T2, Omega0=base["Omega"])
    kind = "f64" if c.dtype == "f64" else "f32"
    g_taus = np.array([x["tau"] for x in st])
    assert np.array_equal(g_taus, ref["taus"])
    scale = np.abs(ref["Omega"]).max()
    assert np.abs(W - ref["Omega"]).max() <= (1e-10 if kind == "f64" else 1e-5) * scale
    assert np.all(W[~mask] == 0)                                 # Eq. 3.8: fixed at zero off S_hat
    f_or = ref["f"][1:]
    assert np.allclose([x["f"] for x in st], f_or, rtol=1e-11 if kind == "f64" else 1e-6)
    k_or = O.kkt_residual(ref["Omega"], pr.Xt, Lm)
    assert abs(kkt - k_or) <= (1e-10 if kind == "f64" else 1e-4) * max(1, k_or)


def test_path_epbic_matches_oracle_f64():
    _cuda()
    pr = make_problem("t_ba_f64")
    Xt = pr.Xt
    S = Xt @ Xt.T / pr.cfg.n
    lmax = np.abs(S - np.diag(np.diag(S))).max()
    grid = lmax * np.array([1.2, 0.5, 0.3, 0.2])
    inv_L = 1.0 / O.spectral_bound(Xt)
    with A.AccordSolver(torch.from_numpy(Xt).cuda(), grid[0], inv_L=inv_L,
                        gemm=A.GEMM_SIMT) as s:
        res = s.path(grid, max_iter=400, tol=1e-9, gamma=0.5)
        W = s.export_csr().to_dense(pr.cfg.p)
        lam_sel = s.info()["lambda_"]
    ref = O.fit_path(Xt, grid, inv_L=inv_L, tol=1e-9, max_iter=400, gamma=0.5)
    assert list(res["iters"]) == ref["iters"]
    assert list(res["nnz_off"]) == ref["nnz_off"]
    np.testing.assert_allclose(res["epbic"], ref["epbic"], rtol=1e-10)
    assert res["best"] == ref["best"] and lam_sel == grid[ref["best"]]
    assert np.abs(W - ref["Omega"][ref["best"]]).max() < 1e-10


def _pc_support(W):
    """supp(Omega) U supp(Omega^T) off the diagonal."""
    M = (W != 0) | (W.T != 0)
    np.fill_diagonal(M, False)
    return M


@pytest.mark.parametrize("key,gemm,T", [("t_ba_f64", A.GEMM_SIMT, 30), ("t_ba_f32", A.GEMM_AUTO, 30),
                                        ("t_hubs_f32", A.GEMM_AUTO, 12)])
def test_theta_and_partial_correlations_match_oracle(key, gemm, T):
    """NEXT(4): Theta-hat = Omega_D Omega and rho-hat on the device vs the
    oracle's T^{-1} and partial_correlations, applied (a) to
    the GPU's own Omega (pins the transform, to rounding) and (b) to the
    oracle's Omega after the same iterations (the parity bar)."""
    _cuda()
    pr = make_problem(key)
    c = pr.cfg
    lam = c.lambdas[0]
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    with A.AccordSolver(torch.from_numpy(pr.Xt).cuda(), lam, inv_L=inv_L, gemm=gemm) as s:
        s.step(T)
        om = s.export_csr()
        th = s.export_transformed(A.EXPORT_THETA)
        pc = s.export_transformed(A.EXPORT_PCORR)
    W = om.to_dense(c.p)
    f64 = c.dtype == "f64"
    eps = 1e-14 if f64 else 2e-7
    # structure: Theta keeps Omega's CSR; rho lives on the symmetrised support, no diagonal
    assert np.array_equal(th.row_ptr, om.row_ptr) and np.array_equal(th.col, om.col)
    R = pc.to_dense(c.p)
    Mpc = np.zeros_like(W, dtype=bool)
    for i in range(c.p):
        Mpc[i, pc.col[pc.row_ptr[i]:pc.row_ptr[i + 1]]] = True
        assert np.all(np.diff(pc.col[pc.row_ptr[i]:pc.row_ptr[i + 1]]) > 0)
    assert np.array_equal(Mpc, _pc_support(W))
    # (a) transform of the GPU's own Omega
    Th_a = O.omega_to_theta(W)
    R_a = O.partial_correlations(W)
    assert np.abs(th.to_dense(c.p) - Th_a).max() <= eps * np.abs(Th_a).max()
    assert np.abs(R - R_a).max() <= eps * max(1.0, np.abs(R_a).max())
    assert np.abs(R - R.T).max() <= eps                        # symmetric by construction
    # (b) against the oracle's own iterate
    ref = O.fbs(pr.Xt, lam, c.tau0, c.beta, inv_L, T=T)["Omega"]
    tol = 1e-10 if f64 else 1e-5
    Th_b = O.omega_to_theta(ref)
    R_b = O.partial_correlations(ref)
    assert np.abs(th.to_dense(c.p) - Th_b).max() <= tol * np.abs(Th_b).max()
    assert np.abs(R - R_b).max() <= tol * max(1.0, np.abs(R_b).max())


def test_transformed_bad_kind_and_identity():
    _cuda()
    pr = make_problem("t_ba_f64")
    with A.AccordSolver(torch.from_numpy(pr.Xt).cuda(), 0.1, gemm=A.GEMM_SIMT) as s:
        with pytest.raises(A.AccordError) as e:
            s.export_transformed(7)
        assert e.value.status == 1
        # identity: Theta = I, rho = empty
        th = s.export_transformed(A.EXPORT_THETA)
        assert np.array_equal(th.val, np.ones(pr.cfg.p))
        pc = s.export_transformed(A.EXPORT_PCORR)
        assert len(pc.col) == 0 and np.all(pc.row_ptr == 0)
