"""Pins of the float64 oracle against what the paper and mathematics fix
(SURVEY.md §8(c) P1-P19). CPU only. None of these re-types the oracle's own
formula: each compares it with brute force, a closed form, a library routine
on a special case, an invariant, or a worked value from tests/golden/.
"""
import itertools
import json
import os

import numpy as np
import pytest

from oracle import accord_oracle as O
from accord_inputs import (Config, get_config, make_omega0, make_problem,
                           omega0_dense, sample_xt, center_rows)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                   "worked_values.json")))


def rand_problem(p, n, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    Xt = rng.standard_normal((p, n)) * scale
    return center_rows(Xt)


# ---------------------------------------------------------------- P1 ---------
def _bisect_diag(y, tau, lam, iters=200):
    """argmin_{w>0} -log w + lam w + (w - y)^2/(2 tau) by bisection on the
    increasing derivative phi(w) = -1/w + lam + (w - y)/tau."""
    lo = np.full_like(y, 1e-300)
    hi = np.maximum(np.abs(y), 1.0) + np.abs(lam) * tau + 10.0 * np.sqrt(tau) + 10
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        ph = -1.0 / mid + lam + (mid - y) / tau
        lo = np.where(ph < 0, mid, lo)
        hi = np.where(ph < 0, hi, mid)
    return 0.5 * (lo + hi)


def test_p1_diag_prox_vs_bisection():
    rng = np.random.default_rng(1)
    N = 10000
    y = rng.uniform(-20, 20, N) * rng.choice([1e-3, 1, 10], N)
    tau = np.exp(rng.uniform(np.log(1e-4), np.log(10), N))
    lam = rng.uniform(0, 2, N)
    w = O.prox_diag(y, tau, lam)
    wb = _bisect_diag(y, tau, lam)
    assert np.all(w > 0)
    np.testing.assert_allclose(w, wb, rtol=1e-12, atol=0)


@pytest.mark.parametrize("case", GOLD["prox_diag"])
def test_p1_diag_prox_worked(case):
    w = O.prox_diag(case["y"], case["tau"], case["lam"])
    assert abs(float(w) - case["expect"]) <= 1e-15 * max(1, case["expect"])


# ---------------------------------------------------------------- P2 ---------
def test_p2_soft_threshold_vs_grid():
    rng = np.random.default_rng(2)
    for _ in range(200):
        y = rng.uniform(-3, 3)
        tau = rng.uniform(0.01, 2)
        lam = rng.uniform(0, 1)
        grid = np.linspace(-4, 4, 400001)
        obj = (grid - y) ** 2 / (2 * tau) + lam * np.abs(grid)
        wg = grid[np.argmin(obj)]
        # golden-section refine on the bracket around the grid minimiser
        a, b = wg - 2e-5, wg + 2e-5
        gr = (np.sqrt(5) - 1) / 2
        f = lambda w: (w - y) ** 2 / (2 * tau) + lam * abs(w)
        for _ in range(80):
            c, d = b - gr * (b - a), a + gr * (b - a)
            if f(c) < f(d):
                b = d
            else:
                a = c
        ws = float(O.soft_threshold(y, tau * lam))
        assert abs(ws - 0.5 * (a + b)) < 1e-7   # golden section resolves ~sqrt(eps)


@pytest.mark.parametrize("case", GOLD["soft_threshold"])
def test_p2_soft_worked(case):
    assert abs(float(O.soft_threshold(case["x"], case["a"])) - case["expect"]) < 1e-15


# ---------------------------------------------------------------- P3 ---------
def test_p3_root_identity_and_branches():
    rng = np.random.default_rng(3)
    y = rng.uniform(-50, 50, 5000)
    tau = rng.uniform(1e-3, 5, 5000)
    lam = rng.uniform(0, 1, 5000)
    w = O.prox_diag(y, tau, lam)
    a = y - tau * lam
    u = np.finfo(np.float64).eps
    assert np.all(np.abs(w * w - a * w - tau) <= 8 * u * np.maximum(w * w, tau) + 8 * u * np.abs(a * w))
    # naive printed form agrees on the a >= 0 branch
    m = a >= 0
    naive = (a + np.sqrt(a * a + 4 * tau)) / 2
    np.testing.assert_allclose(w[m], naive[m], rtol=1e-15)
    # f32-dangerous regime: very negative a still gives a positive, finite root
    w2 = O.prox_diag(-1e8, 1e-3, 0.0)
    assert 0 < w2 < 1e-10


# ---------------------------------------------------------------- P4/P5 ------
def test_p4_objective_at_identity():
    Xt = rand_problem(17, 9, 4)
    n = Xt.shape[1]
    lam = 0.37
    S_trace = float(np.einsum("ij,ij->", Xt, Xt)) / n
    assert abs(O.objective(np.eye(17), Xt, lam) - (S_trace / 2 + lam * 17)) < 1e-12


def test_p4_objective_worked():
    c = GOLD["objective_I2"]
    X = np.array(c["X"], dtype=float)
    assert abs(O.objective(np.eye(2), X.T, c["lam"]) - c["expect"]) < 1e-15


def test_p5_g_equals_trace_form():
    rng = np.random.default_rng(5)
    Xt = rand_problem(12, 8, 5)
    S = Xt @ Xt.T / 8
    Om = rng.standard_normal((12, 12)) * (rng.random((12, 12)) < 0.3)
    assert abs(O.g_value(Om, Xt) - 0.5 * np.trace(Om.T @ Om @ S)) < 1e-12


# ---------------------------------------------------------------- P6 ---------
def test_p6_gradient_finite_differences():
    rng = np.random.default_rng(6)
    Xt = rand_problem(10, 7, 6)
    Om = rng.standard_normal((10, 10))
    G = O.gradient(Om, Xt)
    h = 1e-6
    Gfd = np.zeros_like(G)
    for i in range(10):
        for j in range(10):
            E = np.zeros_like(Om)
            E[i, j] = h
            Gfd[i, j] = (O.g_value(Om + E, Xt) - O.g_value(Om - E, Xt)) / (2 * h)
    np.testing.assert_allclose(G, Gfd, rtol=1e-5, atol=1e-7)
    # Omega = I gives S; diagonal Omega scales rows of S
    S = Xt @ Xt.T / 7
    np.testing.assert_allclose(O.gradient(np.eye(10), Xt), S, atol=1e-14)
    d = rng.uniform(0.5, 2, 10)
    np.testing.assert_allclose(O.gradient(np.diag(d), Xt), d[:, None] * S, atol=1e-13)


# ---------------------------------------------------------------- P17 --------
def test_p17_quadratic_identity():
    rng = np.random.default_rng(17)
    Xt = rand_problem(15, 11, 17)
    Om = rng.standard_normal((15, 15))
    De = rng.standard_normal((15, 15)) * (rng.random((15, 15)) < 0.4)
    lhs = O.g_value(Om + De, Xt) - O.g_value(Om, Xt) - float((O.gradient(Om, Xt) * De).sum())
    D = De @ Xt
    assert abs(lhs - (D * D).sum() / (2 * 11)) < 1e-11


# ---------------------------------------------------------------- P7 ---------
@pytest.mark.parametrize("key", ["t_chain", "t_ba_f64", 1])
def test_p7_monotone_descent(key):
    pr = make_problem(key)
    c = pr.cfg
    r = O.fbs(pr.Xt, c.lambdas[0], c.tau0, c.beta, None, T=c.T)
    f = r["f"]
    assert np.all(f[1:] <= f[:-1] + 1e-12 * np.abs(f[:-1]))
    # the (lit) and (quad) forms of the sufficient-decrease test agree unless
    # the decision is borderline (R8)
    for e in r["ls"]:
        if e["quad"] != e["lit"]:
            assert abs(e["slack_quad"]) < 1e-9
    # diagonal stays positive
    assert np.all(np.diag(r["Omega"]) > 0)
    # step sizes satisfy tau_t >= min(tau0, beta/L)
    assert np.all(r["taus"] >= min(c.tau0, c.beta * r["inv_L"]) * (1 - 1e-15))


# ---------------------------------------------------------------- P8/P9 ------
def _converged(Xt, lam, T=3000, beta=0.5, tau0=0.5, Omega0=None):
    return O.fbs(Xt, lam, tau0, beta, None, T=T, Omega0=Omega0)


def test_p8_kkt_and_p9_fixed_point():
    Xt = rand_problem(25, 60, 8)
    lam = 0.12
    r = _converged(Xt, lam, T=1500)
    Om = r["Omega"]
    assert O.kkt_residual(Om, Xt, lam) <= 1e-6
    L = 1.0 / r["inv_L"]
    G = O.gradient(Om, Xt)
    for tau in (0.1 / L, 1.0 / L, 0.5):
        W = O.prox(Om - tau * G, tau, lam, np.arange(25))
        assert np.abs(W - Om).max() <= 1e-8
    # nonzero off-diagonal entries exist (a nontrivial instance)
    assert ((Om != 0).sum() - 25) > 0


@pytest.mark.parametrize("case", GOLD["kkt_worked"])
def test_p8_kkt_residual_worked_nonstationary(case):
    """Eq. (3.3) at NON-stationary Omega, hand-worked: one case per branch
    (diagonal, zero off-diagonal, nonzero off-diagonal) dominates, so dropping
    a branch or flipping the sign of lam*sign(omega) changes the value."""
    X = np.array(case["X_samples"], dtype=np.float64)     # n x p, samples-major
    Xt = np.ascontiguousarray(X.T)
    if "S_by_hand" in case:
        np.testing.assert_array_equal(Xt @ Xt.T / X.shape[0], np.array(case["S_by_hand"]))
    r = O.kkt_residual(np.array(case["Omega"]), Xt, case["lam"])
    assert abs(r - case["expect"]) <= 1e-14, (case["branch"], r)


def test_p16_candidate_set_worked_exact():
    """C equals the hand-worked set, |G_ik| = lam exactly excluded; and C is
    exactly the union over tau of supp prox(Omega - tau G) plus the diagonal
    (an all-True or a superset C fails)."""
    c = GOLD["candidate_set_worked"]
    Om, G, lam = np.array(c["Omega"]), np.array(c["G"]), c["lam"]
    C = O.candidate_set(Om, G, lam)
    np.testing.assert_array_equal(C, np.array(c["expect"], dtype=bool))
    U = np.eye(4, dtype=bool)
    for tau in 10.0 ** np.arange(-300, 7, 3, dtype=np.float64):
        U |= O.prox(Om - tau * G, tau, lam, np.arange(4)) != 0
    np.testing.assert_array_equal(C, U)


# ---------------------------------------------------------------- P10 --------
def test_p10_lambda0_lowdim_closed_form():
    Xt = rand_problem(20, 200, 10)
    S = Xt @ Xt.T / 200
    Th = np.linalg.inv(S)
    Om_star = Th / np.sqrt(np.diag(Th))[:, None]   # T(S^{-1}) = diag^{-1/2} S^{-1}
    r = _converged(Xt, 0.0, T=4000)
    assert np.abs(r["Omega"] - Om_star).max() <= 1e-8 * np.abs(Om_star).max()


# ---------------------------------------------------------------- P11 --------
@pytest.mark.parametrize("case", GOLD["p1_solutions"])
def test_p11_p_equals_1(case):
    # a single variable with s = (1/n) sum x^2 = case["s"]
    n = 4
    x = np.array([1.0, -1.0, 1.0, -1.0]) * np.sqrt(case["s"])
    r = O.fbs(x[None, :], case["lam"], 0.5, 0.5, None, T=400)
    assert abs(r["Omega"][0, 0] - case["expect"]) < 1e-12


def test_p11_large_lambda_diagonal_solution():
    Xt = rand_problem(15, 40, 11)
    S = Xt @ Xt.T / 40
    s = np.diag(S)
    lam = 3.0 * np.abs(S - np.diag(s)).max() / np.sqrt(s.min())
    r = _converged(Xt, lam, T=500)
    Om = r["Omega"]
    assert np.count_nonzero(Om - np.diag(np.diag(Om))) == 0
    w = (-lam + np.sqrt(lam ** 2 + 4 * s)) / (2 * s)
    np.testing.assert_allclose(np.diag(Om), w, rtol=1e-10)
    assert O.kkt_residual(Om, Xt, lam) < 1e-8


# ---------------------------------------------------------------- P12 --------
def test_p12_fixed_vs_backtracking_and_warm_start():
    Xt = rand_problem(20, 50, 12)
    lam = 0.15
    rb = _converged(Xt, lam, T=2000)
    L = 1.0 / rb["inv_L"]
    rf = O.fbs(Xt, lam, 1.0 / L, 1.0, rb["inv_L"], T=6000)
    assert np.linalg.norm(rb["Omega"] - rf["Omega"]) <= 1e-6
    rng = np.random.default_rng(12)
    W0 = rng.standard_normal((20, 20)) * 0.1
    np.fill_diagonal(W0, rng.uniform(0.5, 2, 20))
    rw = _converged(Xt, lam, T=2000, Omega0=W0)
    assert np.linalg.norm(rb["Omega"] - rw["Omega"]) <= 1e-6


# ---------------------------------------------------------------- P13 --------
def test_p13_chain_symmetric_support_recovery():
    cfg = Config(name="chain_rec", p=100, n=4000, dtype="f64", structure="chain",
                 block=100, lambdas=(0.1,), T=0, graph_seed=13, sample_seed=14)
    pr = make_problem(cfg)
    r = O.fbs(pr.Xt, 0.1, 0.5, 0.5, None, T=300)
    Om = r["Omega"]
    i, j = np.nonzero(Om)
    off = i != j
    assert np.all(np.abs(i[off] - j[off]) == 1)
    assert off.sum() == 2 * 99            # both triangles, every chain edge
    # signs agree with the truth (omega*_ij = theta_ij / sqrt(theta_ii) > 0)
    assert np.all(Om[i[off], j[off]] > 0)


# ---------------------------------------------------------------- P14 --------
def _enumerate_row(S, i, lam):
    """Exact minimiser of f_i(w) = -log w_i + w S w^T / 2 + lam ||w||_1 by
    enumerating off-diagonal sign patterns (row separability PAPER.md:948-957,
    KKT PAPER.md:985-997)."""
    p = S.shape[0]
    others = [k for k in range(p) if k != i]
    sols = []
    for pat in itertools.product((-1, 0, 1), repeat=p - 1):
        A = [k for k, s in zip(others, pat) if s != 0]
        sA = np.array([s for s in pat if s != 0], dtype=float)
        if A:
            SAA = S[np.ix_(A, A)]
            u = np.linalg.solve(SAA, S[A, i])        # S_AA^{-1} S_Ai
            v = np.linalg.solve(SAA, sA)             # S_AA^{-1} s_A
            c1 = S[i, i] - S[i, A] @ u
            c0 = lam - lam * (S[i, A] @ v)
        else:
            c1, c0 = S[i, i], lam
        a = (-c0 + np.sqrt(c0 * c0 + 4 * c1)) / (2 * c1)
        w = np.zeros(p)
        w[i] = a
        if A:
            w[A] = -(u * a + lam * v)
            if np.any(np.sign(w[A]) != sA):
                continue
        g = S @ w
        rest = [k for k in others if k not in A]
        if rest and np.any(np.abs(g[rest]) > lam + 1e-12):
            continue
        sols.append(w)
    assert len(sols) >= 1
    return sols[0]


def test_p14_exact_enumeration_tiny():
    for seed, p, lam in [(140, 4, 0.2), (141, 5, 0.1), (142, 5, 0.3)]:
        Xt = rand_problem(p, 30, seed)
        S = Xt @ Xt.T / 30
        W = np.array([_enumerate_row(S, i, lam) for i in range(p)])
        r = _converged(Xt, lam, T=4000)
        assert np.abs(r["Omega"] - W).max() < 1e-10


# ---------------------------------------------------------------- P15 --------
def test_p15_row_replay_equals_full():
    pr = make_problem("t_ba_f64")
    c = pr.cfg
    r = O.fbs(pr.Xt, c.lambdas[0], c.tau0, c.beta, None, T=c.T)
    rows = np.array([0, 5, 149, 150, 299])
    rr = O.fbs_rows(pr.Xt, rows, c.lambdas[0], r["taus"])
    assert np.abs(rr["Omega_rows"] - r["Omega"][rows]).max() < 1e-12


def test_p15_row_replay_with_trials_and_all_rows_line_search():
    """(a) charging the rejected trials does not change the replay; (b) the
    row-restricted line search on ALL rows is Algorithm 1 itself (same tau
    schedule, trial counts and iterate as fbs)."""
    pr = make_problem("t_ba_f64")
    c = pr.cfg
    r = O.fbs(pr.Xt, c.lambdas[0], c.tau0, c.beta, None, T=8)
    rows = np.array([0, 7, 299])
    tt = [[c.tau0 * c.beta ** j for j in range(k)] for k in r["trials"]]
    a = O.fbs_rows(pr.Xt, rows, c.lambdas[0], r["taus"])
    b = O.fbs_rows(pr.Xt, rows, c.lambdas[0], r["taus"], trial_taus=tt)
    assert np.array_equal(a["Omega_rows"], b["Omega_rows"])
    assert max(r["trials"]) > 1                 # the case does backtrack
    ls = O.fbs_rows_ls(pr.Xt, np.arange(c.p), c.lambdas[0], c.tau0, c.beta, r["inv_L"], T=8)
    assert np.array_equal(ls["taus"], r["taus"])
    assert np.array_equal(ls["trials"], r["trials"])
    assert np.abs(ls["Omega_rows"] - r["Omega"]).max() < 1e-12


# ---------------------------------------------------------------- P16 --------
def test_p16_candidate_set_tau_independent():
    pr = make_problem("t_ba_f64")
    c = pr.cfg
    r = O.fbs(pr.Xt, 0.1, 0.5, 0.5, None, T=4)
    Om = r["Omega"]
    G = O.gradient(Om, pr.Xt)
    C = O.candidate_set(Om, G, 0.1)
    p = Om.shape[0]
    new_sets = []
    for tau in (1e-4, 1e-2, 0.1, 0.5, 2.0):
        W = O.prox(Om - tau * G, tau, 0.1, np.arange(p))
        assert not np.any((W != 0) & ~C)
        new_sets.append((W != 0) & (Om == 0))
    for s in new_sets[1:]:
        assert np.array_equal(s, new_sets[0])
    # exactness: C is the union over tau > 0 of the supports (diagonal always),
    # with tau down to 1e-300 so that every nonzero omega_ik survives somewhere
    U = np.eye(p, dtype=bool)
    for tau in np.concatenate([10.0 ** np.arange(-300, -20, 20.0), [1e-8, 1e-4, 0.1, 0.5, 2.0]]):
        U |= O.prox(Om - tau * G, tau, 0.1, np.arange(p)) != 0
    assert np.array_equal(C, U)
    assert 0 < C.sum() < C.size


# ---------------------------------------------------------------- P18 --------
def test_p18_linear_convergence():
    Xt = rand_problem(40, 100, 18)
    lam = 0.1
    r = O.fbs(Xt, lam, 0.5, 0.5, None, T=600)
    fstar = r["f"][-1]
    gap = r["f"][:80] - fstar
    t = np.arange(len(gap))
    m = gap > 1e-11
    y = np.log(gap[m])
    A = np.vstack([t[m], np.ones(m.sum())]).T
    coef, res, *_ = np.linalg.lstsq(A, y, rcond=None)
    r2 = 1 - res[0] / ((y - y.mean()) ** 2).sum()
    assert coef[0] < 0 and r2 >= 0.95


# ---------------------------------------------------------------- P-L --------
@pytest.mark.parametrize("case", GOLD["spectral"])
def test_spectral_worked(case):
    X = np.array(case["X"], dtype=float)
    assert abs(O.spectral_bound(X.T) - case["expect"]) < 1e-14


def test_spectral_vs_power_iteration():
    Xt = rand_problem(30, 20, 19)
    v = np.ones(30)
    for _ in range(5000):
        v = Xt @ (Xt.T @ v) / 20
        v /= np.linalg.norm(v)
    lam_pi = v @ (Xt @ (Xt.T @ v)) / 20
    assert abs(O.spectral_bound(Xt) - lam_pi) < 1e-8 * lam_pi


# ---------------------------------------------------------------- P19 --------
def test_p19_generator_invariants():
    for key in ["t_chain", "t_ba_f64", "t_hubs_f32", 1, 2]:
        cfg = get_config(key)
        blocks = make_omega0(cfg)
        for b in blocks:
            A = b.dense()
            np.testing.assert_allclose(np.diag(A), 1.0)
            assert np.allclose(A, A.T)
            ev = np.linalg.eigvalsh(A)
            assert ev[0] > 0.19
            if cfg.structure in ("ba", "chain"):
                assert (np.count_nonzero(A) - b.b) // 2 == b.b - 1   # tree
            if cfg.structure == "chain":
                assert np.allclose(A[np.arange(b.b - 1), np.arange(1, b.b)], cfg.rho)
            if cfg.structure != "chain":
                # dominance factor 1.5: M - diag(M)/3 is
                # still diagonally dominant, so the rescaled A >= I/3
                assert ev[0] >= 1 / 3 - 1e-12
    # sampler covariance within 5%
    cfg = Config(name="cov", p=20, n=50000, dtype="f64", structure="ba", block=20,
                 lambdas=(0.1,), T=1, graph_seed=5, sample_seed=6)
    b = make_omega0(cfg)
    Xt = sample_xt(cfg, b)
    S = Xt @ Xt.T / cfg.n
    Sig = np.linalg.inv(omega0_dense(b))
    assert np.abs(S - Sig).max() <= 0.05 * np.abs(Sig).max()


def test_inputs_deterministic_and_centered():
    a = make_problem("t_ba_f32").Xt
    b = make_problem("t_ba_f32").Xt
    assert a.dtype == np.float32 and np.array_equal(a, b)
    assert np.abs(a.astype(np.float64).mean(axis=1)).max() < 1e-6
