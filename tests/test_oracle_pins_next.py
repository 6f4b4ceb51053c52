"""Pins of the oracle's NEXT-row functions: the bias-correction
refit (Eq. 3.8), epBIC (Eq. 3.7) and the lambda path, the reparameterisation
T / T^{-1} and partial correlations."""
import json
import os

import numpy as np
import pytest

from oracle import accord_oracle as O
from accord_inputs import center_rows

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_values.json")))


def rand_problem(p, n, seed):
    return center_rows(np.random.default_rng(seed).standard_normal((p, n)))


def test_refit_phi0_equals_restricted_least_squares():
    """phi = 0: on a fixed support the refit minimises the unpenalised loss;
    per row the KKT system has the closed form
    a = 1/sqrt(S_ii - S_iA S_AA^-1 S_Ai), w_A = -S_AA^-1 S_Ai a."""
    Xt = rand_problem(12, 80, 31)
    S = Xt @ Xt.T / 80
    rng = np.random.default_rng(3)
    mask = rng.random((12, 12)) < 0.3
    np.fill_diagonal(mask, True)
    Lm = O.penalty_matrix(12, 0.2, mask, phi=0.0)
    r = O.fbs(Xt, Lm, 0.5, 0.5, None, T=3000)
    W = np.zeros((12, 12))
    for i in range(12):
        A = [k for k in range(12) if k != i and mask[i, k]]
        u = np.linalg.solve(S[np.ix_(A, A)], S[A, i]) if A else np.zeros(0)
        a = 1.0 / np.sqrt(S[i, i] - (S[i, A] @ u if A else 0.0))
        W[i, i] = a
        if A:
            W[i, A] = -u * a
    assert np.abs(r["Omega"] - W).max() < 1e-9
    assert O.kkt_residual(r["Omega"], Xt, Lm) < 1e-8
    assert np.all(r["Omega"][~mask] == 0)


def test_refit_phi1_on_own_support_is_a_fixed_point_and_full_mask_is_plain():
    Xt = rand_problem(15, 60, 32)
    lam = 0.15
    base = O.fbs(Xt, lam, 0.5, 0.5, None, T=2500)
    W = base["Omega"]
    Lm = O.penalty_matrix(15, lam, W != 0, phi=1.0)
    r = O.fbs(Xt, Lm, 0.5, 0.5, None, T=50, Omega0=W)
    assert np.abs(r["Omega"] - W).max() < 1e-9
    r2 = O.fbs(Xt, Lm, 0.5, 0.5, None, T=2500)            # from the identity
    assert np.abs(r2["Omega"] - W).max() < 1e-6
    full = O.penalty_matrix(15, lam, np.ones((15, 15), bool), phi=1.0)
    a = O.fbs(Xt, full, 0.5, 0.5, None, T=20)
    b = O.fbs(Xt, lam, 0.5, 0.5, None, T=20)
    assert np.array_equal(a["Omega"], b["Omega"]) and np.array_equal(a["taus"], b["taus"])


def test_epbic_worked_value():
    c = GOLD["epbic_2x2"]
    X = np.array(c["X"], float)
    assert abs(O.epbic(np.array(c["Omega"], float), X.T, c["gamma"]) - c["expect"]) < 1e-12


def test_fit_path_warm_starts_reach_each_solution():
    Xt = rand_problem(20, 50, 33)
    S = Xt @ Xt.T / 50
    lmax = np.abs(S - np.diag(np.diag(S))).max()
    grid = lmax * np.array([1.5, 0.6, 0.3, 0.15])
    out = O.fit_path(Xt, grid, tol=1e-10, max_iter=3000)
    for lam, W in zip(grid, out["Omega"]):
        assert O.kkt_residual(W, Xt, lam) < 1e-6
    assert out["nnz_off"][0] == 0                      # large lambda: diagonal estimate
    assert out["nnz_off"][-1] > out["nnz_off"][1]
    assert out["best"] == int(np.argmin(out["epbic"]))


def test_reparameterisation_and_partial_correlations():
    c = GOLD["theta_omega"]
    Th, Om = np.array(c["Theta"], float), np.array(c["Omega"], float)
    assert np.allclose(O.theta_to_omega(Th), Om) and np.allclose(O.omega_to_theta(Om), Th)
    rng = np.random.default_rng(34)
    A = rng.standard_normal((6, 6))
    Th = A @ A.T + 6 * np.eye(6)
    assert np.allclose(O.omega_to_theta(O.theta_to_omega(Th)), Th, atol=1e-12)
    # exact Omega* = T(Theta*) gives rho_ij = -theta_ij / sqrt(theta_ii theta_jj)
    R = O.partial_correlations(O.theta_to_omega(Th))
    d = np.sqrt(np.diag(Th))
    want = -Th / np.outer(d, d)
    np.fill_diagonal(want, 0.0)
    assert np.allclose(R, want, atol=1e-12)
    pc = GOLD["partial_corr"]
    assert abs(O.partial_correlations(np.array(pc["Omega"], float))[0, 1] - pc["rho12"]) < 1e-15
    assert np.all(O.partial_correlations(np.diag([1.0, 2.0, 3.0])) == 0)


# ---------------------------------------------------------- lambda grid ------
@pytest.mark.parametrize("case", GOLD["lambda_grid_worked"])
def test_lambda_max_worked(case):
    """lambda_max = max off-diagonal |S_ij| on worked cases (SPEC.md
    lambda_grid example; by hand)."""
    Xt = np.ascontiguousarray(np.array(case["X_samples"], dtype=np.float64).T)
    assert O.lambda_max(Xt) == case["expect_lambda_max"]


def test_lambda_max_brute_force_pairs():
    """Against plain Python dot products over every pair i != k."""
    Xt = rand_problem(9, 13, 77)
    n = Xt.shape[1]
    best = 0.0
    for i in range(9):
        for k in range(9):
            if i != k:
                best = max(best, abs(sum(float(Xt[i, m]) * float(Xt[k, m]) for m in range(n)) / n))
    assert abs(O.lambda_max(Xt) - best) <= 1e-14 * best


@pytest.mark.parametrize("case", GOLD["lambda_grid_spacing"])
def test_lambda_grid_spacing_worked(case):
    # a 2-variable X with S_01 = lambda_max: columns (a, a) scaled
    a = np.sqrt(case["lambda_max"])
    Xt = np.array([[a, -a], [a, -a]])
    g = O.lambda_grid(Xt, case["k"], case["ratio"])
    np.testing.assert_allclose(g, case["expect"], rtol=1e-14)


def test_lambda_max_gives_empty_first_step():
    """At lambda >= lambda_max no off-diagonal entry enters C from Omega = I
    (|G_ik| = |S_ik| <= lambda, Eq. 3.5 / P16): the first FBS step is diagonal."""
    Xt = rand_problem(12, 40, 78)
    lm = O.lambda_max(Xt)
    r = O.fbs(Xt, lm, 0.5, 0.5, None, T=1)
    assert np.count_nonzero(r["Omega"] - np.diag(np.diag(r["Omega"]))) == 0
    r2 = O.fbs(Xt, lm * 0.999, 0.5, 0.5, None, T=1)
    assert np.count_nonzero(r2["Omega"] - np.diag(np.diag(r2["Omega"]))) > 0
