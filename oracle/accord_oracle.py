"""ACCORD-FBS oracle: a plain, slow, float64 CPU implementation of what the
hot path computes, written from PAPER.md (arXiv 2412.11554).

*** TEST INFRASTRUCTURE ***
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import or call this module. The product path
(paper_2412_11554_b200) never imports it and shares no code with it; the only
module both sides use is accord_inputs (seeded data, no method arithmetic).

Everything is float64 (the paper never states a precision).
X is taken as given (the caller centers it; SURVEY.md §8(c) ambiguity row 12)
and passed variable-major as Xt (p x n, Xt = X^T); float32 inputs are upcast
exactly. Library primitives used as steps: numpy matmul (the two-step
gradient), numpy.linalg.eigvalsh (L). No blocking, fusion or reordering beyond
what the definitions state.

Readings of the paper (listed again in DESIGN.md §3):
  R1 line-search inner product is <Delta, grad g(Omega)> (PAPER.md:259 omits
     the nabla; the proof at PAPER.md:1200 has it).
  R2 the trial Omega+ = Omega^{(t+1)}(tau); Omega^{(t)} is kept until accept.
  R3 grad g is computed once per outer iteration (it does not depend on tau).
  R4 accept the first trial with tau <= 1/L as is (no clamp to 1/L).
  R5 beta = 0.5, tau resets to tau0 each outer iteration.
  R8 canonical test = (quad) ||Delta X^T||^2/n <= ||Delta||_F^2/tau, which is
     algebraically identical to the printed test (lit) because g is quadratic;
     both are evaluated and logged.
  R9 the diagonal is penalised (Eq. 3.2 penalises all entries).
  R10 diagonal prox evaluated in the cancellation-free branch form.
  R11 S_a(x) at |x| = a is exactly 0.

Functions whose parity is pinned by tests/test_oracle_pins.py: prox_diag (P1,
P3), soft_threshold (P2), objective (P4, P5), gradient (P6), fbs (P7-P14, P16,
P17, P18), fbs_rows (P15), kkt_residual (P8, P11), spectral_bound (P-L).
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "prox_diag", "soft_threshold", "prox", "g_value", "objective", "gradient",
    "spectral_bound", "kkt_residual", "fbs", "fbs_rows", "fbs_rows_ls", "candidate_set",
    "penalty_matrix", "epbic", "fit_path", "omega_to_theta", "theta_to_omega",
    "partial_correlations", "lambda_max", "lambda_grid",
]


# ---------------------------------------------------------------------------
# Eq. (3.5): the closed-form backward step
# ---------------------------------------------------------------------------

def prox_diag(y, tau, lam):
    """omega_ii^{(t+1)} = (y - tau*lam + sqrt((y - tau*lam)^2 + 4 tau)) / 2
    (PAPER.md:229), the positive root of w^2 - a w - tau = 0 with
    a = y - tau*lam. Evaluated as
        a >= 0:  (a + sqrt(a^2 + 4 tau)) / 2
        a <  0:  2 tau / (sqrt(a^2 + 4 tau) - a)
    which is the same number without cancellation (reading R10)."""
    y = np.asarray(y, dtype=np.float64)
    a = y - tau * lam
    r = np.sqrt(a * a + 4.0 * tau)
    with np.errstate(divide="ignore", invalid="ignore"):
        neg = 2.0 * tau / (r - a)
    return np.where(a >= 0, 0.5 * (a + r), neg)


def soft_threshold(x, a):
    """S_a(x) = (|x| - a)_+ sign(x); exactly 0 at |x| = a."""
    x = np.asarray(x, dtype=np.float64)
    return np.sign(x) * np.maximum(np.abs(x) - a, 0.0)


def prox(Z, tau, lam, diag_cols):
    """Apply Eq. (3.5) to the forward-step values Z (rows of Omega - tau*G).
    diag_cols[r] is the column of row r's diagonal entry. `lam` is a scalar or
    an entrywise penalty matrix (np.inf = entry fixed at 0, Eq. 3.8)."""
    W = soft_threshold(Z, tau * np.asarray(lam))
    r = np.arange(Z.shape[0])
    lam_d = lam[r, diag_cols] if np.ndim(lam) == 2 else lam
    W[r, diag_cols] = prox_diag(Z[r, diag_cols], tau, lam_d)
    return W


def penalty_matrix(p, lam, mask=None, phi=1.0):
    """Entrywise penalty of the bias-correction refit, Eq. (3.8)
    (PAPER.md:384-398): phi*lam on the support mask S_hat (and the diagonal),
    +inf (entry fixed at zero) off it. mask=None gives the plain lam."""
    if mask is None:
        return lam
    L = np.where(mask, phi * lam, np.inf)
    np.fill_diagonal(L, phi * lam)
    return L


def _l1(Omega, lam):
    if np.ndim(lam) == 0:
        return float(lam * np.abs(Omega).sum())
    fin = np.isfinite(lam)
    return float((lam[fin] * np.abs(Omega[fin])).sum())


# ---------------------------------------------------------------------------
# Objective pieces (Eq. 3.2 / 3.4; g computed from Y = Omega X^T)
# ---------------------------------------------------------------------------

def g_value(Omega, Xt):
    """g(Omega) = 1/2 tr(Omega^T Omega S) = ||Omega X^T||_F^2 / (2n)."""
    n = Xt.shape[1]
    Y = Omega @ np.asarray(Xt, dtype=np.float64)
    return float((Y * Y).sum() / (2.0 * n))


def objective(Omega, Xt, lam):
    """f(Omega) = -log det Omega_D + 1/2 tr(Omega^T Omega S) + lam ||Omega||_1
    (Eq. 3.2); +inf off the domain (omega_ii <= 0). An
    entrywise lam (Eq. 3.8) sums lam_ij |omega_ij| over finite entries (the
    infinite ones are zero by construction)."""
    d = np.diag(Omega)
    if np.any(d <= 0):
        return float("inf")
    return float(-np.log(d).sum() + g_value(Omega, Xt) + _l1(Omega, lam))


def gradient(Omega, Xt):
    """grad g(Omega) = Omega S computed in two steps, Y = Omega X^T then
    (1/n) Y X."""
    Xt = np.asarray(Xt, dtype=np.float64)
    n = Xt.shape[1]
    Y = Omega @ Xt
    return (Y @ Xt.T) / n


def spectral_bound(Xt):
    """L = sigma_max(S), S = X^T X / n. The nonzero spectrum of
    X^T X / n equals that of X X^T / n, so the smaller Gram is used."""
    Xt = np.asarray(Xt, dtype=np.float64)
    p, n = Xt.shape
    M = (Xt.T @ Xt) / n if n <= p else (Xt @ Xt.T) / n
    return float(np.linalg.eigvalsh(M)[-1])


def kkt_residual(Omega, Xt, lam):
    """Max violation of the KKT condition -Omega_D^{-1} + Omega S + lam Z = 0,
    Z in d||Omega||_1 (Eq. 3.3; supp. :985-997):
      diagonal:           | -1/omega_ii + [Omega S]_ii + lam |
      nonzero off-diag:   | [Omega S]_ij + lam sign(omega_ij) |
      zero off-diag:      max(0, |[Omega S]_ij| - lam)."""
    G = gradient(Omega, Xt)
    p = Omega.shape[0]
    lam = np.asarray(lam, dtype=np.float64)
    with np.errstate(invalid="ignore"):
        R = np.where(Omega != 0, np.abs(G + lam * np.sign(Omega)),
                     np.maximum(0.0, np.abs(G) - lam))
    if lam.ndim == 2:          # masked (Eq. 3.8): entries fixed at zero are skipped
        R = np.where(np.isfinite(lam), R, 0.0)
    i = np.arange(p)
    lam_d = lam[i, i] if lam.ndim == 2 else lam
    R[i, i] = np.abs(-1.0 / Omega[i, i] + G[i, i] + lam_d)
    return float(R.max())


def candidate_set(Omega, G, lam):
    """C = diag U supp(Omega) U {|G| > lam}: the entries that can be nonzero
    after one step for ANY tau > 0 (derived from Eq. 3.5)."""
    C = (Omega != 0) | (np.abs(G) > lam)
    np.fill_diagonal(C, True)
    return C


# ---------------------------------------------------------------------------
# Algorithm 1, ACCORD-FBS
# ---------------------------------------------------------------------------

def _trial(Om, G, tau, lam, Xt, diag_cols):
    """One pass of the tau loop body of Algorithm 1 on the
    rows held in Om (reading R2, R3)."""
    Z = Om - tau * G                     # forward step
    On = prox(Z, tau, lam, diag_cols)    # backward step, Eq. (3.5)
    Delta = On - Om
    D = Delta @ Xt                       # Delta X^T
    return Z, On, Delta, D


def fbs(Xt, lam, tau0=0.5, beta=0.5, inv_L=None, T=10, Omega0=None,
        tau_schedule=None):
    """Run T outer iterations of Algorithm 1 with backtracking (beta < 1) or a
    fixed step (beta = 1) from Omega0 (default I).

    If tau_schedule is given, the line search is skipped and tau_t is taken
    from it (used for borderline replays; SURVEY.md §8(c) ambiguity row 14).

    Returns a dict with the final Omega, the accepted tau_t, trial counts, the
    objective trace f(Omega^{(t)}) for t = 0..T, the relative slacks of both
    sufficient-decrease forms for every trial, and the final step's
    off-diagonal threshold margins |y_ij| - tau_T lam."""
    Xt = np.asarray(Xt, dtype=np.float64)
    p, n = Xt.shape
    if inv_L is None:
        inv_L = 1.0 / spectral_bound(Xt)
    Om = np.eye(p) if Omega0 is None else np.array(Omega0, dtype=np.float64)
    diag_cols = np.arange(p)
    taus, trials, f_trace, ls_log = [], [], [objective(Om, Xt, lam)], []
    ncand, nnz = [], []
    margins = None
    for t in range(T):
        Y = Om @ Xt                       # Y = Omega X^T
        G = (Y @ Xt.T) / n                # grad g = (1/n) Y X
        gO = float((Y * Y).sum() / (2 * n))
        ncand.append(int(candidate_set(Om, G, lam).sum()) if np.ndim(lam) == 0 else -1)
        tau = tau0 if tau_schedule is None else float(tau_schedule[t])
        k = 0
        while True:
            k += 1
            Z, On, Delta, D = _trial(Om, G, tau, lam, Xt, diag_cols)
            dd = float((Delta * Delta).sum())
            lhs_q = float((D * D).sum()) / n          # ||Delta X^T||^2 / n
            rhs_q = dd / tau
            Yn = On @ Xt
            g_new = float((Yn * Yn).sum() / (2 * n))
            rhs_l = gO + float((Delta * G).sum()) + dd / (2 * tau)
            quad = lhs_q <= rhs_q
            lit = g_new <= rhs_l
            ls_log.append(dict(t=t, tau=tau, quad=quad, lit=lit,
                               slack_quad=(rhs_q - lhs_q) / max(abs(rhs_q), 1e-300),
                               slack_lit=(rhs_l - g_new) / max(abs(rhs_l), 1e-300),
                               dd=dd, dxx=float((D * D).sum())))
            if tau_schedule is not None or quad or tau <= inv_L:
                break
            tau *= beta
        off = ~np.eye(p, dtype=bool)
        with np.errstate(invalid="ignore"):
            margins = np.where(off & np.isfinite(np.broadcast_to(lam, Z.shape)),
                               np.abs(Z) - tau * np.asarray(lam), np.inf)
        Om = On
        taus.append(tau)
        trials.append(k)
        nnz.append(int((Om != 0).sum()))
        f_trace.append(objective(Om, Xt, lam))
    return dict(Omega=Om, taus=np.array(taus), trials=np.array(trials),
                f=np.array(f_trace), ls=ls_log, margins=margins, inv_L=inv_L,
                ncand=np.array(ncand), nnz=np.array(nnz))


def fbs_rows(Xt, rows, lam, taus, Omega0_rows=None, chunk=16384, trial_taus=None):
    """Sampled-row replay: evolve rows R of Omega
    independently with a given step schedule tau_t. Exact because f separates
    over rows, f = sum_i [-log w_ii + (1/2n)||X w_i^T||^2 + lam ||w_i||_1]
     and Algorithm 1 couples rows only through tau_t.

    trial_taus[t] (optional) lists every step size the line search of
    iteration t evaluated, the accepted taus[t] last: the rejected trials are
    evaluated too (forward step, prox, Delta X^T) and
    discarded, so that a timing of the replay pays for every trial.

    Returns the final rows (|R| x p) and, per iteration, the per-row summands
    ||D_i||^2 and ||Delta_i||^2 of the line-search test."""
    rows = np.asarray(rows, dtype=np.int64)
    p, n = Xt.shape
    Om = np.zeros((len(rows), p))
    if Omega0_rows is None:
        Om[np.arange(len(rows)), rows] = 1.0
    else:
        Om[:] = Omega0_rows
    dsum, ddsum, margins = [], [], None
    for t, tau in enumerate(taus):
        Y = _times_xt(Om, Xt, chunk)                # rows of Omega X^T
        G = _y_times_x(Y, Xt, chunk) / n            # rows of (1/n) Y X
        if trial_taus is not None:
            assert trial_taus[t][-1] == tau
            for tr in trial_taus[t][:-1]:           # rejected trials (evaluated, discarded)
                Zr = Om - tr * G
                Dr = _times_xt(prox(Zr, tr, lam, rows) - Om, Xt, chunk)
                float((Dr * Dr).sum())
        Z = Om - tau * G
        On = prox(Z, tau, lam, rows)
        Delta = On - Om
        D = _times_xt(Delta, Xt, chunk)
        dsum.append((D * D).sum(axis=1))
        ddsum.append((Delta * Delta).sum(axis=1))
        off = np.ones_like(Om, dtype=bool)
        off[np.arange(len(rows)), rows] = False
        margins = np.where(off, np.abs(Z) - tau * lam, np.inf)
        Om = On
    return dict(Omega_rows=Om, D2=np.array(dsum), Delta2=np.array(ddsum),
                margins=margins)


def fbs_rows_ls(Xt, rows, lam, tau0=0.5, beta=0.5, inv_L=None, T=1, Omega0_rows=None,
                chunk=16384):
    """Algorithm 1 restricted to the rows R, with the
    backtracking test ||Delta X^T||_F^2 / n <= ||Delta||_F^2 / tau (reading
    R8) or tau <= 1/L evaluated on those rows' sums only. With R = all rows
    this IS Algorithm 1 (the sums are the global ones; pinned against fbs);
    with a sample of rows the test is an estimate of the global one. Used by
    bench.py's reference arm to time the oracle on a bounded sample of the
    workload with every line-search trial paid for.

    Returns the rows, the accepted taus and the trial counts."""
    rows = np.asarray(rows, dtype=np.int64)
    p, n = Xt.shape
    if inv_L is None:
        inv_L = 1.0 / spectral_bound(Xt)
    Om = np.zeros((len(rows), p))
    if Omega0_rows is None:
        Om[np.arange(len(rows)), rows] = 1.0
    else:
        Om[:] = Omega0_rows
    taus, trials = [], []
    for t in range(T):
        Y = _times_xt(Om, Xt, chunk)
        G = _y_times_x(Y, Xt, chunk) / n
        tau, k = tau0, 0
        while True:
            k += 1
            On = prox(Om - tau * G, tau, lam, rows)
            Delta = On - Om
            D = _times_xt(Delta, Xt, chunk)
            if float((D * D).sum()) / n <= float((Delta * Delta).sum()) / tau or tau <= inv_L:
                break
            tau *= beta
        Om = On
        taus.append(tau)
        trials.append(k)
    return dict(Omega_rows=Om, taus=np.array(taus), trials=np.array(trials))


def _times_xt(A, Xt, chunk):
    """A @ Xt with Xt upcast to float64 chunk by chunk (only nonzero columns
    of A contribute)."""
    cols = np.nonzero(np.any(A != 0, axis=0))[0]
    out = np.zeros((A.shape[0], Xt.shape[1]))
    for s in range(0, len(cols), chunk):
        c = cols[s:s + chunk]
        out += A[:, c] @ np.asarray(Xt[c], dtype=np.float64)
    return out


def _y_times_x(Y, Xt, chunk):
    p = Xt.shape[0]
    out = np.empty((Y.shape[0], p))
    for s in range(0, p, chunk):
        out[:, s:s + chunk] = Y @ np.asarray(Xt[s:s + chunk], dtype=np.float64).T
    return out


# ---------------------------------------------------------------------------
# Tuning and post-processing
# ---------------------------------------------------------------------------

def epbic(Omega, Xt, gamma=0.5):
    """Extended pseudo-BIC, Eq. (3.7):
    2n{-log det Omega_D + 1/2 tr(Omega^T Omega S)} + ||Omega||_0 log n
      + 4 gamma ||Omega||_0 log p,
    ||Omega||_0 = number of nonzero OFF-diagonal entries."""
    Xt = np.asarray(Xt, dtype=np.float64)
    p, n = Xt.shape
    loss = -np.log(np.diag(Omega)).sum() + g_value(Omega, Xt)
    k = int((Omega != 0).sum() - np.count_nonzero(np.diag(Omega)))
    return float(2 * n * loss + k * np.log(n) + 4 * gamma * k * np.log(p))


def lambda_max(Xt):
    """lambda_max = max_{i != k} |S_ik|, S = X^T X / n: the
    top of the lambda grid of a path (SPEC.md lambda_grid)."""
    Xt = np.asarray(Xt, dtype=np.float64)
    S = (Xt @ Xt.T) / Xt.shape[1]
    np.fill_diagonal(S, 0.0)
    return float(np.abs(S).max())


def lambda_grid(Xt, k, ratio):
    """k lambdas evenly spaced in log scale from lambda_max down to
    ratio * lambda_max ("an evenly spaced grid of lambda's
    in logarithmic scale"; SPEC.md lambda_grid)."""
    lm = lambda_max(Xt)
    if k == 1:
        return np.array([lm])
    return lm * ratio ** (np.arange(k) / (k - 1))


def fit_path(Xt, lambdas, tau0=0.5, beta=0.5, inv_L=None, tol=1e-6, max_iter=500,
             gamma=0.5):
    """Regularisation path with warm starts: for each lambda
    in the given order, run Algorithm 1 from the previous estimate until
    ||Omega^(t+1) - Omega^(t)||_F < tol (reading R13) or max_iter, and score it
    by epBIC (Eq. 3.7). Returns estimates, epBIC values, iteration counts and
    the index of the minimum."""
    Om = None
    out = dict(Omega=[], epbic=[], iters=[], nnz_off=[])
    if inv_L is None:
        inv_L = 1.0 / spectral_bound(Xt)
    for lam in lambdas:
        it = 0
        while it < max_iter:
            r = fbs(Xt, lam, tau0, beta, inv_L, T=1, Omega0=Om)
            d = np.linalg.norm(r["Omega"] - (np.eye(Xt.shape[0]) if Om is None else Om))
            Om = r["Omega"]
            it += 1
            if d < tol:
                break
        out["Omega"].append(Om)
        out["epbic"].append(epbic(Om, Xt, gamma))
        out["iters"].append(it)
        out["nnz_off"].append(int((Om != 0).sum() - Om.shape[0]))
    out["best"] = int(np.argmin(out["epbic"]))
    return out


def theta_to_omega(Theta):
    """T: Theta -> Theta_D^{-1/2} Theta."""
    return Theta / np.sqrt(np.diag(Theta))[:, None]


def omega_to_theta(Omega):
    """T^{-1}: Omega -> Omega_D Omega."""
    return np.diag(Omega)[:, None] * Omega


def partial_correlations(Omega):
    """rho_ij = -1/2 (omega_ij / omega_jj + omega_ji / omega_ii), i != j
    (PAPER.md:167-169); symmetric, zero diagonal."""
    d = np.diag(Omega)
    R = -0.5 * (Omega / d[None, :] + Omega.T / d[:, None])
    np.fill_diagonal(R, 0.0)
    return R
