"""Shared helpers for the GPU-vs-oracle parity tests (test infrastructure).

Parity bar (BASELINE.json north_star; SURVEY.md §8(c) parity procedure):
  * tau schedule identical (tau_t in {tau0 beta^k} is exact in binary), except
    after a borderline decision, after which the oracle replays the GPU
    schedule. Borderline = the oracle's relative slack of the (quad) test at
    that trial is within what an entry-wise perturbation of the iterate by the
    value bar e = tol_val * max|omega| can move it: ||Delta|| and ||Delta X^T||
    each move by at most 2 e sqrt(nnz) (times ||X||_2), so the relative slack
    by at most 4 e sqrt(nnz) (1 / ||Delta|| + ||X||_2 / ||Delta X^T||)
    (replaces round 1's flat 1e-5);
  * values: max |omega_gpu - omega_oracle| <= 1e-5 * max |omega_oracle| (f32);
    1e-10 for the float64 path;
  * support: identical except entries whose final-step threshold margin
    | |y_ik| - tau lambda | <= 1e-6 (exempt);
  * objective trace within 1e-6 relative (f32) / 1e-11 (f64).
"""
from __future__ import annotations

import numpy as np

from oracle import accord_oracle as O

TOL = {
    "f32": dict(val=1e-5, f=1e-6, margin=1e-6),
    "f64": dict(val=1e-10, f=1e-11, margin=1e-9),
}


def borderline_slack(entry, nnz, scale, xnorm, tol_val):
    """Largest |relative slack| of the (quad) test that an entry-wise error of
    tol_val * scale in the iterate can explain (see the module docstring)."""
    e = tol_val * scale
    d = max(np.sqrt(entry["dd"]), 1e-300)
    dx = max(np.sqrt(entry["dxx"]), 1e-300)
    return 4.0 * e * np.sqrt(nnz) * (1.0 / d + xnorm / dx)


def csr_to_dense(csr, p):
    return csr.to_dense(p)


def oracle_run(Xt, lam, T, inv_L, tau0=0.5, beta=0.5, tau_schedule=None):
    return O.fbs(Xt, lam, tau0, beta, inv_L, T=T, tau_schedule=tau_schedule)


def compare_full(Xt, lam, T, inv_L, gpu_dense, gpu_stats, kind, tau0=0.5, beta=0.5,
                 check_trace=True):
    """Compare a GPU run (dense Omega rows 0..p-1, per-iteration stats) with the
    oracle. Returns a report dict; raises AssertionError on failure."""
    tol = TOL[kind]
    ref = oracle_run(Xt, lam, T, inv_L, tau0, beta)
    g_taus = np.array([s["tau"] for s in gpu_stats])
    replayed = False
    borderline = 0
    if not np.array_equal(g_taus, ref["taus"]):
        t_star = int(np.nonzero(g_taus != ref["taus"])[0][0])
        # the last trial evaluated by the oracle at t_star decided differently
        ls = [e for e in ref["ls"] if e["t"] == t_star]
        slacks = [abs(e["slack_quad"]) for e in ls]
        nnz = ref["nnz"][t_star - 1] if t_star > 0 else Xt.shape[0]
        scale = np.abs(ref["Omega"]).max()
        xnorm = np.sqrt(np.linalg.eigvalsh((np.asarray(Xt, float).T @ np.asarray(Xt, float)))[-1])
        allowed = [borderline_slack(e, max(nnz, 1), scale, xnorm, tol["val"]) for e in ls]
        assert any(sl <= al for sl, al in zip(slacks, allowed)), (
            f"tau schedule differs at t={t_star} (gpu {g_taus[t_star]}, oracle "
            f"{ref['taus'][t_star]}) with non-borderline slacks {slacks} (allowed {allowed})")
        borderline = 1
        ref = oracle_run(Xt, lam, T, inv_L, tau0, beta, tau_schedule=g_taus)
        replayed = True
    W = ref["Omega"]
    scale = np.abs(W).max()
    sg, so = gpu_dense != 0, W != 0
    diff_support = sg != so
    exempt = np.abs(ref["margins"]) <= tol["margin"]
    bad_support = diff_support & ~exempt
    err = np.abs(gpu_dense - W).max()
    rep = dict(max_abs_err=float(err), rel_err=float(err / scale),
               support_mismatch=int(diff_support.sum()),
               support_exempt=int((diff_support & exempt).sum()),
               bad_support=int(bad_support.sum()), replayed=replayed, borderline=borderline,
               nnz_gpu=int(sg.sum()), nnz_oracle=int(so.sum()))
    assert bad_support.sum() == 0, f"support mismatch outside the exempt band: {rep}"
    assert err <= tol["val"] * scale, f"value error too large: {rep}"
    if check_trace:
        f_or = ref["f"][1:]
        f_g = np.array([s["f"] for s in gpu_stats])
        ftol = tol["f"] * np.abs(f_or)
        assert np.all(np.abs(f_g - f_or) <= ftol), (f_g - f_or, rep)
        rep["max_f_rel"] = float(np.max(np.abs(f_g - f_or) / np.abs(f_or)))
    return rep
