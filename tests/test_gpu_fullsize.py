"""Parity at BASELINE.json's full sizes (configs 3, 4, 5, and the optional
TCGA-shaped config 6 of SURVEY.md §8(d)), in the launch
configuration bench.py times (default tensor-core path, L from the device
Lanczos, one GPU).

  * config 3 in FULL-oracle mode: the oracle's free-running 100 iterations
    are stored by tools/golden_c3.py (oracle only, about an hour of CPU) and
    the GPU must take the identical tau schedule, follow the f trace within
    1e-6 and match 128 stored rows of the final Omega;
  * configs 3-6 by sampled rows: the oracle evolves rows R independently with
    the step schedule the GPU took (exact by row separability,
    PAPER.md:948-957); the GPU's rows must match element by element (values
    within 1e-5 of max|omega|, support identical outside the 1e-6 threshold
    band), and the per-row line-search summands ||D_i||^2, ||Delta_i||^2 of
    EVERY iteration must match (the inputs of every tau decision);
  * properties that hold at any size: every accepted tau is tau0 beta^(k-1)
    with k the trial count, the accepted trial satisfies the sufficient-
    decrease test (or hit the 1/L floor), the objective descends, and the
    exported Omega has a positive diagonal and sorted columns.
"""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

from accord_inputs import get_config, make_problem, xt_sha256   # noqa: E402
from oracle import accord_oracle as O                 # noqa: E402
import paper_2412_11554_b200 as A                     # noqa: E402


def sample_rows(pr, k=48, seed=0):
    p = pr.cfg.p
    rng = np.random.default_rng(seed)
    rows = set(rng.choice(p, size=k, replace=False).tolist())
    rows |= {0, 1, 255, 256, p - 1}
    # highest-degree nodes of the true graph (hubs)
    deg = np.zeros(p, dtype=np.int64)
    off = 0
    for b in pr.blocks:
        np.add.at(deg, off + b.rows, 1)
        off += b.b
    rows |= set(np.argsort(-deg)[:8].tolist())
    return np.array(sorted(rows))


def row_summand_tol(b, lens, scale, xnorm):
    """Tolerance on a per-row line-search summand compared as a norm (b =
    oracle ||Delta_i|| or ||D_i||): 1e-5 relative (SURVEY.md:485) plus what
    an entry-wise value error within the parity bar e = 1e-5 max|omega| can
    move it by: Delta = omega+ - omega carries two such errors, so
    | ||Delta_g|| - ||Delta_o|| | <= 2 e sqrt(len_i), and D = Delta X^T adds
    the factor ||X||_2 = xnorm."""
    return 1e-5 * b + 2e-5 * scale * np.sqrt(lens) * xnorm


@pytest.mark.parametrize("key", [3, 4, 5, 6])
def test_fullsize_sampled_rows(key):
    if not torch.cuda.is_available():
        pytest.fail("CUDA not available on a -m gpu run")
    cfg = get_config(key)
    pr = make_problem(cfg)
    lam = cfg.lambdas[0]
    T = cfg.T
    rows = sample_rows(pr)
    X = torch.from_numpy(pr.Xt).cuda()
    stats, d2_g, dd_g = [], [], []
    with A.AccordSolver(X, lam, tau0=cfg.tau0, beta=cfg.beta, inv_L=0.0) as s:
        info = s.info()
        f0 = s.objective()[0]
        for t in range(T):       # one iteration at a time: the summands of EVERY iteration
            stats += s.step(1)
            d2, dd = s.row_stats(rows)
            d2_g.append(d2)
            dd_g.append(dd)
        csr = s.export_csr()
    assert info["gemm"] == A.GEMM_BF16_FILTER
    del X
    # ---- properties of the step schedule and the objective ----
    f_prev = f0
    for st in stats:
        k = st["trials"]
        assert st["tau"] == cfg.tau0 * cfg.beta ** (k - 1)
        assert st["ls_lhs"] <= st["ls_rhs"] or st["floor_hit"] == 1
        assert st["f"] <= f_prev + 1e-6 * abs(f_prev)
        f_prev = st["f"]
    # ---- exported CSR invariants ----
    rp, col, val = csr.row_ptr, csr.col, csr.val
    assert rp[0] == 0 and rp[-1] == len(col)
    # ---- sampled rows vs the oracle's row replay with the GPU's schedule ----
    taus = [st["tau"] for st in stats]
    ref = O.fbs_rows(pr.Xt, rows, lam, taus)
    W = ref["Omega_rows"]
    G = np.zeros_like(W)
    for q, i in enumerate(rows):
        s0, s1 = rp[i], rp[i + 1]
        c = col[s0:s1]
        assert np.all(np.diff(c) > 0) and i in c
        G[q, c] = val[s0:s1]
        assert G[q, i] > 0
    scale = np.abs(W).max()
    err = np.abs(G - W).max()
    diff = (G != 0) != (W != 0)
    exempt = np.abs(ref["margins"]) <= 1e-6
    assert not np.any(diff & ~exempt), (int(diff.sum()), int((diff & exempt).sum()))
    assert err <= 1e-5 * scale, err / scale
    # ---- per-row line-search summands ||D_i||^2, ||Delta_i||^2 at EVERY
    # iteration (the inputs of every tau decision), compared as norms ----
    xnorm = np.sqrt(O.spectral_bound(pr.Xt) * cfg.n)     # ||X||_2
    d2_g, dd_g = np.array(d2_g), np.array(dd_g)
    lens = (rp[rows + 1] - rp[rows]).astype(float) + 1.0
    for t in range(T):
        a, b = np.sqrt(dd_g[t]), np.sqrt(ref["Delta2"][t])
        tol = row_summand_tol(b, lens, scale, 1.0)
        assert np.all(np.abs(a - b) <= tol), (t, float(np.max(np.abs(a - b) / (b + 1e-300))))
        a, b = np.sqrt(d2_g[t]), np.sqrt(ref["D2"][t])
        tol = row_summand_tol(b, lens, scale, xnorm)
        assert np.all(np.abs(a - b) <= tol), (t, float(np.max(np.abs(a - b) / (b + 1e-300))))


GOLDEN_C3 = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                         "c3_full_oracle.json")


def test_config3_full_oracle_schedule():
    """BASELINE config 3 in FULL-oracle mode (SURVEY.md §8(c) parity procedure
    step 1): the float64 oracle's free-running Algorithm 1 (100 iterations,
    stored by tools/golden_c3.py, which calls only oracle/) against the GPU
    run with the same inv_L: identical tau schedule and trial counts, the
    objective trace within 1e-6, the final nnz within the exempt band, and
    128 stored rows of the final Omega element by element."""
    if not torch.cuda.is_available():
        pytest.fail("CUDA not available on a -m gpu run")
    if not os.path.exists(GOLDEN_C3):
        pytest.skip("tests/golden/c3_full_oracle.json not generated")
    g = json.load(open(GOLDEN_C3))
    cfg = get_config(3)
    pr = make_problem(cfg)
    if xt_sha256(pr.Xt) != g["xt_sha256"]:
        pytest.fail("config-3 X differs from the golden's (numpy / generator drift)")
    inv_L = float.fromhex(g["inv_L_hex"])
    T = g["T"]
    with A.AccordSolver(torch.from_numpy(pr.Xt).cuda(), g["lambda"], tau0=g["tau0"],
                        beta=g["beta"], inv_L=inv_L) as s:
        assert s.info()["gemm"] == A.GEMM_BF16_FILTER
        stats = s.step(T)
        csr = s.export_csr()
    taus = np.array([x["tau"] for x in stats])
    trials = np.array([x["trials"] for x in stats])
    g_taus = np.array(g["taus"])
    if not np.array_equal(taus, g_taus):
        t_star = int(np.nonzero(taus != g_taus)[0][0])
        sl = [abs(e[2]) for e in g["slack_quad"] if e[0] == t_star]
        pytest.fail(f"tau schedule differs at t={t_star} (gpu {taus[t_star]}, oracle "
                    f"{g_taus[t_star]}); oracle slacks there {sl}")
    assert np.array_equal(trials, np.array(g["trials"]))
    f_or = np.array(g["f"][1:])
    f_g = np.array([x["f"] for x in stats])
    assert np.all(np.abs(f_g - f_or) <= 1e-6 * np.abs(f_or)), np.max(np.abs(f_g - f_or) / f_or)
    assert abs(int(csr.row_ptr[-1]) - g["nnz"][-1]) <= g["n_exempt"]
    scale = g["max_abs_omega"]
    rp, col, val = csr.row_ptr, csr.col, csr.val
    worst = 0.0
    for i_s, r in g["rows"].items():
        i = int(i_s)
        oc = np.array(r["cols"], dtype=np.int64)
        ov = np.array([float.fromhex(v) for v in r["vals"]])
        gc = col[rp[i]:rp[i + 1]].astype(np.int64)
        gv = val[rp[i]:rp[i + 1]].astype(np.float64)
        sym = set(oc.tolist()) ^ set(gc.tolist())
        assert sym <= set(r["exempt"]), (i, sorted(sym - set(r["exempt"])))
        allc = np.union1d(oc, gc)
        a = np.zeros(len(allc))
        b = np.zeros(len(allc))
        a[np.searchsorted(allc, gc)] = gv
        b[np.searchsorted(allc, oc)] = ov
        worst = max(worst, float(np.abs(a - b).max()))
    assert worst <= 1e-5 * scale, worst / scale


