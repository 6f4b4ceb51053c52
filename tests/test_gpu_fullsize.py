"""Parity at BASELINE.json's full sizes (configs 3, 4, 5, and the optional
TCGA-shaped config 6 of SURVEY.md §8(d)), in the launch
configuration bench.py times (default tensor-core path, L from the device
Lanczos, one GPU).

The full oracle is too slow at these sizes (2 p^2 n = 2e15 FLOP per iteration
at config 5), so the checks are:
  * sampled rows: the oracle evolves rows R independently with the step
    schedule the GPU took (exact by row separability) and
    the GPU's rows must match element by element (values within 1e-5 of
    max|omega|, support identical outside the 1e-6 threshold band), and the
    per-row line-search summands ||D_i||^2, ||Delta_i||^2 of the last trial
    must match;
  * properties that hold at any size: every accepted tau is tau0 beta^(k-1)
    with k the trial count, the accepted trial satisfies the sufficient-
    decrease test (or hit the 1/L floor), the objective descends, and the
    exported Omega has a positive diagonal and sorted columns.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

from accord_inputs import get_config, make_problem   # noqa: E402
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


@pytest.mark.parametrize("key", [3, 4, 5, 6])
def test_fullsize_sampled_rows(key):
    if not torch.cuda.is_available():
        pytest.fail("CUDA not available on a -m gpu run")
    cfg = get_config(key)
    pr = make_problem(cfg)
    lam = cfg.lambdas[0]
    T = cfg.T
    X = torch.from_numpy(pr.Xt).cuda()
    with A.AccordSolver(X, lam, tau0=cfg.tau0, beta=cfg.beta, inv_L=0.0) as s:
        info = s.info()
        f0 = s.objective()[0]
        stats = s.step(T)
        rows = sample_rows(pr)
        d2_gpu, dd_gpu = s.row_stats(rows)
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
    # per-row line-search summands of the last trial of the last iteration,
    # compared as norms: an entry-wise error e <= 1e-5 max|omega| moves
    # ||Delta_i|| by at most e sqrt(len_i) and ||Delta_i X^T|| by at most
    # e sqrt(len_i) max_k ||x_k||
    lens = (rp[rows + 1] - rp[rows]).astype(float)
    e = 1e-5 * scale * np.sqrt(lens + 1)
    xmax = np.sqrt((pr.Xt.astype(np.float64) ** 2).sum(axis=1).max())
    a, b = np.sqrt(dd_gpu), np.sqrt(ref["Delta2"][-1])
    assert np.all(np.abs(a - b) <= 1e-3 * b + e), np.max(np.abs(a - b) - 1e-3 * b - e)
    a, b = np.sqrt(d2_gpu), np.sqrt(ref["D2"][-1])
    assert np.all(np.abs(a - b) <= 1e-3 * b + e * xmax), np.max(np.abs(a - b) - 1e-3 * b)
