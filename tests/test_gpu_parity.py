"""GPU parity: the CUDA path through the C ABI vs the float64 oracle on the
same seeded inputs (BASELINE.json configs 1-2 in full; small cases of the
same recipes spanning several tiles and ragged tails)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from accord_inputs import make_problem, get_config   # noqa: E402
from oracle import accord_oracle as O                 # noqa: E402
from tests.parity_util import compare_full            # noqa: E402
import paper_2412_11554_b200 as A                     # noqa: E402


def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA not available on a -m gpu run")


def run_gpu(Xt, lam, T, inv_L, gemm, layout="variables", tau0=0.5, beta=0.5, **kw):
    X = torch.from_numpy(Xt if layout == "variables" else np.ascontiguousarray(Xt.T)).cuda()
    with A.AccordSolver(X, lam, layout=layout, tau0=tau0, beta=beta, inv_L=inv_L, gemm=gemm,
                        **kw) as s:
        stats = s.step(T)
        csr = s.export_csr()
        info = s.info()
    return csr, stats, info


@pytest.mark.parametrize("key", ["t_chain", "t_ba_f64", 1])
def test_parity_f64_simt(key):
    _cuda()
    pr = make_problem(key)
    c = pr.cfg
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    for lam in c.lambdas:
        csr, stats, info = run_gpu(pr.Xt, lam, c.T, inv_L, A.GEMM_SIMT)
        assert info["gemm"] == A.GEMM_SIMT and info["dtype"] == A.F64
        rep = compare_full(pr.Xt, lam, c.T, inv_L, csr.to_dense(c.p), stats, "f64")
        assert not rep["replayed"]


@pytest.mark.parametrize("gemm", [A.GEMM_SIMT, A.GEMM_BF16X3, A.GEMM_BF16_FILTER])
@pytest.mark.parametrize("key", ["t_ba_f32", "t_hubs_f32"])
@pytest.mark.parametrize("spmm", ["default", "tma"])
def test_parity_f32_small(key, gemm, spmm, monkeypatch):
    """spmm = tma forces the TMA-staged SpMM (used by default for row blocks of
    >= 65536 rows) on these small cases too."""
    _cuda()
    if spmm == "tma":
        monkeypatch.setenv("ACCORD_SPMM_TMA", "1")
    pr = make_problem(key)
    c = pr.cfg
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    csr, stats, info = run_gpu(pr.Xt, c.lambdas[0], c.T, inv_L, gemm)
    assert info["gemm"] == gemm
    compare_full(pr.Xt, c.lambdas[0], c.T, inv_L, csr.to_dense(c.p), stats, "f32")


@pytest.mark.parametrize("lam", [0.05, 0.1, 0.2])
def test_parity_config2_full(lam):
    """BASELINE config 2 (p=2000, n=500, f32, BA tree), 100 iterations, all lambdas."""
    _cuda()
    pr = make_problem(2)
    c = pr.cfg
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    csr, stats, info = run_gpu(pr.Xt, lam, c.T, inv_L, A.GEMM_AUTO)
    assert info["gemm"] in (A.GEMM_BF16_FILTER, A.GEMM_I8_FILTER)   # AUTO: bf16, then int8
    compare_full(pr.Xt, lam, c.T, inv_L, csr.to_dense(c.p), stats, "f32")


def test_sample_major_layout_matches_variable_major():
    _cuda()
    pr = make_problem("t_ba_f64")
    c = pr.cfg
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    a, sa, _ = run_gpu(pr.Xt, 0.1, 5, inv_L, A.GEMM_SIMT, layout="variables")
    b, sb, _ = run_gpu(pr.Xt, 0.1, 5, inv_L, A.GEMM_SIMT, layout="samples")
    assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col, b.col)
    assert np.array_equal(a.val, b.val)


def test_objective_at_identity_and_export_invariants():
    _cuda()
    pr = make_problem("t_ba_f32")
    X = torch.from_numpy(pr.Xt).cuda()
    lam = 0.1
    with A.AccordSolver(X, lam, inv_L=0.0) as s:
        f0, parts = s.objective()
        Xd = pr.Xt.astype(np.float64)
        want = (Xd * Xd).sum() / (2 * pr.cfg.n) + lam * pr.cfg.p
        assert abs(f0 - want) <= 1e-6 * want
        info = s.info()
        L = O.spectral_bound(pr.Xt)
        assert L <= info["L"] <= L * 1.01      # device Lanczos, inflated: safe side
        assert abs(info["L"] / (1 + 2e-3) - L) <= 1e-9 * L   # Lanczos converged to sigma_max(S)
        s.step(3)
        csr = s.export_csr()
    p = pr.cfg.p
    for i in range(p):
        cols = csr.col[csr.row_ptr[i]:csr.row_ptr[i + 1]]
        vals = csr.val[csr.row_ptr[i]:csr.row_ptr[i + 1]]
        assert np.all(np.diff(cols) > 0)
        assert i in cols and vals[list(cols).index(i)] > 0
        assert np.all((vals != 0) | (cols == i))


def test_lanczos_exactly_centered_and_zero_x():
    """L from the device Lanczos on EXACTLY centered data (balanced +-1
    columns: X^T 1 = 0 in exact arithmetic, so a constant start vector would
    be mapped to 0) is sigma_max(S), and X = 0 is
    reported instead of silently disabling the tau <= 1/L floor."""
    _cuda()
    rng = np.random.default_rng(5)
    p, n = 300, 64
    half = np.array([1.0] * (n // 2) + [-1.0] * (n // 2), dtype=np.float32)
    Xt = np.stack([rng.permutation(half) for _ in range(p)])
    assert np.all(Xt.sum(axis=1) == 0)
    L = O.spectral_bound(Xt)
    with A.AccordSolver(torch.from_numpy(Xt).cuda(), 0.1, inv_L=0.0) as s:
        info = s.info()
        assert abs(info["L"] / (1 + 2e-3) - L) <= 1e-9 * L
        st = s.step(2)
        assert all(x["tau"] >= min(0.5, 0.5 * info["inv_L"]) for x in st)
    with pytest.raises(A.AccordError) as e:
        A.AccordSolver(torch.zeros((50, 40), dtype=torch.float32).cuda(), 0.1, inv_L=0.0)
    assert e.value.status == A.E_NUMERIC


@pytest.mark.parametrize("refine", ["block", "ff"])
def test_filter_path_beyond_4096_samples(refine, monkeypatch):
    """n = 5000 (ldk = 5056; the refine reads each X^T row in 5 float4 passes,
    the last partial): AUTO is the certified bf16 filter for any n (round 1
    fell back to BF16X3 above n = 4096); parity with the oracle, the float64
    refine and its float-float A-B variant."""
    _cuda()
    monkeypatch.setenv("ACCORD_REFINE", refine)
    from accord_inputs import Config
    cfg = Config(name="t_bign_p600_n5000_f32", p=600, n=5000, dtype="f32", structure="ba",
                 block=300, lambdas=(0.05,), T=8, graph_seed=61, sample_seed=62)
    pr = make_problem(cfg)
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    csr, stats, info = run_gpu(pr.Xt, 0.05, cfg.T, inv_L, A.GEMM_AUTO)
    assert info["gemm"] in (A.GEMM_BF16_FILTER, A.GEMM_I8_FILTER) and info["ldk"] == 5056
    compare_full(pr.Xt, 0.05, cfg.T, inv_L, csr.to_dense(cfg.p), stats, "f32")


@pytest.mark.parametrize("spmm", ["tma", "plain"])
def test_bitwise_reproducible(spmm, monkeypatch):
    """Race check by repetition (compute-sanitizer is closed on this pool):
    every kernel reduces in a fixed order, so three runs of the same problem
    must agree bitwise -- iterates, objective trace, tau schedule and the
    candidate counts. A race in the warp-specialised GEMM pipeline (mbarrier
    / TMA / TMEM), the TMA SpMM ring, the hub-row split reductions or the
    chunked pool compaction would show up as run-to-run differences."""
    _cuda()
    monkeypatch.setenv("ACCORD_SPMM_TMA" if spmm == "tma" else "ACCORD_SPMM_PLAIN", "1")
    pr = make_problem("t_hubs_f32")
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    runs = []
    for _ in range(3):
        csr, stats, _ = run_gpu(pr.Xt, 0.05, 12, inv_L, A.GEMM_AUTO)
        runs.append((csr, [(x["tau"], x["f"], x["n_cand"], x["nnz"]) for x in stats]))
    for csr, st in runs[1:]:
        assert st == runs[0][1]
        assert np.array_equal(csr.row_ptr, runs[0][0].row_ptr)
        assert np.array_equal(csr.col, runs[0][0].col)
        assert np.array_equal(csr.val, runs[0][0].val)


@pytest.mark.parametrize("cols", ["4", "8"])
def test_spmm_parallel_producer_issue_is_bitwise(cols, monkeypatch):
    """The TMA SpMM's warp-parallel producer issue (every kept entry of a
    32-entry batch fills its own ring stage in one round, up to `stages` per
    round) stages the same X^T rows in the same order as the serial producer
    (ACCORD_SPMM_SERIAL=1), so the sums are bitwise the same: equal iterates,
    tau schedule and objective on a problem with hub rows and short rows,
    with rings shallower than a batch (2 and 4 stages: several issue rounds
    per batch, wrapping the ring) and a deep one."""
    _cuda()
    monkeypatch.setenv("ACCORD_SPMM_TMA", "1")
    monkeypatch.setenv("ACCORD_SPMM_COLS", cols)
    pr = make_problem("t_hubs_f32")
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    runs = []
    for serial, stages in (("1", "8"), ("0", "8"), ("0", "2"), ("0", "4"), ("0", "16")):
        monkeypatch.setenv("ACCORD_SPMM_SERIAL", serial)
        monkeypatch.setenv("ACCORD_SPMM_STAGES", stages)
        csr, stats, _ = run_gpu(pr.Xt, 0.05, 12, inv_L, A.GEMM_AUTO)
        runs.append((csr, [(x["tau"], x["f"], x["n_cand"], x["nnz"]) for x in stats]))
    c0, s0 = runs[0]
    for c1, s1 in runs[1:]:
        assert s0 == s1
        assert np.array_equal(c0.row_ptr, c1.row_ptr) and np.array_equal(c0.col, c1.col)
        assert np.array_equal(c0.val, c1.val)


def test_warm_start_roundtrip():
    _cuda()
    pr = make_problem("t_ba_f64")
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    X = torch.from_numpy(pr.Xt).cuda()
    with A.AccordSolver(X, 0.1, inv_L=inv_L, gemm=A.GEMM_SIMT) as s:
        s.step(4)
        mid = s.export_csr()
        s.step(3)
        end = s.export_csr()
    with A.AccordSolver(X, 0.1, inv_L=inv_L, gemm=A.GEMM_SIMT) as s2:
        s2.set_omega_csr(mid.row_ptr, mid.col, mid.val)
        s2.step(3)
        end2 = s2.export_csr()
    assert np.array_equal(end.col, end2.col) and np.allclose(end.val, end2.val, rtol=0,
                                                              atol=1e-13)


def test_errors_are_loud():
    _cuda()
    X = torch.zeros((10, 5), dtype=torch.float32).cuda()
    with pytest.raises(A.AccordError):
        A.AccordSolver(X, -1.0)
    Xn = torch.ones((10, 5), dtype=torch.float32)
    Xn[3, 2] = float("nan")
    with pytest.raises(A.AccordError) as e:
        A.AccordSolver(Xn.cuda(), 0.1)
    assert "row 3, col 2" in str(e.value)


@pytest.mark.parametrize("p,n,lam,T", [(4000, 60, 0.05, 2), (17000, 40, 0.02, 1)])
def test_parity_dense_candidate_rows(p, n, lam, T):
    """Rows with thousands (block bitonic) and > 16384 (runs + merge path)
    candidates: small n makes |S_ik| > lambda for most pairs."""
    _cuda()
    from accord_inputs import Config
    cfg = Config(name=f"dense_p{p}", p=p, n=n, dtype="f32", structure="ba", block=p // 4,
                 lambdas=(lam,), T=T, graph_seed=61, sample_seed=62)
    pr = make_problem(cfg)
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    csr, stats, info = run_gpu(pr.Xt, lam, T, inv_L, A.GEMM_AUTO)
    assert stats[-1]["max_row_cand"] > (16384 if p > 16384 else 1024)
    compare_full(pr.Xt, lam, T, inv_L, csr.to_dense(p), stats, "f32")


@pytest.mark.parametrize("cols", ["4", "8"])
@pytest.mark.parametrize("p,n,lam,T", [(4000, 60, 0.05, 3), (1100, 333, 0.1, 8)])
def test_tma_spmm_matches_block_per_row_spmm(p, n, lam, T, cols, monkeypatch):
    """The TMA-staged SpMM (producer warp + cp.async.bulk ring, hub rows split
    into work items with a deterministic last-block sum) and the block-per-row
    SpMM compute the same Y+ and D (both float64-accumulated): identical tau
    schedule, objective and Omega to rounding, on a case whose candidate rows
    exceed one work item (2048 entries)."""
    _cuda()
    monkeypatch.setenv("ACCORD_SPMM_COLS", cols)    # columns per consumer thread
    rng = np.random.default_rng(5 + p)
    Xt = rng.standard_normal((p, n)).astype(np.float32)
    Xt -= Xt.mean(axis=1, keepdims=True)
    inv_L = 1.0 / O.spectral_bound(Xt.astype(np.float64))
    out = {}
    for plain in (False, True):
        if plain:
            monkeypatch.setenv("ACCORD_SPMM_PLAIN", "1")
            monkeypatch.delenv("ACCORD_SPMM_TMA", raising=False)
        else:
            monkeypatch.delenv("ACCORD_SPMM_PLAIN", raising=False)
            monkeypatch.setenv("ACCORD_SPMM_TMA", "1")   # small p: force the TMA path
        with A.AccordSolver(torch.from_numpy(Xt).cuda(), lam, inv_L=inv_L) as s:
            st = s.step(T)
            out[plain] = ([x["tau"] for x in st], [x["f"] for x in st], s.export_csr(),
                          max(x["max_row_cand"] for x in st))
    (t0, f0, c0, m0), (t1, f1, c1, m1) = out[False], out[True]
    assert t0 == t1
    np.testing.assert_allclose(f0, f1, rtol=1e-12)
    assert np.array_equal(c0.row_ptr, c1.row_ptr) and np.array_equal(c0.col, c1.col)
    assert np.abs(c0.val - c1.val).max() <= 1e-6 * np.abs(c1.val).max()
    if p == 4000:
        assert m0 > 2048   # multi-item rows were exercised


@pytest.mark.parametrize("gemm", [A.GEMM_SIMT, A.GEMM_BF16X3, A.GEMM_BF16_FILTER])
@pytest.mark.parametrize("p,n,lam", [(1, 7, 0.1), (2, 1, 0.3), (3, 5, 0.2), (257, 65, 0.05),
                                     (5, 300, 0.0)])
def test_degenerate_and_ragged_shapes(p, n, lam, gemm):
    """Edge cases of the method and of the tiling: p = 1 (Omega is the single
    diagonal root), n = 1 (rank-one S), lambda = 0 with n > p
    (no shrinkage), one more row/column than a 256 tile and one more sample
    than a 64-sample K block, against the oracle."""
    _cuda()
    rng = np.random.default_rng(1000 * p + n)
    Xt = rng.standard_normal((p, n))
    if n > 1:
        Xt -= Xt.mean(axis=1, keepdims=True)
    Xt = Xt.astype(np.float32)
    inv_L = 1.0 / max(O.spectral_bound(Xt.astype(np.float64)), 1e-12)
    T = 6
    csr, stats, info = run_gpu(Xt, lam, T, inv_L, gemm)
    assert info["gemm"] == gemm
    compare_full(Xt, lam, T, inv_L, csr.to_dense(p), stats, "f32")
    if p == 1:
        # converged, the single entry is the closed form (-lam + sqrt(lam^2 + 4s)) / (2s)
        s = float(Xt[0].astype(np.float64) @ Xt[0].astype(np.float64)) / n
        w_hat = (-lam + np.sqrt(lam ** 2 + 4 * s)) / (2 * s)
        X1 = torch.from_numpy(Xt).cuda()
        with A.AccordSolver(X1, lam, inv_L=inv_L, gemm=gemm) as sv:
            sv.solve(max_iter=500, tol=1e-9)
            c1 = sv.export_csr()
        assert c1.col.tolist() == [0]
        assert abs(c1.val[0] - w_hat) <= 1e-6 * w_hat


def test_empty_rank_block_rejected_and_bad_params():
    _cuda()
    X = torch.ones((8, 4), dtype=torch.float32).cuda()
    with pytest.raises(A.AccordError):
        A.AccordSolver(X, 0.1, row_begin=4, row_end=4)      # empty row block
    with pytest.raises(A.AccordError):
        A.AccordSolver(X, 0.1, tau0=0.0)
    with pytest.raises(A.AccordError):
        A.AccordSolver(X, 0.1, beta=1.5)
    with pytest.raises(A.AccordError):
        A.AccordSolver(X.double(), 0.1, gemm=A.GEMM_BF16_FILTER)   # tensor cores need F32


@pytest.mark.parametrize("p,n,lam,T", [(4000, 60, 0.05, 4), (1100, 333, 0.1, 10)])
def test_paired_line_search_is_bitwise_sequential(p, n, lam, T, monkeypatch):
    """Paired trials (one gather pass evaluates tau and beta*tau) take exactly
    the sequential decisions of Algorithm 1: same tau
    schedule, trial counts and bitwise-identical iterates."""
    _cuda()
    rng = np.random.default_rng(17 + p)
    Xt = rng.standard_normal((p, n)).astype(np.float32)
    Xt -= Xt.mean(axis=1, keepdims=True)
    inv_L = 1.0 / O.spectral_bound(Xt.astype(np.float64))
    monkeypatch.setenv("ACCORD_SPMM_TMA", "1")
    out = {}
    for pairs in ("1", "0"):
        monkeypatch.setenv("ACCORD_LS_PAIRS", pairs)
        with A.AccordSolver(torch.from_numpy(Xt).cuda(), lam, inv_L=inv_L, tau0=4.0) as s:
            st = s.step(T)
            out[pairs] = ([(x["tau"], x["trials"], x["f"]) for x in st], s.export_csr())
    (s1, c1), (s0, c0) = out["1"], out["0"]
    assert s1 == s0
    assert max(t for _, t, _ in s1) >= 2          # rejected trials were exercised
    assert np.array_equal(c1.row_ptr, c0.row_ptr) and np.array_equal(c1.col, c0.col)
    assert np.array_equal(c1.val, c0.val)


@pytest.mark.parametrize("p,n,lam,T", [(4000, 60, 0.3, 3), (700, 250, 0.1, 3), (257, 65, 0.08, 3),
                                       (1100, 333, 0.02, 2)])
def test_symmetric_first_gemm_matches_full(p, n, lam, T, monkeypatch):
    """At Omega^(0) = I the gradient is S = X^T X / n (symmetric; PAPER.md:54-57,
    Alg. 1 at t = 0), so the first GEMM runs only the tiles on and above the
    diagonal and mirrors each filter survivor. The candidate set is a
    different certified superset, the refine recomputes every value exactly,
    so the iterates, tau schedule and objective are bitwise those of the full
    GEMM (ACCORD_GEMM_NOSYM=1); ragged p (not a multiple of 256) included.
    The refine of that C gathers only the entries k >= i and copies the rest
    from their twins (C = C^T; the float64 dot product of exact f32 products
    in a fixed order is symmetric bitwise); a twin the filter did not emit is
    recomputed, which ACCORD_DEBUG_MIRROR_MISS forces for every entry.
    (Rows stay below one work item, 2048 candidates, so the extra zero-valued
    candidates cannot regroup any partial sum.)"""
    _cuda()
    rng = np.random.default_rng(29 + p)
    Xt = rng.standard_normal((p, n)).astype(np.float32)
    Xt[1::3] += 0.6 * Xt[0::3][: Xt[1::3].shape[0]]      # correlated pairs: real off-diagonals
    Xt -= Xt.mean(axis=1, keepdims=True)
    inv_L = 1.0 / O.spectral_bound(Xt.astype(np.float64))
    out = {}
    modes = {"sym": {}, "miss": {"ACCORD_DEBUG_MIRROR_MISS": "1"},
             "refine_nosym": {"ACCORD_REFINE_NOSYM": "1"}, "nosym": {"ACCORD_GEMM_NOSYM": "1"}}
    for mode, env in modes.items():
        for k in ("ACCORD_DEBUG_MIRROR_MISS", "ACCORD_REFINE_NOSYM", "ACCORD_GEMM_NOSYM"):
            if k in env:
                monkeypatch.setenv(k, env[k])
            else:
                monkeypatch.delenv(k, raising=False)
        with A.AccordSolver(torch.from_numpy(Xt).cuda(), lam, inv_L=inv_L,
                            gemm=A.GEMM_BF16_FILTER) as s:
            st = s.step(T)
            out[mode] = ([(x["tau"], x["trials"], x["f"], x["nnz"]) for x in st],
                         st[0]["n_cand"], s.export_csr())
    for mode in ("miss", "refine_nosym"):
        s_, nc_, c_ = out[mode]
        assert s_ == out["sym"][0] and nc_ == out["sym"][1], mode
        assert np.array_equal(c_.col, out["sym"][2].col), mode
        assert np.array_equal(c_.val, out["sym"][2].val), mode
    (s1, nc1, c1), (s0, nc0, c0) = out["sym"], out["nosym"]
    assert s1 == s0
    assert s1[0][3] > p                          # off-diagonal support after iteration 1
    assert nc1 >= s1[0][3] and nc0 >= s0[0][3]
    assert np.array_equal(c1.row_ptr, c0.row_ptr) and np.array_equal(c1.col, c0.col)
    assert np.array_equal(c1.val, c0.val)


@pytest.mark.parametrize("p,n,lam,tau0", [(1100, 333, 0.05, 4.0), (700, 250, 0.1, 0.5),
                                          (4000, 60, 0.3, 1.0)])
def test_first_iteration_line_search_from_identity(p, n, lam, tau0, monkeypatch):
    """From Omega^(0) = I every trial of iteration 1 is
    Y+_i = a_i(tau) x_i + tau z_i with one SpMM z = S_lam(-G) X^T (exact for
    power-of-two tau, Eq. 3.5). Against the per-trial SpMM passes
    (ACCORD_LS_NODIAG=1): the same tau schedule and trial counts; objective
    and iterates equal to f32 rounding (z is stored in f32 before the
    expansion, the plain pass rounds Y+ once from float64 accumulators, and
    the later iterations start from Y that differ in the last bit)."""
    _cuda()
    rng = np.random.default_rng(41 + p)
    Xt = rng.standard_normal((p, n)).astype(np.float32)
    Xt[1::3] += 0.6 * Xt[0::3][: Xt[1::3].shape[0]]
    Xt -= Xt.mean(axis=1, keepdims=True)
    inv_L = 1.0 / O.spectral_bound(Xt.astype(np.float64))
    out = {}
    for nodiag in ("0", "1"):
        if nodiag == "1":
            monkeypatch.setenv("ACCORD_LS_NODIAG", "1")
        else:
            monkeypatch.delenv("ACCORD_LS_NODIAG", raising=False)
        with A.AccordSolver(torch.from_numpy(Xt).cuda(), lam, inv_L=inv_L, tau0=tau0,
                            gemm=A.GEMM_BF16_FILTER) as s:
            st = s.step(4)
            out[nodiag] = ([(x["tau"], x["trials"]) for x in st], [x["f"] for x in st],
                           s.export_csr(), s.export_csr().to_dense(p))
    (s1, f1, c1, d1), (s0, f0, c0, d0) = out["0"], out["1"]
    assert s1 == s0
    assert s1[0][1] >= 2 or tau0 <= 1.0          # rejected trials exercised where tau0 is large
    np.testing.assert_allclose(f1, f0, rtol=1e-8, atol=0)
    assert abs(len(c1.col) - len(c0.col)) <= max(2, len(c0.col) // 10000)
    assert np.abs(d1 - d0).max() <= 1e-6 * np.abs(d0).max()
