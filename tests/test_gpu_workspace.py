"""Caller-owned device memory (SURVEY.md §8(b) workspace query; VERDICT r1
item 5): accord_workspace_size + a torch-allocated workspace in which every
device buffer of the context lives. The inputs are Alg. 1's;
no paper passage governs memory."""
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


def _run(X, lam, T, inv_L, **kw):
    with A.AccordSolver(X, lam, inv_L=inv_L, **kw) as s:
        st = s.step(T)
        return s.export_csr(), st, s.info()


@pytest.mark.parametrize("host_x", [False, True])
def test_config2_runs_inside_a_torch_workspace(host_x):
    """BASELINE config 2 (100 iterations) in a workspace of exactly
    accord_workspace_size bytes: bitwise the run with library-allocated
    memory, no device allocation by the library (free memory does not move
    beyond the module's lazily loaded code), high-water within the query."""
    _cuda()
    pr = make_problem(2)
    lam = 0.1
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    X = torch.from_numpy(pr.Xt)
    X = X if host_x else X.cuda()
    ref, st_ref, _ = _run(X, lam, 100, inv_L)
    need = A.workspace_size(X, lam, inv_L=inv_L)
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    csr, st, info = _run(X, lam, 100, inv_L, workspace=ws)
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 < (64 << 20), (free0 - free1)      # nothing taken from the device
    assert info["workspace_bytes"] <= need and 0 < info["workspace_high"] <= need
    assert [x["tau"] for x in st] == [x["tau"] for x in st_ref]
    assert np.array_equal(csr.row_ptr, ref.row_ptr) and np.array_equal(csr.col, ref.col)
    assert np.array_equal(csr.val, ref.val)


def test_workspace_too_small_and_pool_overflow_are_capacity_errors():
    """Half the queried size: create fails with ACCORD_E_CAPACITY. A pool of
    p entries (the first GEMM needs far more) in an exactly sized workspace:
    the step fails with ACCORD_E_CAPACITY and the bytes needed, nothing is
    committed (Omega = I and f(I) intact); with room to grow inside the
    workspace the same run succeeds and equals the default run."""
    _cuda()
    pr = make_problem("t_mid_f32")
    c = pr.cfg
    lam = 0.1
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    X = torch.from_numpy(pr.Xt).cuda()
    need = A.workspace_size(X, lam, inv_L=inv_L)
    with pytest.raises(A.AccordError) as e:
        A.AccordSolver(X, lam, inv_L=inv_L,
                       workspace=torch.empty(need // 2, dtype=torch.uint8, device="cuda"))
    assert e.value.status == A.E_CAPACITY
    small = A.workspace_size(X, lam, inv_L=inv_L, cand_capacity=c.p)
    ws = torch.empty(small, dtype=torch.uint8, device="cuda")
    with A.AccordSolver(X, lam, inv_L=inv_L, cand_capacity=c.p, workspace=ws) as s:
        f0 = s.objective()[0]
        with pytest.raises(A.AccordError) as e:
            s.step(1)
        assert e.value.status == A.E_CAPACITY and "more bytes needed" in str(e.value)
        assert s.objective()[0] == f0 and s.info()["iterations"] == 0
        I = s.export_csr()
        assert np.array_equal(I.row_ptr, np.arange(c.p + 1)) and np.all(I.val == 1)
    ref, st_ref, _ = _run(X, lam, 5, inv_L)
    big = torch.empty(need + (256 << 20), dtype=torch.uint8, device="cuda")
    csr, st, info = _run(X, lam, 5, inv_L, cand_capacity=c.p, workspace=big)
    assert [x["tau"] for x in st] == [x["tau"] for x in st_ref]
    assert np.array_equal(csr.col, ref.col) and np.array_equal(csr.val, ref.val)
    assert info["cand_capacity"] > c.p          # grew inside the workspace


def test_workspace_with_next_rows():
    """The NEXT calls that allocate temporaries (lambda_max, refit, KKT,
    transformed export, path) run inside the workspace when it has room."""
    _cuda()
    pr = make_problem("t_ba_f32")
    lam = 0.1
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    X = torch.from_numpy(pr.Xt).cuda()
    need = A.workspace_size(X, lam, inv_L=inv_L)
    ws = torch.empty(need + (64 << 20), dtype=torch.uint8, device="cuda")
    with A.AccordSolver(X, lam, inv_L=inv_L, workspace=ws) as s:
        lm = s.lambda_max()
        s.step(10)
        th = s.export_transformed(A.EXPORT_PCORR)
        k = s.kkt_residual()
        s.refit(0.0)
        s.step(3)
        info = s.info()
    assert abs(lm - O.lambda_max(pr.Xt)) <= 1e-12 * lm
    assert len(th.col) > 0 and np.isfinite(k)
    assert info["workspace_high"] <= info["workspace_bytes"]
