"""Multi-rank logic.

CPU (-m "not gpu"): world_size-2 gloo processes exercise the host
communicator (the 8-double line-search allreduce and the CSR gather blob
exchange) and the row partition; a 3-thread ThreadComm does the same in one
process.

GPU (-m gpu): P contexts on ONE GPU, each driven by its own host thread with
ThreadComm (the kernels never wait on each other; the host threads meet at a
barrier), must reproduce the P = 1 run: identical tau schedule and Omega.
"""
import os
import socket
import threading

import numpy as np
import pytest

import paper_2412_11554_b200 as A
from paper_2412_11554_b200.comm import ThreadComm


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, q):
    import ctypes as C
    import torch.distributed as dist
    from paper_2412_11554_b200.comm import TorchDistComm
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchDistComm()
        # line-search sums: every rank must see the same totals
        buf = (C.c_double * 8)(*[rank + 1.0 + k for k in range(8)])
        assert comm.allreduce(None, buf, 8) == 0
        tot = list(buf)
        # CSR block gather: rank r contributes r+1 bytes of value r
        mine = (C.c_uint8 * (rank + 1))(*([rank] * (rank + 1)))
        counts = (C.c_int64 * world)()
        assert comm.allgatherv(None, C.addressof(mine), rank + 1, None, counts) == 0
        out = (C.c_uint8 * sum(counts))()
        assert comm.allgatherv(None, C.addressof(mine), rank + 1, C.addressof(out), counts) == 0
        # row partition is identical on every rank and covers p
        parts = A.partition_rows(100000, world)
        q.put((rank, tot, list(counts), list(out), parts))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_host_comm_and_partition():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    want = [(1.0 + k) + (2.0 + k) for k in range(8)]
    for rank, tot, counts, out, parts in res:
        assert tot == want
        assert counts == [1, 2]
        assert out == [0, 1, 1]
        assert parts == res[0][4] and parts[0][0] == 0 and parts[-1][1] == 100000


def test_thread_comm_three_ranks():
    import ctypes as C
    P = 3
    comm = ThreadComm(P)
    results = [None] * P

    def run(r):
        comm.bind(r)
        buf = (C.c_double * 4)(*[float(r * 10 + k) for k in range(4)])
        assert comm.allreduce(None, buf, 4) == 0
        mine = (C.c_uint8 * 2)(r, r)
        counts = (C.c_int64 * P)()
        comm.allgatherv(None, C.addressof(mine), 2, None, counts)
        out = (C.c_uint8 * 6)()
        comm.allgatherv(None, C.addressof(mine), 2, C.addressof(out), counts)
        results[r] = (list(buf), list(counts), list(out))

    th = [threading.Thread(target=run, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for buf, counts, out in results:
        assert buf == [0 + 10 + 20 + 3 * k for k in range(4)]
        assert counts == [2, 2, 2] and out == [0, 0, 1, 1, 2, 2]


# ----------------------------------------------------------------- GPU -----
def run_ranks(Xt, lam, T, inv_L, P, gemm, align=256, infos=None):
    import torch
    comm = ThreadComm(P)
    bounds = A.partition_rows(Xt.shape[0], P, align=align)
    X = torch.from_numpy(Xt).cuda()
    out = [None] * P
    errs = []

    def run(r):
        try:
            comm.bind(r)
            stream = torch.cuda.Stream()
            s = A.AccordSolver(X, lam, inv_L=inv_L, gemm=gemm, row_begin=bounds[r][0],
                               row_end=bounds[r][1], rank=r, world=P, comm=A.COMM_HOST,
                               allreduce=comm.allreduce, allgatherv=comm.allgatherv,
                               stream=stream)
            st = s.step(T)
            g = s.export_csr(A.SCOPE_GATHER)
            loc = s.export_csr(A.SCOPE_LOCAL)
            f = s.objective()[0]
            if infos is not None:
                infos[r] = s.info()
            s.close()
            out[r] = (st, g, loc, f)
        except Exception as e:      # surface in the main thread
            errs.append(e)
            comm.barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return out, bounds


@pytest.mark.gpu
@pytest.mark.parametrize("gemm", [A.GEMM_SIMT, A.GEMM_BF16_FILTER, A.GEMM_I8_FILTER, A.GEMM_AUTO])
def test_p_invariance_one_gpu(gemm):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA not available on a -m gpu run")
    from accord_inputs import make_problem
    from oracle import accord_oracle as O
    pr = make_problem("t_hubs_f32")
    c = pr.cfg
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    ref, _ = run_ranks(pr.Xt, c.lambdas[0], c.T, inv_L, 1, gemm)
    taus1 = [s["tau"] for s in ref[0][0]]
    W1 = ref[0][1].to_dense(c.p)
    for P, align in [(2, 256), (3, 1), (4, 256), (8, 1)]:   # P in {1, 2, 4, 8}
        out, bounds = run_ranks(pr.Xt, c.lambdas[0], c.T, inv_L, P, gemm, align)
        for r in range(P):
            st, g, loc, f = out[r]
            assert [s["tau"] for s in st] == taus1          # identical decisions
            assert abs(f - ref[0][3]) <= 1e-9 * abs(f)
            Wg = g.to_dense(c.p)                            # every rank gathers all rows
            assert np.abs(Wg - W1).max() <= 1e-6 * np.abs(W1).max()
            b, e = bounds[r]
            assert np.array_equal(loc.to_dense(c.p), Wg[b:e])


@pytest.mark.gpu
def test_mixed_block_sizes_agree_on_the_spmm_kind():
    """p = 131,000, P = 2: rank 0's block (65,536 rows) qualifies for the TMA
    SpMM with paired line-search passes, rank 1's (65,464) alone would not.
    The ranks must run the same passes (each ends in an allreduce of 8 or 16
    sums), so create agrees on one kind; the run equals P = 1 (decisions, f,
    gathered Omega)."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA not available on a -m gpu run")
    from accord_inputs import Config, make_problem
    cfg = Config(name="t_mixed_p131000_n256_f32", p=131000, n=256, dtype="f32", structure="ba",
                 block=1000, lambdas=(0.35,), T=4, graph_seed=71, sample_seed=72)
    pr = make_problem(cfg)
    b = A.partition_rows(cfg.p, 2)
    assert b[0][1] - b[0][0] >= 65536 > b[1][1] - b[1][0]
    ref, _ = run_ranks(pr.Xt, 0.35, cfg.T, 0.0, 1, A.GEMM_BF16_FILTER)
    out, bounds = run_ranks(pr.Xt, 0.35, cfg.T, 0.0, 2, A.GEMM_BF16_FILTER)
    for r in range(2):
        st, g, loc, f = out[r]
        assert [x["tau"] for x in st] == [x["tau"] for x in ref[0][0]]
        assert [x["trials"] for x in st] == [x["trials"] for x in ref[0][0]]
        assert abs(f - ref[0][3]) <= 1e-9 * abs(f)
        assert np.array_equal(g.row_ptr, ref[0][1].row_ptr) and np.array_equal(g.col, ref[0][1].col)
        assert np.abs(g.val - ref[0][1].val).max() <= 1e-6 * np.abs(ref[0][1].val).max()


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 3, 4])
def test_symmetric_first_gemm_across_ranks(P, monkeypatch):
    """At Omega = I several ranks run the cyclic half of the symmetric GEMM
    (each unordered pair of 256-tiles once, ~half of every rank's tiles) and
    send the mirrored candidate positions of other ranks' rows to their owner
    (host transport here; NCCL send/recv in production). The run equals the
    P = 1 run and the P-rank run without the symmetric schedule."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA not available on a -m gpu run")
    from accord_inputs import make_problem
    from oracle import accord_oracle as O
    pr = make_problem("t_mid_f32")          # p = 3000: 12 tiles, blocks on tile boundaries
    c = pr.cfg
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    ref, _ = run_ranks(pr.Xt, c.lambdas[0], 6, inv_L, 1, A.GEMM_BF16_FILTER)
    infos = [None] * P
    out, bounds = run_ranks(pr.Xt, c.lambdas[0], 6, inv_L, P, A.GEMM_BF16_FILTER, infos=infos)
    assert all(b % 256 == 0 for b, _ in bounds)
    assert sum(i["mirrored_sent"] for i in infos) > 0          # the exchange ran
    monkeypatch.setenv("ACCORD_GEMM_NOSYM", "1")
    full, _ = run_ranks(pr.Xt, c.lambdas[0], 6, inv_L, P, A.GEMM_BF16_FILTER)
    W1 = ref[0][1].to_dense(c.p)
    for r in range(P):
        for run in (out, full):
            st, g, loc, f = run[r]
            assert [x["tau"] for x in st] == [x["tau"] for x in ref[0][0]]
            assert abs(f - ref[0][3]) <= 1e-9 * abs(f)
            Wg = g.to_dense(c.p)
            assert np.array_equal(Wg != 0, W1 != 0)
            assert np.abs(Wg - W1).max() <= 1e-6 * np.abs(W1).max()
    # the schedule is the symmetric one: iteration 1's |C| equals the P = 1 run's
    # (the same certified rule from the mirrored side) within the filter slack
    n1 = ref[0][0][0]["n_cand"]
    assert abs(out[0][0][0]["n_cand"] - n1) <= 0.05 * n1


@pytest.mark.gpu
def test_transformed_exports_p_invariant_one_gpu():
    """NEXT(4) with P = 2 row blocks (ThreadComm): PCORR needs the transpose
    across ranks (gathered), THETA is rank-local; both must equal P = 1."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA not available on a -m gpu run")
    from accord_inputs import make_problem
    from oracle import accord_oracle as O
    pr = make_problem("t_hubs_f32")
    c = pr.cfg
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    X = torch.from_numpy(pr.Xt).cuda()
    T = 8
    res = {}
    for P in (1, 2):
        comm = ThreadComm(P)
        bounds = A.partition_rows(c.p, P, align=1)
        out = [None] * P
        errs = []

        def run(r):
            try:
                comm.bind(r)
                s = A.AccordSolver(X, c.lambdas[0], inv_L=inv_L, row_begin=bounds[r][0],
                                   row_end=bounds[r][1], rank=r, world=P, comm=A.COMM_HOST,
                                   allreduce=comm.allreduce, allgatherv=comm.allgatherv,
                                   stream=torch.cuda.Stream())
                s.step(T)
                got = {}
                for kind in (A.EXPORT_THETA, A.EXPORT_PCORR):
                    for sc in (A.SCOPE_LOCAL, A.SCOPE_GATHER):
                        got[(kind, sc)] = s.export_transformed(kind, sc)
                out[r] = got
                s.close()
            except Exception as e:
                errs.append(e)
                comm.barrier.abort()

        th = [threading.Thread(target=run, args=(r,)) for r in range(P)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if errs:
            raise errs[0]
        res[P] = (out, bounds)
    one = res[1][0][0]
    for kind in (A.EXPORT_THETA, A.EXPORT_PCORR):
        full = one[(kind, A.SCOPE_GATHER)].to_dense(c.p)
        out, bounds = res[2]
        for r in range(2):
            g = out[r][(kind, A.SCOPE_GATHER)].to_dense(c.p)
            assert np.abs(g - full).max() <= 1e-6 * max(1.0, np.abs(full).max())
            b, e = bounds[r]
            loc = out[r][(kind, A.SCOPE_LOCAL)]
            assert loc.row_begin == b
            assert np.array_equal(loc.to_dense(c.p), g[b:e])


def test_thread_comm_sendrecv_ring():
    """The ring exchange of the sharded-X mode (NEXT(3)): rank r sends its
    block to r-1 and receives r+1's; blocks of different sizes."""
    import ctypes as C
    P = 3
    comm = ThreadComm(P)
    results = [None] * P

    def run(r):
        comm.bind(r)
        mine = (C.c_uint8 * (r + 2))(*([r] * (r + 2)))
        src = (r + 1) % P
        got = (C.c_uint8 * (src + 2))()
        rc = comm.sendrecv(None, C.addressof(mine), r + 2, (r - 1) % P, C.addressof(got),
                           src + 2, src)
        results[r] = (rc, list(got))

    th = [threading.Thread(target=run, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for r, (rc, got) in enumerate(results):
        src = (r + 1) % P
        assert rc == 0 and got == [src] * (src + 2)


def _gloo_ring_worker(rank, world, port, q):
    import ctypes as C
    import torch.distributed as dist
    from paper_2412_11554_b200.comm import TorchDistComm
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchDistComm()
        src = (rank + 1) % world
        mine = (C.c_uint8 * (rank + 3))(*([rank + 7] * (rank + 3)))
        got = (C.c_uint8 * (src + 3))()
        rc = comm.sendrecv(None, C.addressof(mine), rank + 3, (rank - 1) % world,
                           C.addressof(got), src + 3, src)
        q.put((rank, rc, list(got)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sendrecv_ring():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_ring_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, rc, got in res:
        src = (rank + 1) % 2
        assert rc == 0 and got == [src + 7] * (src + 3)


def run_ranks_sharded(Xt, lam, T, inv_L, P, gemm, layout="variables", extra=None):
    """P ranks on one GPU, each holding only its slab of X (x_sharded)."""
    import torch
    comm = ThreadComm(P)
    p = Xt.shape[0]
    bounds = A.partition_rows(p, P)
    out = [None] * P
    errs = []

    def run(r):
        try:
            comm.bind(r)
            b, e = bounds[r]
            slab = np.ascontiguousarray(Xt[b:e] if layout == "variables" else Xt[b:e].T)
            s = A.AccordSolver(torch.from_numpy(slab).cuda(), lam, layout=layout, inv_L=inv_L,
                               gemm=gemm, row_begin=b, row_end=e, rank=r, world=P,
                               comm=A.COMM_HOST, allreduce=comm.allreduce,
                               allgatherv=comm.allgatherv, sendrecv=comm.sendrecv,
                               x_sharded=True, p_global=p, stream=torch.cuda.Stream())
            st = s.step(T)
            res = {"st": st, "g": s.export_csr(A.SCOPE_GATHER), "f": s.objective()[0],
                   "L": s.info()["L"]}
            if extra:
                res.update(extra(s))
            s.close()
            out[r] = res
        except Exception as ex:
            errs.append(ex)
            comm.barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return out, bounds


@pytest.mark.gpu
@pytest.mark.parametrize("key,gemm", [("t_ba_f64", A.GEMM_SIMT), ("t_hubs_f32", A.GEMM_SIMT),
                                      ("t_hubs_f32", A.GEMM_BF16_FILTER),
                                      ("t_hubs_f32", A.GEMM_BF16X3)])
def test_sharded_x_ring_matches_replicated(key, gemm):
    """NEXT(3): X split by variables over P ranks, every pass over X done as a
    ring of slab exchanges (Alg. 2), must reproduce the replicated P = 1 run:
    identical tau schedule, Omega within rounding (the SpMM sums the slabs in
    ring order, in float64), and the oracle within the parity bar."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA not available on a -m gpu run")
    from accord_inputs import make_problem
    from oracle import accord_oracle as O
    pr = make_problem(key)
    c = pr.cfg
    lam = c.lambdas[0]
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    ref, _ = run_ranks(pr.Xt, lam, c.T, inv_L, 1, gemm)
    taus1 = [s["tau"] for s in ref[0][0]]
    W1 = ref[0][1].to_dense(c.p)
    orc = O.fbs(pr.Xt, lam, c.tau0, c.beta, inv_L, T=c.T)
    f64 = c.dtype == "f64"
    for P in (2, 3) if c.p >= 768 else (2,):
        out, bounds = run_ranks_sharded(pr.Xt, lam, c.T, inv_L, P, gemm)
        for r in range(P):
            o = out[r]
            assert [s["tau"] for s in o["st"]] == taus1
            assert abs(o["f"] - ref[0][3]) <= (1e-12 if f64 else 1e-9) * abs(o["f"])
            W = o["g"].to_dense(c.p)
            assert np.abs(W - W1).max() <= (1e-12 if f64 else 1e-6) * np.abs(W1).max()
            assert np.array_equal(W != 0, W1 != 0) or not f64
            assert np.abs(W - orc["Omega"]).max() <= (1e-10 if f64 else 1e-5) * \
                np.abs(orc["Omega"]).max()


@pytest.mark.gpu
def test_sharded_x_power_iteration_refit_kkt_and_layout():
    """Sharded mode end to end: L by the sharded Lanczos iteration (allreduce of
    X v), samples-major slabs, refit (refine ring) and the KKT certificate."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA not available on a -m gpu run")
    from accord_inputs import make_problem
    from oracle import accord_oracle as O
    pr = make_problem("t_hubs_f32")
    c = pr.cfg
    lam = c.lambdas[0]

    def extra(s):
        kkt = s.kkt_residual()
        s.refit(0.0)
        st2 = s.step(5)
        return {"kkt": kkt, "st2": st2, "g2": s.export_csr(A.SCOPE_GATHER)}

    # reference: replicated single context, same calls
    X = torch.from_numpy(pr.Xt).cuda()
    with A.AccordSolver(X, lam, inv_L=0.0) as s:
        st = s.step(6)
        L1 = s.info()["L"]
        ref = {"st": st, **extra(s)}
    out, _ = run_ranks_sharded(pr.Xt, lam, 6, 0.0, 2, A.GEMM_AUTO, layout="samples", extra=extra)
    for o in out:
        assert abs(o["L"] - L1) <= 1e-9 * L1
        assert [x["tau"] for x in o["st"]] == [x["tau"] for x in ref["st"]]
        assert [x["tau"] for x in o["st2"]] == [x["tau"] for x in ref["st2"]]
        assert abs(o["kkt"] - ref["kkt"]) <= 1e-6 * max(1.0, ref["kkt"])
        W, Wr = o["g2"].to_dense(c.p), ref["g2"].to_dense(c.p)
        assert np.abs(W - Wr).max() <= 1e-6 * np.abs(Wr).max()


@pytest.mark.gpu
def test_sharded_x_ring_config3_scale():
    """Sharded ring at BASELINE config 3 scale (p = 20000, n = 1000, many GEMM
    tiles per slab, ragged last slab): P = 2 and 3 must reproduce the
    replicated run (tau schedule, objective, Omega)."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA not available on a -m gpu run")
    from accord_inputs import get_config, make_problem
    cfg = get_config("3")
    pr = make_problem(cfg, with_blocks=False)
    lam, T = cfg.lambdas[0], 6
    X = torch.from_numpy(pr.Xt).cuda()
    with A.AccordSolver(X, lam, inv_L=0.0) as s:
        st1 = s.step(T)
        W1 = s.export_csr()
        f1 = s.objective()[0]
        L1 = s.info()["L"]
    del X
    for P in (2, 3):
        out, bounds = run_ranks_sharded(pr.Xt, lam, T, 1.0 / L1, P, A.GEMM_AUTO)
        for o in out:
            assert [x["tau"] for x in o["st"]] == [x["tau"] for x in st1]
            assert abs(o["f"] - f1) <= 1e-9 * abs(f1)
            g = o["g"]
            assert np.array_equal(g.row_ptr, W1.row_ptr) and np.array_equal(g.col, W1.col)
            assert np.abs(g.val - W1.val).max() <= 1e-6 * np.abs(W1.val).max()


@pytest.mark.gpu
@pytest.mark.slow
def test_sharded_x_ring_config5_scale():
    """The sharded-X ring at the p = 1e6 config: 2 contexts on one GPU, each
    holding half of X (2 GB) and passing slabs through the host transport,
    reproduce the replicated run's tau schedule, objective and Omega for the
    first iterations (GEMM ring of 2 x 1954 x 1954 tiles, refine and SpMM
    rings, sharded Lanczos iteration)."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA not available on a -m gpu run")
    from accord_inputs import get_config, make_problem
    cfg = get_config("5")
    pr = make_problem(cfg, with_blocks=False)
    lam, T = cfg.lambdas[0], 2
    X = torch.from_numpy(pr.Xt).cuda()
    with A.AccordSolver(X, lam, inv_L=0.0) as s:
        st1 = s.step(T)
        W1 = s.export_csr()
        f1 = s.objective()[0]
        L1 = s.info()["L"]
    del X
    torch.cuda.empty_cache()
    out, bounds = run_ranks_sharded(pr.Xt, lam, T, 0.0, 2, A.GEMM_AUTO)
    for o in out:
        assert abs(o["L"] - L1) <= 1e-9 * L1
        assert [x["tau"] for x in o["st"]] == [x["tau"] for x in st1]
        # the replicated run uses the TMA SpMM (hub rows summed in chunk order),
        # the ring the block-per-row kernel (slabs in ring order): Y+ agrees to
        # f32 rounding, the objective to ~1e-8 relative
        assert abs(o["f"] - f1) <= 1e-7 * abs(f1)
        g = o["g"]
        assert np.array_equal(g.row_ptr, W1.row_ptr) and np.array_equal(g.col, W1.col)
        assert np.abs(g.val - W1.val).max() <= 1e-6 * np.abs(W1.val).max()


@pytest.mark.gpu
def test_nccl_code_path_with_one_rank():
    """The NCCL path of the library (dlopen'ed libnccl, CommInitRank, the
    per-trial AllReduce of the line-search sums, the KKT max-AllReduce, the
    Broadcast gather of the export) run for real on a 1-rank communicator and
    must reproduce the communicator-free run exactly."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA not available on a -m gpu run")
    from accord_inputs import make_problem
    from oracle import accord_oracle as O
    pr = make_problem("t_hubs_f32")
    c = pr.cfg
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    X = torch.from_numpy(pr.Xt).cuda()
    res = {}
    for comm in (A.COMM_NONE, A.COMM_NCCL):
        kw = dict(comm=comm, nccl_id=A.nccl_unique_id()) if comm == A.COMM_NCCL else {}
        with A.AccordSolver(X, c.lambdas[0], inv_L=inv_L, **kw) as s:
            st = s.step(c.T)
            res[comm] = ([(x["tau"], x["f"]) for x in st], s.export_csr(A.SCOPE_GATHER),
                         s.kkt_residual())
    (a, ca, ka), (b, cb, kb) = res[A.COMM_NONE], res[A.COMM_NCCL]
    assert a == b and ka == kb
    assert np.array_equal(ca.row_ptr, cb.row_ptr) and np.array_equal(ca.col, cb.col)
    assert np.array_equal(ca.val, cb.val)


@pytest.mark.gpu
def test_nccl_watchdog_gives_up_on_a_stalled_stream(monkeypatch):
    """Every host wait on a stream with NCCL work is a watchdog: with the
    stream held for 4 s (ACCORD_DEBUG_STALL_MS, a stand-in for a peer that
    never joins the allreduce) and ACCORD_NCCL_TIMEOUT_S = 1, the step gives
    up with ACCORD_E_NCCL and aborts the communicators, and the context can
    still be destroyed. (ncclCommAbort returns once the stream's work has
    drained -- here the 4 s stand-in kernel, which NCCL cannot interrupt;
    a real dead peer leaves NCCL's own kernels waiting, which it aborts.)"""
    import time
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA not available on a -m gpu run")
    from accord_inputs import make_problem
    pr = make_problem("t_ba_f32")
    X = torch.from_numpy(pr.Xt).cuda()
    s = A.AccordSolver(X, 0.1, inv_L=0.01, comm=A.COMM_NCCL, nccl_id=A.nccl_unique_id())
    s.step(1)
    monkeypatch.setenv("ACCORD_DEBUG_STALL_MS", "4000")
    monkeypatch.setenv("ACCORD_NCCL_TIMEOUT_S", "1")
    t0 = time.perf_counter()
    with pytest.raises(A.AccordError) as e:
        s.step(1)
    el = time.perf_counter() - t0
    assert e.value.status == A.E_NCCL and "watchdog" in str(e.value)
    assert el < 30, el
    torch.cuda.synchronize()
    s.close()
