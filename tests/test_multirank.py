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
def run_ranks(Xt, lam, T, inv_L, P, gemm, align=256):
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
@pytest.mark.parametrize("gemm", [A.GEMM_SIMT, A.GEMM_BF16_FILTER])
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
    for P, align in [(2, 256), (3, 1)]:
        out, bounds = run_ranks(pr.Xt, c.lambdas[0], c.T, inv_L, P, gemm, align)
        for r in range(P):
            st, g, loc, f = out[r]
            assert [s["tau"] for s in st] == taus1          # identical decisions
            assert abs(f - ref[0][3]) <= 1e-9 * abs(f)
            Wg = g.to_dense(c.p)                            # every rank gathers all rows
            assert np.abs(Wg - W1).max() <= 1e-6 * np.abs(W1).max()
            b, e = bounds[r]
            assert np.array_equal(loc.to_dense(c.p), Wg[b:e])
