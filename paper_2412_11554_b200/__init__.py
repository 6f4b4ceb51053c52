"""Thin Python binding of libaccord.so (include/accord.h): argument
marshalling only. Every step of the ACCORD-FBS hot path runs in the CUDA
kernels behind the C ABI; PyTorch is used here only for device memory,
streams and process groups.

There is no CPU fallback: if the extension is missing, importing the binding
succeeds but every call raises AccordLibraryMissing.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ACCORD_LIB") or os.path.join(HERE, "libaccord.so")   # override: A-B tools

# enums (accord.h)
OK = 0
STATUS = {0: "ok", 1: "invalid", 2: "cuda", 3: "nccl", 4: "capacity", 5: "numeric",
          6: "domain", 7: "nomem", 8: "unsupported", 9: "comm"}
(E_INVALID, E_CUDA, E_NCCL, E_CAPACITY, E_NUMERIC, E_DOMAIN, E_NOMEM, E_UNSUPPORTED,
 E_COMM) = range(1, 10)
LAYOUT_SAMPLES, LAYOUT_VARIABLES = 0, 1
F32, F64 = 0, 1
GEMM_AUTO, GEMM_BF16X3, GEMM_SIMT, GEMM_BF16_FILTER, GEMM_I8_FILTER = 0, 1, 2, 3, 4
COMM_NONE, COMM_NCCL, COMM_HOST = 0, 1, 2
SCOPE_LOCAL, SCOPE_GATHER = 0, 1
EXPORT_OMEGA, EXPORT_THETA, EXPORT_PCORR = 0, 1, 2
GEMM_NAMES = {GEMM_AUTO: "auto", GEMM_BF16X3: "bf16x3_tcgen05", GEMM_SIMT: "simt",
              GEMM_BF16_FILTER: "bf16_filter_tcgen05+sddmm", GEMM_I8_FILTER: "i8_filter_tcgen05+sddmm"}

ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int32)
ALLGATHERV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                            C.POINTER(C.c_int64))
SENDRECV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p,
                          C.c_int64, C.c_int32)


class InitParams(C.Structure):
    _fields_ = [
        ("abi_version", C.c_int32), ("device", C.c_int32),
        ("n", C.c_int64), ("p", C.c_int64),
        ("X", C.c_void_p), ("ldx", C.c_int64),
        ("layout", C.c_int32), ("dtype", C.c_int32), ("x_on_device", C.c_int32),
        ("gemm", C.c_int32),
        ("lambda_", C.c_double), ("tau0", C.c_double), ("beta", C.c_double),
        ("inv_L", C.c_double),
        ("row_begin", C.c_int64), ("row_end", C.c_int64),
        ("rank", C.c_int32), ("world", C.c_int32), ("comm", C.c_int32),
        ("nccl_id", C.c_void_p),
        ("allreduce", ALLREDUCE_FN), ("allgatherv", ALLGATHERV_FN),
        ("comm_user", C.c_void_p), ("stream", C.c_void_p),
        ("cand_capacity", C.c_int64),
        ("x_sharded", C.c_int32), ("sendrecv", SENDRECV_FN),
        ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t),
    ]


class IterStats(C.Structure):
    _fields_ = [
        ("tau", C.c_double), ("f", C.c_double), ("logdet_part", C.c_double),
        ("g_part", C.c_double), ("l1_part", C.c_double), ("delta_fro", C.c_double),
        ("ls_lhs", C.c_double), ("ls_rhs", C.c_double),
        ("nnz", C.c_int64), ("n_cand", C.c_int64),
        ("trials", C.c_int32), ("floor_hit", C.c_int32),
        ("ms_gemm", C.c_float), ("ms_finalize", C.c_float), ("ms_refine", C.c_float),
        ("ms_prox", C.c_float),
        ("ms_spmm", C.c_float), ("ms_reduce", C.c_float), ("ms_total", C.c_float),
        ("max_row_cand", C.c_int64), ("gemm_i8", C.c_int32), ("pad_", C.c_int32),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Info(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("p", C.c_int64), ("row_begin", C.c_int64), ("row_end", C.c_int64),
        ("ldk", C.c_int64),
        ("L", C.c_double), ("inv_L", C.c_double), ("lambda_", C.c_double),
        ("tau0", C.c_double), ("beta", C.c_double),
        ("dtype", C.c_int32), ("gemm", C.c_int32),
        ("sm_count", C.c_int32), ("cc_major", C.c_int32), ("cc_minor", C.c_int32),
        ("iterations", C.c_int64), ("nnz_local", C.c_int64), ("cand_capacity", C.c_int64),
        ("kernel_launches", C.c_int64), ("gemm_launches", C.c_int64),
        ("f", C.c_double), ("device_bytes", C.c_size_t),
        ("workspace_bytes", C.c_size_t), ("workspace_high", C.c_size_t),
        ("mirrored_sent", C.c_int64), ("gemm_launches_i8", C.c_int64),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class AccordError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"accord: {STATUS.get(status, status)}: {msg}")
        self.status = status


class AccordLibraryMissing(RuntimeError):
    pass


_LIB = None

EXPORTED = ["accord_default_params", "accord_workspace_size", "accord_create", "accord_step", "accord_objective",
            "accord_export_csr", "accord_set_omega_csr", "accord_row_stats",
            "accord_get_info", "accord_nccl_unique_id", "accord_destroy",
            "accord_status_string", "accord_last_error", "accord_abi_version",
            "accord_set_lambda", "accord_refit", "accord_solve", "accord_kkt_residual",
            "accord_path", "accord_export_transformed", "accord_lambda_max",
            "accord_lambda_grid", "accord_filter_audit"]


def lib():
    """Load libaccord.so (built by paper_2412_11554_b200.build / __graft_entry__.build)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise AccordLibraryMissing(
            f"{LIB_PATH} not found: run `python -m paper_2412_11554_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    L.accord_default_params.argtypes = [C.POINTER(InitParams)]
    L.accord_default_params.restype = None
    L.accord_create.argtypes = [C.POINTER(C.c_void_p), C.POINTER(InitParams)]
    L.accord_workspace_size.argtypes = [C.POINTER(InitParams), C.POINTER(C.c_size_t)]
    L.accord_step.argtypes = [C.c_void_p, C.c_int32, C.POINTER(IterStats)]
    L.accord_objective.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.accord_export_csr.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_int64, C.POINTER(C.c_int64), C.c_int32]
    L.accord_export_transformed.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                            C.c_void_p, C.c_void_p, C.c_int64,
                                            C.POINTER(C.c_int64), C.c_int32]
    L.accord_set_omega_csr.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_int64]
    L.accord_row_stats.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
    L.accord_get_info.argtypes = [C.c_void_p, C.POINTER(Info)]
    L.accord_set_lambda.argtypes = [C.c_void_p, C.c_double]
    L.accord_refit.argtypes = [C.c_void_p, C.c_double]
    L.accord_solve.argtypes = [C.c_void_p, C.c_int32, C.c_double, C.POINTER(C.c_int32),
                               C.POINTER(IterStats)]
    L.accord_kkt_residual.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
    L.accord_path.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_double,
                              C.c_double, C.c_void_p, C.c_void_p, C.c_void_p,
                              C.POINTER(C.c_int32)]
    L.accord_lambda_max.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
    L.accord_lambda_grid.argtypes = [C.c_void_p, C.c_int32, C.c_double, C.c_void_p]
    L.accord_filter_audit.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                      C.c_void_p, C.c_void_p, C.POINTER(C.c_double), C.c_void_p,
                                      C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
    L.accord_nccl_unique_id.argtypes = [C.c_void_p]
    L.accord_destroy.argtypes = [C.c_void_p]
    L.accord_destroy.restype = None
    L.accord_status_string.argtypes = [C.c_int]
    L.accord_status_string.restype = C.c_char_p
    L.accord_last_error.argtypes = [C.c_void_p]
    L.accord_last_error.restype = C.c_char_p
    L.accord_abi_version.restype = C.c_int32
    for name in EXPORTED:
        if name not in ("accord_default_params", "accord_destroy", "accord_status_string",
                        "accord_last_error", "accord_abi_version"):
            getattr(L, name).restype = C.c_int
    _LIB = L
    return L


def _check(st, ctx=None):
    if st != OK:
        msg = lib().accord_last_error(ctx).decode(errors="replace")
        raise AccordError(st, msg)


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib().accord_nccl_unique_id(buf))
    return bytes(buf)


def partition_rows(p: int, world: int, align: int = 256):
    """Contiguous row blocks R_k, boundaries aligned to the GEMM tile
    (SURVEY.md §8(e)); every rank gets >= 1 row when p >= world."""
    if world < 1 or p < world:
        raise ValueError("need 1 <= world <= p")
    per = -(-p // world)
    per = -(-per // align) * align if p >= world * align else per
    bounds = []
    for k in range(world):
        b = min(p, k * per)
        e = min(p, (k + 1) * per)
        bounds.append((b, e))
    if any(b >= e for b, e in bounds):   # too coarse an alignment: plain split
        base, rem = divmod(p, world)
        bounds, s = [], 0
        for k in range(world):
            e = s + base + (1 if k < rem else 0)
            bounds.append((s, e))
            s = e
    return bounds


@dataclass
class CSR:
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray
    row_begin: int = 0

    def to_dense(self, p: int) -> np.ndarray:
        rows = len(self.row_ptr) - 1
        A = np.zeros((rows, p), dtype=np.float64)
        for i in range(rows):
            s, e = self.row_ptr[i], self.row_ptr[i + 1]
            A[i, self.col[s:e]] = self.val[s:e]
        return A


def _build_params(X, lam, *, layout="variables", tau0=0.5, beta=0.5, inv_L=0.0,
                  row_begin=0, row_end=None, rank=0, world=1, comm=COMM_NONE,
                  nccl_id: bytes | None = None, allreduce=None, allgatherv=None,
                  gemm=GEMM_AUTO, cand_capacity=0, stream=None, device=None,
                  x_sharded=False, p_global=None, sendrecv=None):
    """accord_init_params for X (argument marshalling only)."""
    import torch
    L = lib()
    keep = []
    if isinstance(X, np.ndarray):
        X = torch.from_numpy(np.ascontiguousarray(X))
    if X.dtype not in (torch.float32, torch.float64):
        raise TypeError("X must be float32 or float64")
    if X.dim() != 2 or not X.is_contiguous():
        raise ValueError("X must be a contiguous 2-D tensor")
    lay = LAYOUT_VARIABLES if layout.startswith("var") else LAYOUT_SAMPLES
    p = X.shape[0] if lay == LAYOUT_VARIABLES else X.shape[1]
    n = X.shape[1] if lay == LAYOUT_VARIABLES else X.shape[0]
    if x_sharded:
        # X holds this rank's variables [row_begin, row_end) only (NEXT(3))
        if row_end is None or p_global is None:
            raise ValueError("x_sharded needs row_begin, row_end and p_global")
        if p != int(row_end) - int(row_begin):
            raise ValueError("sharded X must hold exactly the rank's variables")
        p = int(p_global)
    prm = InitParams()
    L.accord_default_params(C.byref(prm))
    if device is None:
        device = X.device.index if X.is_cuda else (torch.cuda.current_device()
                                                   if torch.cuda.is_available() else 0)
    prm.device = int(device)
    prm.n, prm.p = n, p
    prm.X = X.data_ptr()
    prm.ldx = 0
    prm.layout = lay
    prm.dtype = F64 if X.dtype == torch.float64 else F32
    prm.x_on_device = 1 if X.is_cuda else 0
    prm.gemm = gemm
    prm.lambda_ = float(lam)
    prm.tau0, prm.beta, prm.inv_L = float(tau0), float(beta), float(inv_L)
    prm.row_begin = int(row_begin)
    prm.row_end = int(p if row_end is None else row_end)
    prm.rank, prm.world, prm.comm = int(rank), int(world), int(comm)
    if nccl_id is not None:
        idbuf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
        keep.append(idbuf)
        prm.nccl_id = C.addressof(idbuf)
    if allreduce is not None:
        cb = ALLREDUCE_FN(allreduce)
        keep.append(cb)
        prm.allreduce = cb
    if allgatherv is not None:
        cb2 = ALLGATHERV_FN(allgatherv)
        keep.append(cb2)
        prm.allgatherv = cb2
    if sendrecv is not None:
        cb3 = SENDRECV_FN(sendrecv)
        keep.append(cb3)
        prm.sendrecv = cb3
    prm.x_sharded = 1 if x_sharded else 0
    if stream is None and torch.cuda.is_available():
        stream = torch.cuda.current_stream(prm.device)
    prm.stream = (stream.cuda_stream if hasattr(stream, "cuda_stream") else stream) or None
    prm.cand_capacity = int(cand_capacity)
    return prm, keep, dict(X=X, n=n, p=p)


def workspace_size(X, lam, **kw) -> int:
    """accord_workspace_size for the context AccordSolver(X, lam, **kw) would
    create (pure: no device work)."""
    prm, _keep, _meta = _build_params(X, lam, **kw)
    b = C.c_size_t()
    _check(lib().accord_workspace_size(C.byref(prm), C.byref(b)), None)
    return int(b.value)


class AccordSolver:
    """One rank's ACCORD-FBS solver context (accord_create .. accord_destroy).

    X: torch tensor (CUDA or CPU) or numpy array. layout: "variables" (p x n,
    X^T) or "samples" (n x p, the paper's X). The library copies X.
    x_sharded=True (with p_global and a communicator): X holds only this
    rank's variables [row_begin, row_end) and every pass over X runs as a ring
    of slab exchanges (Alg. 2; include/accord.h `x_sharded`).
    workspace: None (the library allocates), "torch" (a torch uint8 tensor of
    accord_workspace_size() bytes, owned by this object) or a CUDA tensor the
    caller owns (every device buffer of the context is carved out of it).
    """

    def __init__(self, X, lam, *, workspace=None, **kw):
        import torch
        L = lib()
        prm, self._keep, meta = _build_params(X, lam, **kw)
        self._ws = None
        if workspace is not None:
            if isinstance(workspace, str):
                need = workspace_size(X, lam, **kw)
                workspace = torch.empty(need, dtype=torch.uint8,
                                        device=torch.device("cuda", prm.device))
            if not workspace.is_cuda:
                raise ValueError("workspace must be a CUDA tensor")
            self._ws = workspace
            prm.workspace = workspace.data_ptr()
            prm.workspace_bytes = workspace.numel() * workspace.element_size()
        self._X = meta["X"]            # keep alive through create
        self.ctx = C.c_void_p()
        _check(L.accord_create(C.byref(self.ctx), C.byref(prm)), None)
        self._X = None
        self.n, self.p = meta["n"], meta["p"]
        self.dtype = np.float64 if prm.dtype == F64 else np.float32
        self.row_begin, self.row_end = prm.row_begin, prm.row_end
        self.world = prm.world

    # -- calls -------------------------------------------------------------
    def step(self, iters=1):
        st = (IterStats * max(1, iters))()
        _check(lib().accord_step(self.ctx, int(iters), st), self.ctx)
        return [st[i].as_dict() for i in range(iters)]

    def objective(self):
        f = C.c_double()
        parts = (C.c_double * 3)()
        _check(lib().accord_objective(self.ctx, C.byref(f), parts), self.ctx)
        return f.value, tuple(parts)

    def export_csr(self, scope=SCOPE_LOCAL) -> CSR:
        nnz = C.c_int64()
        L = lib()
        _check(L.accord_export_csr(self.ctx, scope, None, None, None, 0, C.byref(nnz), 0),
               self.ctx)
        rows = (self.row_end - self.row_begin) if (scope == SCOPE_LOCAL or self.world == 1) \
            else self.p
        rp = np.zeros(rows + 1, dtype=np.int64)
        col = np.zeros(max(1, nnz.value), dtype=np.int32)
        val = np.zeros(max(1, nnz.value), dtype=self.dtype)
        _check(L.accord_export_csr(self.ctx, scope, rp.ctypes.data, col.ctypes.data,
                                   val.ctypes.data, nnz.value, C.byref(nnz), 0), self.ctx)
        rb = self.row_begin if (scope == SCOPE_LOCAL or self.world == 1) else 0
        return CSR(rp, col[:nnz.value], val[:nnz.value], rb)

    def export_transformed(self, kind, scope=SCOPE_LOCAL) -> CSR:
        """Theta-hat = Omega_D Omega (EXPORT_THETA) or the partial correlations
        (EXPORT_PCORR), computed on the device (accord_export_transformed)."""
        nnz = C.c_int64()
        L = lib()
        _check(L.accord_export_transformed(self.ctx, kind, scope, None, None, None, 0,
                                           C.byref(nnz), 0), self.ctx)
        local = scope == SCOPE_LOCAL or self.world == 1
        rows = (self.row_end - self.row_begin) if local else self.p
        rp = np.zeros(rows + 1, dtype=np.int64)
        col = np.zeros(max(1, nnz.value), dtype=np.int32)
        val = np.zeros(max(1, nnz.value), dtype=self.dtype)
        _check(L.accord_export_transformed(self.ctx, kind, scope, rp.ctypes.data,
                                           col.ctypes.data, val.ctypes.data, nnz.value,
                                           C.byref(nnz), 0), self.ctx)
        return CSR(rp, col[:nnz.value], val[:nnz.value], self.row_begin if local else 0)

    def set_omega_csr(self, row_ptr, col, val):
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        cc = np.ascontiguousarray(col, dtype=np.int32)
        vv = np.ascontiguousarray(val, dtype=self.dtype)
        _check(lib().accord_set_omega_csr(self.ctx, rp.ctypes.data, cc.ctypes.data,
                                          vv.ctypes.data, int(rp[-1])), self.ctx)

    def set_lambda(self, lam):
        _check(lib().accord_set_lambda(self.ctx, float(lam)), self.ctx)

    def refit(self, phi=0.0):
        """Bias-correction refit (Eq. 3.8) on the current support."""
        _check(lib().accord_refit(self.ctx, float(phi)), self.ctx)

    def solve(self, max_iter=1000, tol=1e-8):
        it = C.c_int32()
        st = IterStats()
        _check(lib().accord_solve(self.ctx, int(max_iter), float(tol), C.byref(it),
                                  C.byref(st)), self.ctx)
        return it.value, st.as_dict()

    def kkt_residual(self):
        v = C.c_double()
        _check(lib().accord_kkt_residual(self.ctx, C.byref(v)), self.ctx)
        return v.value

    def path(self, lambdas, max_iter=1000, tol=1e-8, gamma=0.5):
        """Warm-started lambda path with epBIC (Eq. 3.7); leaves the selected
        estimate in the context."""
        lam = np.ascontiguousarray(lambdas, dtype=np.float64)
        k = len(lam)
        e = np.zeros(k)
        nz = np.zeros(k, dtype=np.int64)
        it = np.zeros(k, dtype=np.int32)
        best = C.c_int32()
        _check(lib().accord_path(self.ctx, lam.ctypes.data, k, int(max_iter), float(tol),
                                 float(gamma), e.ctypes.data, nz.ctypes.data, it.ctypes.data,
                                 C.byref(best)), self.ctx)
        return dict(epbic=e, nnz_off=nz, iters=it, best=best.value)

    def lambda_max(self):
        """max_{i != k} |S_ik| on the device (accord_lambda_max, NEXT(2))."""
        v = C.c_double()
        _check(lib().accord_lambda_max(self.ctx, C.byref(v)), self.ctx)
        return v.value

    def lambda_grid(self, k, ratio):
        """k log-spaced lambdas from lambda_max down to ratio * lambda_max."""
        out = np.zeros(int(k))
        _check(lib().accord_lambda_grid(self.ctx, int(k), float(ratio), out.ctypes.data),
               self.ctx)
        return out

    def filter_audit(self):
        """Diagnostic: the next GEMM's raw fp32 accumulator (torch, device),
        Y, the filter's row / column constants, gamma and the candidate set C
        (accord_filter_audit)."""
        import torch
        pk = self.row_end - self.row_begin
        dev = torch.device("cuda", torch.cuda.current_device())
        acc = torch.full((pk, self.p), float("nan"), dtype=torch.float32, device=dev)
        y = torch.empty((pk, self.n), dtype=torch.float32, device=dev)
        ab = np.zeros(2 * pk, dtype=np.float32)
        sd = np.zeros(2 * self.p, dtype=np.float32)
        gam = C.c_double()
        nc = C.c_int64()
        L = lib()
        _check(L.accord_filter_audit(self.ctx, acc.data_ptr(), self.p, None, 0, None, None, None,
                                     None, None, 0, C.byref(nc)), self.ctx)
        acc.fill_(float("nan"))
        rp = np.zeros(pk + 1, dtype=np.int64)
        col = np.zeros(max(1, nc.value), dtype=np.int32)
        _check(L.accord_filter_audit(self.ctx, acc.data_ptr(), self.p, y.data_ptr(), self.n,
                                     ab.ctypes.data, sd.ctypes.data, C.byref(gam),
                                     rp.ctypes.data, col.ctypes.data, nc.value, C.byref(nc)),
               self.ctx)
        return dict(acc=acc, y=y, row_A=ab[:pk], row_B=ab[pk:], col_s=sd[0::2], col_d=sd[1::2],
                    gamma=gam.value, c_ptr=rp, c_col=col[:nc.value])

    def row_stats(self, rows):
        r = np.ascontiguousarray(rows, dtype=np.int64)
        d2 = np.zeros(len(r))
        dd = np.zeros(len(r))
        _check(lib().accord_row_stats(self.ctx, r.ctypes.data, len(r), d2.ctypes.data,
                                      dd.ctypes.data), self.ctx)
        return d2, dd

    def info(self):
        inf = Info()
        _check(lib().accord_get_info(self.ctx, C.byref(inf)), self.ctx)
        return inf.as_dict()

    def close(self):
        if getattr(self, "ctx", None) and self.ctx.value:
            lib().accord_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
