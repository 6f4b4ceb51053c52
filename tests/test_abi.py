"""CPU checks of the boundary: libaccord.so loads, exports every symbol that
include/accord.h declares, and the ctypes mirrors of the C structs have the
header's layout (compiled with gcc here). No compute calls (no GPU)."""
import ctypes as C
import os
import re
import subprocess
import sys
import tempfile

import pytest

import paper_2412_11554_b200 as A

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "accord.h")


def declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(accord_[a-z_0-9]+)\s*\(", src))
    return sorted(n for n in names if not n.endswith("_fn"))


def test_library_exports_every_declared_symbol():
    if not os.path.exists(A.LIB_PATH):
        from paper_2412_11554_b200 import build
        build.build()
    L = C.CDLL(A.LIB_PATH)
    decl = declared_functions()
    assert len(decl) >= 12
    missing = [n for n in decl if not hasattr(L, n)]
    assert not missing, missing
    assert set(decl) == set(A.EXPORTED)
    assert A.lib().accord_abi_version() == 4


def test_status_strings_and_create_error_without_gpu():
    L = A.lib()
    assert L.accord_status_string(0) == b"ok"
    assert L.accord_status_string(4) == b"buffer capacity too small"
    # invalid arguments are rejected before any device work
    prm = A.InitParams()
    L.accord_default_params(C.byref(prm))
    prm.n, prm.p = 0, 5
    ctx = C.c_void_p()
    st = L.accord_create(C.byref(ctx), C.byref(prm))
    assert st == 1 and not ctx.value
    assert b"n >= 1" in L.accord_last_error(None)


STRUCT_PROBE = r'''
#include <stdio.h>
#include <stddef.h>
#include "accord.h"
#define P(T, f) printf(#T "." #f " %zu\n", offsetof(T, f));
int main(void) {
  printf("accord_init_params %zu\n", sizeof(accord_init_params));
  printf("accord_iter_stats %zu\n", sizeof(accord_iter_stats));
  printf("accord_info %zu\n", sizeof(accord_info));
  P(accord_init_params, lambda) P(accord_init_params, row_begin) P(accord_init_params, nccl_id)
  P(accord_init_params, stream) P(accord_init_params, cand_capacity)
  P(accord_init_params, x_sharded) P(accord_init_params, sendrecv)
  P(accord_init_params, workspace) P(accord_init_params, workspace_bytes)
  P(accord_info, workspace_bytes) P(accord_info, workspace_high) P(accord_info, mirrored_sent)
  P(accord_iter_stats, nnz) P(accord_iter_stats, trials) P(accord_iter_stats, ms_total)
  P(accord_iter_stats, gemm_i8) P(accord_info, gemm_launches_i8)
  P(accord_info, f) P(accord_info, device_bytes) P(accord_info, kernel_launches)
  return 0;
}
'''


def test_ctypes_layout_matches_header():
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "probe.c")
        exe = os.path.join(d, "probe")
        open(src, "w").write(STRUCT_PROBE)
        subprocess.check_call(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), src,
                               "-o", exe])
        out = dict(l.rsplit(" ", 1) for l in subprocess.check_output([exe], text=True).split("\n") if l)
    assert int(out["accord_init_params"]) == C.sizeof(A.InitParams)
    assert int(out["accord_iter_stats"]) == C.sizeof(A.IterStats)
    assert int(out["accord_info"]) == C.sizeof(A.Info)
    m = {"lambda": "lambda_"}
    for k, v in out.items():
        if "." in k:
            s, f = k.split(".")
            cls = {"accord_init_params": A.InitParams, "accord_iter_stats": A.IterStats,
                   "accord_info": A.Info}[s]
            assert getattr(cls, m.get(f, f)).offset == int(v), k


@pytest.mark.parametrize("p,world", [(100, 1), (100, 2), (1000, 3), (100000, 8), (9, 8),
                                     (1000000, 8)])
def test_partition_rows_covers_and_balances(p, world):
    b = A.partition_rows(p, world)
    assert b[0][0] == 0 and b[-1][1] == p
    assert all(b[k][1] == b[k + 1][0] for k in range(world - 1))
    assert all(e > s for s, e in b)
    sizes = [e - s for s, e in b]
    assert max(sizes) - min(sizes) <= max(256, 1 + p // world // 8) or p < 256 * world


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: with the extension absent every call raises
    AccordLibraryMissing (run in a subprocess with ACCORD_LIB pointing at a
    nonexistent file)."""
    code = ("import paper_2412_11554_b200 as A\n"
            "try:\n"
            "    A.lib()\n"
            "except A.AccordLibraryMissing:\n"
            "    print('missing-ok')\n")
    env = dict(os.environ, ACCORD_LIB=str(tmp_path / "nope.so"))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       cwd=ROOT, timeout=120)
    assert "missing-ok" in r.stdout, r.stdout + r.stderr


def test_header_cites_the_paper_for_every_entry_point():
    """Every declared entry point's comment block cites PAPER.md / SPEC.md or
    the ABI conventions (include/accord.h)."""
    import re
    h = open(os.path.join(ROOT, "include", "accord.h")).read()
    assert h.count("PAPER.md") >= 15
    for name in re.findall(r"\baccord_status\s+(accord_\w+)\s*\(", h):
        i = h.index(name + "(")
        block = h[max(0, i - 1500):i]
        assert "/*" in block, name


def _prm(n, p, dtype=A.F32, gemm=A.GEMM_AUTO, x_on_device=0, cap=0, inv_L=0.0, rows=None):
    L = A.lib()
    prm = A.InitParams()
    L.accord_default_params(C.byref(prm))
    prm.n, prm.p, prm.X = n, p, 1          # X is not read by the size query
    prm.dtype, prm.gemm, prm.x_on_device = dtype, gemm, x_on_device
    prm.lambda_, prm.inv_L, prm.cand_capacity = 0.1, inv_L, cap
    prm.row_begin, prm.row_end = (0, p) if rows is None else rows
    return prm


def _size(prm):
    b = C.c_size_t()
    st = A.lib().accord_workspace_size(C.byref(prm), C.byref(b))
    return st, b.value


def test_workspace_size_query_is_pure_and_accounts_the_layout():
    """accord_workspace_size without a GPU: config 5 needs
    X^T (4 GB f32) + its bf16 copy (2 GB) + Y x 2 (8 GB) + their bf16 copies
    (4 GB) + the pool at ~512 candidates per row (52 B per entry, 26.6 GB)
    + the host-X staging (4 GB) + AUTO's int8 operands (X^T 1 GB, Y x 2
    2 GB); monotone in the pool capacity; bad parameters are rejected like
    accord_create."""
    st, b = _size(_prm(1000, 1000000))
    assert st == 0
    p, ldk = 1000000, 1024
    parts = p * ldk * 4 + p * ldk * 2 + 2 * p * ldk * 4 + 2 * p * ldk * 2 + 512 * p * 52 \
        + 1000 * p * 4 + 3 * p * ldk
    assert parts <= b <= parts * 1.05, (b, parts)
    st2, b2 = _size(_prm(1000, 1000000, x_on_device=1))
    assert st2 == 0 and b2 < b                       # no host staging
    st3, b3 = _size(_prm(1000, 1000000, cap=2 * 512 * 1000000))
    assert st3 == 0 and b3 > b + 512 * p * 50
    st4, b4 = _size(_prm(50, 100, dtype=A.F64, gemm=A.GEMM_SIMT))
    assert st4 == 0 and 0 < b4 < 16 << 20
    st5, _ = _size(_prm(0, 100))
    assert st5 == 1 and b"n >= 1" in A.lib().accord_last_error(None)
    # a rank's block needs less than the whole problem
    st6, b6 = _size(_prm(1000, 1000000, rows=(0, 125000)))
    assert st6 == 0 and b6 < b / 2
