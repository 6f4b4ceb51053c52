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
    assert A.lib().accord_abi_version() == 2


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
  P(accord_iter_stats, nnz) P(accord_iter_stats, trials) P(accord_iter_stats, ms_total)
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
