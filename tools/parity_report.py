"""Parity report (test infrastructure): GPU path vs the float64 oracle on every
BASELINE config, printed as one JSON document.

  configs 1-2: full oracle (Algorithm 1 in float64), T from BASELINE.json
  config 3:    full oracle too, from tests/golden/c3_full_oracle.json (the
               oracle's free-running 100 iterations, tools/golden_c3.py)
  configs 3-6: sampled-row replay with the GPU's step schedule

Run on the GPU box: python tools/parity_report.py > profiles/<round>/parity_report.json
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2412_11554_b200 as A  # noqa: E402
from accord_inputs import get_config, make_problem  # noqa: E402
from oracle import accord_oracle as O  # noqa: E402
from tests.parity_util import compare_full  # noqa: E402
from tests.test_gpu_fullsize import sample_rows  # noqa: E402


def full(key, lam, gemm=A.GEMM_AUTO):
    pr = make_problem(key)
    c = pr.cfg
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    X = torch.from_numpy(pr.Xt).cuda()
    t0 = time.perf_counter()
    with A.AccordSolver(X, lam, tau0=c.tau0, beta=c.beta, inv_L=inv_L, gemm=gemm) as s:
        st = s.step(c.T)
        csr = s.export_csr()
        info = s.info()
    tg = time.perf_counter() - t0
    kind = "f64" if c.dtype == "f64" else "f32"
    rep = compare_full(pr.Xt, lam, c.T, inv_L, csr.to_dense(c.p), st, kind)
    rep.update(config=c.name, lam=lam, T=c.T, mode="full oracle", gemm=A.GEMM_NAMES[info["gemm"]],
               gpu_seconds=tg, taus_equal=not rep["replayed"])
    return rep


def sampled(key):
    cfg = get_config(key)
    pr = make_problem(cfg)
    lam = cfg.lambdas[0]
    X = torch.from_numpy(pr.Xt).cuda()
    with A.AccordSolver(X, lam, tau0=cfg.tau0, beta=cfg.beta, inv_L=0.0) as s:
        st = s.step(cfg.T)
        rows = sample_rows(pr)
        csr = s.export_csr()
        info = s.info()
    del X
    taus = [x["tau"] for x in st]
    ref = O.fbs_rows(pr.Xt, rows, lam, taus)
    W = ref["Omega_rows"]
    G = np.zeros_like(W)
    for q, i in enumerate(rows):
        a, b = csr.row_ptr[i], csr.row_ptr[i + 1]
        G[q, csr.col[a:b]] = csr.val[a:b]
    scale = np.abs(W).max()
    diff = (G != 0) != (W != 0)
    exempt = np.abs(ref["margins"]) <= 1e-6
    return dict(config=cfg.name, lam=lam, T=cfg.T, mode=f"sampled rows ({len(rows)})",
                gemm=A.GEMM_NAMES[info["gemm"]], rel_err=float(np.abs(G - W).max() / scale),
                support_mismatch=int(diff.sum()), support_exempt=int((diff & exempt).sum()),
                bad_support=int((diff & ~exempt).sum()), taus=taus,
                trials=[x["trials"] for x in st], nnz=int(st[-1]["nnz"]),
                n_cand=int(st[-1]["n_cand"]))


def golden_c3():
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "c3_full_oracle.json")))
    cfg = get_config(3)
    pr = make_problem(cfg)
    X = torch.from_numpy(pr.Xt).cuda()
    with A.AccordSolver(X, g["lambda"], tau0=g["tau0"], beta=g["beta"],
                        inv_L=float.fromhex(g["inv_L_hex"])) as s:
        st = s.step(g["T"])
        csr = s.export_csr()
    taus = [x["tau"] for x in st]
    f_g = np.array([x["f"] for x in st])
    f_o = np.array(g["f"][1:])
    worst, mism, exempt = 0.0, 0, 0
    for i_s, r in g["rows"].items():
        i = int(i_s)
        oc = np.array(r["cols"], dtype=np.int64)
        ov = np.array([float.fromhex(v) for v in r["vals"]])
        gc = csr.col[csr.row_ptr[i]:csr.row_ptr[i + 1]].astype(np.int64)
        gv = csr.val[csr.row_ptr[i]:csr.row_ptr[i + 1]].astype(np.float64)
        d = set(oc.tolist()) ^ set(gc.tolist())
        mism += len(d)
        exempt += len(d & set(r["exempt"]))
        allc = np.union1d(oc, gc)
        a = np.zeros(len(allc))
        b = np.zeros(len(allc))
        a[np.searchsorted(allc, gc)] = gv
        b[np.searchsorted(allc, oc)] = ov
        worst = max(worst, float(np.abs(a - b).max()))
    return dict(config=cfg.name, lam=g["lambda"], T=g["T"],
                mode=f"full oracle (golden, {len(g['rows'])} stored rows)",
                taus_equal=taus == g["taus"],
                trials_equal=[x["trials"] for x in st] == g["trials"],
                max_f_rel=float(np.max(np.abs(f_g - f_o) / np.abs(f_o))),
                rel_err=worst / g["max_abs_omega"], support_mismatch=mism,
                support_exempt=exempt, nnz_gpu=int(csr.row_ptr[-1]), nnz_oracle=g["nnz"][-1])


if __name__ == "__main__":
    out = []
    for lam in get_config(1).lambdas:
        out.append(full(1, lam))
    for lam in get_config(2).lambdas:
        out.append(full(2, lam))
    out.append(golden_c3())
    for key in (3, 4, 5, 6):
        out.append(sampled(key))
    print(json.dumps(out, indent=1))
