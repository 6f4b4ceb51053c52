"""Write tests/golden/c3_full_oracle.json: the float64 oracle's FREE-RUNNING
Algorithm 1 on BASELINE.json config 3 (p = 20,000, n = 1,000, lambda = 0.1,
100 iterations from Omega = I), so that the GPU test can
check config 3 in full-oracle mode (SURVEY.md §8(c) parity procedure, step 1:
identical tau schedule) instead of by sampled-row replay.

Calls only oracle/ (and accord_inputs for the seeded X). Nothing here comes
from the CUDA path. Run on a CPU box with >= 40 GB of RAM (dense p x p float64
arrays, ~3.2 GB each); about an hour on 8 cores:

    python tools/golden_c3.py [--T 100] [--out tests/golden/c3_full_oracle.json]

Stored: the X SHA-256 (the test refuses a different X), inv_L (float64, hex),
the accepted tau_t, trial counts, every trial's relative slack of the (quad)
test (borderline detection), the f trace, nnz and |C| per iteration, max|Omega|,
the number of entries inside the exempt band |margin| <= 1e-6, and 128 sampled
rows of the final Omega (sparse) with their exempt columns.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from accord_inputs import get_config, make_problem, xt_sha256   # noqa: E402
from oracle import accord_oracle as O                             # noqa: E402


def golden_rows(p, blocks, k=112, seed=3):
    """Seeded random rows, the first/last rows and tile edges, and the
    highest-degree rows of the true graph."""
    rng = np.random.default_rng(seed)
    rows = set(rng.choice(p, size=k, replace=False).tolist())
    rows |= {0, 1, 255, 256, p // 2, p - 1}
    deg = np.zeros(p, dtype=np.int64)
    off = 0
    for b in blocks:
        np.add.at(deg, off + b.rows, 1)
        off += b.b
    rows |= set(np.argsort(-deg, kind="stable")[:10].tolist())
    return sorted(int(r) for r in rows)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="3")
    ap.add_argument("--T", type=int, default=None)
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "c3_full_oracle.json"))
    args = ap.parse_args()
    cfg = get_config(args.config)
    pr = make_problem(cfg)
    T = args.T or cfg.T
    lam = cfg.lambdas[0]
    inv_L = 1.0 / O.spectral_bound(pr.Xt)
    t0 = time.time()
    r = O.fbs(pr.Xt, lam, cfg.tau0, cfg.beta, inv_L, T=T)
    el = time.time() - t0
    W = r["Omega"]
    rows = golden_rows(cfg.p, pr.blocks)
    exempt = np.abs(r["margins"]) <= 1e-6
    out = {
        "_doc": __doc__.split("\n\n")[0],
        "config": cfg.name, "p": cfg.p, "n": cfg.n, "lambda": lam, "tau0": cfg.tau0,
        "beta": cfg.beta, "T": T, "xt_sha256": xt_sha256(pr.Xt), "numpy": np.__version__,
        "inv_L_hex": float(inv_L).hex(), "seconds": el,
        "taus": [float(x) for x in r["taus"]],
        "trials": [int(x) for x in r["trials"]],
        "f": [float(x) for x in r["f"]],
        "nnz": [int(x) for x in r["nnz"]],
        "ncand": [int(x) for x in r["ncand"]],
        "slack_quad": [[e["t"], e["tau"], e["slack_quad"], bool(e["quad"]), bool(e["lit"])]
                       for e in r["ls"]],
        "max_abs_omega": float(np.abs(W).max()),
        "n_exempt": int(exempt.sum()),
        "rows": {},
    }
    for i in rows:
        c = np.nonzero(W[i])[0]
        out["rows"][str(i)] = {"cols": c.tolist(), "vals": [float(v).hex() for v in W[i, c]],
                               "exempt": np.nonzero(exempt[i])[0].tolist()}
    with open(args.out, "w") as f:
        json.dump(out, f, indent=0)
    print(f"wrote {args.out}: T={T} {el:.0f}s nnz={out['nnz'][-1]} taus={out['taus'][:5]}...")


if __name__ == "__main__":
    main()
