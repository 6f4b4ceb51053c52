"""Diagnostic (not the product): time the gradient GEMM on config 5 with the
epilogue or the MMAs disabled via ACCORD_DEBUG_GEMM, to see what bounds it.
Usage: python tools/gemm_diag.py [config] -> one line per mode (0 normal,
1 no epilogue, 2 no MMA). Results of modes 1/2 are discarded."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_11554_b200 as A  # noqa: E402
from accord_inputs import get_config, make_problem  # noqa: E402

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "5")
pr = make_problem(cfg, with_blocks=False)
X = torch.from_numpy(pr.Xt).cuda()
s = A.AccordSolver(X, cfg.lambdas[0], inv_L=0.0)
s.step(3)                       # reach the steady-state support with the real kernel
for mode in ("0", "1", "2", "0"):
    os.environ["ACCORD_DEBUG_GEMM"] = mode
    st = s.step(1)
    os.environ["ACCORD_DEBUG_GEMM"] = "0"
    print("mode", mode, "ms_gemm", round(st[0]["ms_gemm"], 1), flush=True)
    if mode != "0":
        s.close()
        s = A.AccordSolver(X, cfg.lambdas[0], inv_L=0.0)
        s.step(3)
