"""Diagnostic (not the product): time the c5 gradient GEMM under different
tile schedules (ACCORD_GEMM_GN = N-blocks per L2-resident X^T group,
ACCORD_GEMM_UNIT = consecutive N-blocks per work unit), alternating settings
so that slow drift in clocks hits all of them alike.
Usage: python tools/gemm_sweep.py [config] [GN,UNIT ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_11554_b200 as A  # noqa: E402
from accord_inputs import get_config, make_problem  # noqa: E402

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "5")
settings = [tuple(int(x) for x in a.split(",")) for a in sys.argv[2:]] or \
    [(64, 0), (32, 0), (16, 0), (48, 0)]
pr = make_problem(cfg, with_blocks=False)
X = torch.from_numpy(pr.Xt).cuda()
s = A.AccordSolver(X, cfg.lambdas[0], inv_L=0.0)
s.step(3)
res = {st: [] for st in settings}
for rep in range(3):
    for gn, un in settings:
        os.environ["ACCORD_GEMM_GN"] = str(gn)
        if un:
            os.environ["ACCORD_GEMM_UNIT"] = str(un)
        else:
            os.environ.pop("ACCORD_GEMM_UNIT", None)
        st = s.step(1)
        res[(gn, un)].append(st[0]["ms_gemm"])
for k, v in res.items():
    print("GN", k[0], "UNIT", k[1], "ms_gemm", [round(x, 1) for x in v],
          "min", round(min(v), 1), flush=True)
