"""Diagnostic (not the product): time the c5 gradient GEMM under kernel
variants and tile schedules, alternating the settings so that slow clock
drift hits all of them alike. Each setting is "VAR,GN[,UNIT[,L2HINT]]" (UNIT 0 = default):
ACCORD_GEMM_VARIANT (0 default, 1 = 7-stage ring, 2 = no FMNMX3 fast path),
ACCORD_GEMM_GN (N-blocks per L2-resident X^T group), ACCORD_GEMM_UNIT.
--kfull runs a second solver built with ACCORD_GEMM_KFULL (no K-tail trim).
Usage: python tools/gemm_sweep.py [config] [--kfull] VAR,GN[,UNIT] ..."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_11554_b200 as A  # noqa: E402
from accord_inputs import get_config, make_problem  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
kfull = "--kfull" in sys.argv
cfg = get_config(args[0] if args else "5")
settings = [tuple(int(x) for x in a.split(",")) for a in args[1:]] or [(0, 64)]
pr = make_problem(cfg, with_blocks=False)
X = torch.from_numpy(pr.Xt).cuda()


def run(solver, tag):
    res = {st: [] for st in settings}
    for rep in range(int(os.environ.get("SWEEP_REPS", "3"))):
        for st in settings:
            os.environ["ACCORD_GEMM_VARIANT"] = str(st[0])
            os.environ["ACCORD_GEMM_GN"] = str(st[1])
            if len(st) > 2 and st[2]:
                os.environ["ACCORD_GEMM_UNIT"] = str(st[2])
            else:
                os.environ.pop("ACCORD_GEMM_UNIT", None)
            os.environ["ACCORD_GEMM_L2HINT"] = str(st[3]) if len(st) > 3 else "0"
            res[st].append(solver.step(1)[0]["ms_gemm"])
    for k, v in res.items():
        print(tag, "VAR,GN,UNIT", k, "ms_gemm", [round(x, 1) for x in v], "min",
              round(min(v), 1), flush=True)


s = A.AccordSolver(X, cfg.lambdas[0], inv_L=0.0)
s.step(3)
run(s, "ktrim")
s.close()
if kfull:
    os.environ["ACCORD_GEMM_KFULL"] = "1"
    s = A.AccordSolver(X, cfg.lambdas[0], inv_L=0.0)
    s.step(3)
    run(s, "kfull")
    s.close()
