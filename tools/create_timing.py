"""Diagnostic (not the product): where accord_create's time goes at c5
(device X; L by power iteration vs given; host X)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_11554_b200 as A  # noqa: E402
from accord_inputs import get_config, make_problem  # noqa: E402

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "5")
pr = make_problem(cfg, with_blocks=False)
Xd = torch.from_numpy(pr.Xt).cuda()
Xh = torch.from_numpy(pr.Xt).pin_memory()
torch.cuda.synchronize()
for label, X, invL in (("device X, L computed", Xd, 0.0), ("device X, L computed", Xd, 0.0),
                       ("device X, L given", Xd, None), ("pinned host X, L computed", Xh, 0.0)):
    if invL is None:
        invL = 1.0 / L
    t0 = time.perf_counter()
    s = A.AccordSolver(X, cfg.lambdas[0], inv_L=invL)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    info = s.info()
    L = info["L"]
    t1 = time.perf_counter()
    s.close()
    torch.cuda.synchronize()
    print(f"{label}: create {dt:.3f} s, destroy {time.perf_counter() - t1:.3f} s, "
          f"device bytes {info['device_bytes'] / 1e9:.1f} GB, launches {info['kernel_launches']}",
          flush=True)
