"""Diagnostic (not the product): power and SM clock of the c5 gradient GEMM
with parts of it disabled (ACCORD_DEBUG_GEMM: 0 normal, 1 no epilogue, 2 no
MMAs, 3 epilogue reads TMEM only, 4 TMEM reads + max test only), to see where
the 1 kW budget goes. Results of modes != 0 are discarded. Only the FIRST
launch of a diagnostic mode is meaningful: the broken iterate it produces
(e.g. Y = 0) changes the tensor cores' data-dependent energy for the next ones.
Usage: python tools/gemm_power.py [config] [modes, e.g. 0,1,3,4,0]"""
import os
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_11554_b200 as A  # noqa: E402
from accord_inputs import get_config, make_problem  # noqa: E402

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "5")
pr = make_problem(cfg, with_blocks=False)
X = torch.from_numpy(pr.Xt).cuda()


def sample(stop, out):
    p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=power.draw,clocks.sm",
                          "--format=csv,noheader,nounits", "-lms", "100"],
                         stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        line = p.stdout.readline()
        if line:
            try:
                w, c = (float(x) for x in line.split(","))
                out.append((w, c))
            except ValueError:
                pass
    p.terminate()


for mode in sys.argv[2].split(",") if len(sys.argv) > 2 else ("0", "1", "2", "0"):
    s = A.AccordSolver(X, cfg.lambdas[0], inv_L=0.0)
    s.step(3)
    os.environ["ACCORD_DEBUG_GEMM"] = mode
    stop, out = threading.Event(), []
    th = threading.Thread(target=sample, args=(stop, out))
    th.start()
    time.sleep(0.3)
    ms = [s.step(1)[0]["ms_gemm"] for _ in range(3)]
    stop.set()
    th.join()
    os.environ["ACCORD_DEBUG_GEMM"] = "0"
    s.close()
    hi = [w for w, c in out if w > 300] or [0]
    cl = sorted(c for w, c in out if w > 300) or [0]
    print(f"mode {mode}: ms_gemm {[round(x) for x in ms]} power_W median "
          f"{sorted(hi)[len(hi) // 2]:.0f} max {max(hi):.0f} sm_MHz median {cl[len(cl) // 2]:.0f}",
          flush=True)
