"""Small end-to-end run of every hand-written kernel family for
compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool racecheck python tools/sanitize_run.py

tcgen05 GEMM (BF16_FILTER and BF16X3, symmetric first GEMM and the full
schedule), TMA SpMM (single and paired trials, forced on at this size),
refine (TMA ring, flat, block variants), prox / finalize / compaction,
lambda_max max-reduce pass, the filter audit, the post-processing kernels.
p = 700, n = 250 (several 256-tiles, ragged tails), a few iterations.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np      # noqa: E402
import torch            # noqa: E402

import paper_2412_11554_b200 as A       # noqa: E402
from accord_inputs import make_problem  # noqa: E402


def main():
    os.environ["ACCORD_SPMM_TMA"] = "1"
    pr = make_problem("t_ba_f32")
    X = torch.from_numpy(pr.Xt).cuda()
    for gemm, refine in ((A.GEMM_BF16_FILTER, "tma"), (A.GEMM_BF16_FILTER, "flat"),
                         (A.GEMM_BF16_FILTER, "block"), (A.GEMM_BF16X3, "tma")):
        os.environ["ACCORD_REFINE"] = refine
        with A.AccordSolver(X, 0.1, inv_L=0.0, gemm=gemm) as s:
            st = s.step(4)
            if gemm == A.GEMM_BF16_FILTER and refine == "tma":
                s.lambda_max()
                a = s.filter_audit()
                assert not torch.isnan(a["acc"]).any()
                s.export_transformed(A.EXPORT_PCORR)
                s.kkt_residual()
            print(gemm, refine, [x["tau"] for x in st], st[-1]["nnz"], flush=True)
    torch.cuda.synchronize()
    print("sanitize_run: done")


if __name__ == "__main__":
    main()
