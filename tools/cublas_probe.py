"""Context probe (not the product): cuBLAS bf16 GEMM throughput and SM clocks
for the K = n = 1000-shaped products of config 5 vs the square 8192^3 shape
that MEASURED_PEAKS uses. Run on the GPU box; prints one JSON line."""
import json
import subprocess
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import ClockSampler  # noqa: E402


def run(M, N, K, seconds=4.0):
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        torch.matmul(a, b.t(), out=c)
    torch.cuda.synchronize()
    props = torch.cuda.get_device_properties(0)
    cs = ClockSampler(f"GPU-{props.uuid}")
    cs.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 0
    t0 = time.perf_counter()
    e0.record()
    while time.perf_counter() - t0 < seconds:
        for _ in range(5):
            torch.matmul(a, b.t(), out=c)
        it += 5
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    clk = cs.stop()
    ms = e0.elapsed_time(e1)
    return {"M": M, "N": N, "K": K, "tflops": 2.0 * M * N * K * it / (ms / 1e3) / 1e12,
            "clocks": clk}


if __name__ == "__main__":
    out = [run(8192, 8192, 8192), run(32768, 32768, 1024), run(16384, 65536, 1024)]
    print(json.dumps(out))
