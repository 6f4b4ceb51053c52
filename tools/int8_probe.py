"""Probe: sustained library GEMM rates under the power cap for bf16, int8
(torch._int_mm, cuBLASLt IMMA) and fp8 (torch._scaled_mm), 8192^3, to size
the int8 certified-filter GEMM against the bf16 one. Prints one JSON line per
dtype with TOPS and the median SM clock sampled during the loop."""
import json, subprocess, threading, time
import torch

def clocks(stop, out):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                           capture_output=True, text=True)
        try:
            a, b = r.stdout.strip().split(",")
            out.append((float(a), float(b)))
        except Exception:
            pass
        time.sleep(0.2)

def run(name, fn, N, secs=6.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, out = threading.Event(), []
    th = threading.Thread(target=clocks, args=(s, out)); th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time(); it = 0
    e0.record()
    while time.time() - t0 < secs:
        for _ in range(10):
            fn()
        it += 10
        torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    s.set(); th.join()
    ms = e0.elapsed_time(e1) / it
    tops = 2 * N ** 3 / (ms * 1e-3) / 1e12
    half = out[len(out) // 3:]
    mhz = sorted(x[0] for x in half)[len(half) // 2] if half else None
    pw = sorted(x[1] for x in half)[len(half) // 2] if half else None
    print(json.dumps({"dtype": name, "N": N, "ms": ms, "tops": tops, "sm_mhz": mhz, "power_w": pw}), flush=True)

N = 8192
a = torch.randn(N, N, device="cuda").to(torch.bfloat16)
b = torch.randn(N, N, device="cuda").to(torch.bfloat16)
run("bf16", lambda: a @ b.t(), N)
ai = torch.randint(-127, 128, (N, N), device="cuda", dtype=torch.int8)
bi = torch.randint(-127, 128, (N, N), device="cuda", dtype=torch.int8)
try:
    run("int8", lambda: torch._int_mm(ai, bi.t()), N)
except Exception as e:
    print(json.dumps({"dtype": "int8", "error": str(e)[:200]}))
af = torch.randn(N, N, device="cuda").to(torch.float8_e4m3fn)
bf = torch.randn(N, N, device="cuda").to(torch.float8_e4m3fn)
one = torch.ones((), device="cuda")
try:
    run("fp8", lambda: torch._scaled_mm(af, bf.t(), scale_a=one, scale_b=one, out_dtype=torch.bfloat16), N)
except Exception as e:
    print(json.dumps({"dtype": "fp8", "error": str(e)[:200]}))
