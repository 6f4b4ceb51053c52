"""Benchmark of the ACCORD-FBS hot path (BASELINE.json metric: prox-grad
iterations/s and effective TFLOP/s of Omega S at p = 1e6).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

One step = one accepted outer iteration of Algorithm 1:
gradient GEMM + fused epilogue, candidate finalize + exact refine, all line-
search trials (prox, SpMM, allreduce), compaction. N > 1: launched by torchrun,
one rank per GPU, rows of Omega sharded (strong scaling of one problem; NCCL
allreduce of 8 doubles per trial). Rank 0 prints ONE JSON line on stdout.

--impl reference times the float64 oracle (oracle/accord_oracle.py) on the
host cores on a bounded sample of the same workload (sampled-row replay,
exact per-row Algorithm 1 given the step; PAPER.md:948-957 row separability),
extrapolated to full iterations/s.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                  "sm_max_mhz": 1965.0}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        with open(MEASURED_PEAKS) as f:
            d = json.load(f)
        return d, "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_PEAKS, "fallback (B200_PROFILING.md)"


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id):
        self.gpu_id = gpu_id
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu_id), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception as e:   # no nvidia-smi: record nothing
            log("clock sampler unavailable:", e)
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            parts = [x.strip() for x in l.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- oracle
def oracle_sample(Xt, lam, tau0, rows, steps):
    """Time the oracle's exact per-row Algorithm 1 (row-replay mode) on a
    bounded sample; returns seconds per full iteration (extrapolated)."""
    from oracle import accord_oracle as O
    from threadpoolctl import threadpool_info
    times = []
    Om0 = None
    for s in range(steps):
        t0 = time.perf_counter()
        r = O.fbs_rows(Xt, rows, lam, [tau0], Omega0_rows=Om0)
        times.append(time.perf_counter() - t0)
        Om0 = r["Omega_rows"]
    cores = 0
    for d in threadpool_info():
        cores = max(cores, int(d.get("num_threads", 0)))
    p = Xt.shape[0]
    per_iter = statistics.median(times) * p / len(rows)
    return per_iter, cores or os.cpu_count(), times


def cfg_problem(key):
    from accord_inputs import get_config, make_problem
    cfg = get_config(key)
    t0 = time.perf_counter()
    pr = make_problem(cfg, with_blocks=False)
    log(f"generated {cfg.name}: Xt {pr.Xt.shape} {pr.Xt.dtype} in "
        f"{time.perf_counter() - t0:.1f}s")
    return cfg, pr


# --------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return
    cfg, pr = cfg_problem(args.config)
    lam = cfg.lambdas[0]
    p = cfg.p
    rng = np.random.default_rng(7)
    R = args.ref_rows
    rows = np.sort(rng.choice(p, size=min(R, p), replace=False))
    # warmup
    for _ in range(max(0, args.warmup)):
        oracle_sample(pr.Xt, lam, cfg.tau0, rows[:max(2, R // 8)], 1)
    per_iter, cores, times = oracle_sample(pr.Xt, lam, cfg.tau0, rows, args.steps)
    value = 1.0 / per_iter
    sample = (f"{len(rows)} seeded rows of {cfg.name}, {args.steps} row-replay iterations "
              f"(exact per-row Algorithm 1, float64), extrapolated x p/{len(rows)}")
    out = {
        "impl": "reference",
        "metric": metric_name(cfg), "value": value, "unit": "iterations/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_iter * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE.json recipe, seeded)",
        "config": workload_config(cfg, world, "oracle (numpy/OpenBLAS host)"),
        "effective_tflops": 2.0 * p * p * cfg.n * value / 1e12,
        "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": cores,
                         "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def metric_name(cfg):
    return f"prox-grad iterations/s (ACCORD-FBS, p={cfg.p}, n={cfg.n})"


def workload_config(cfg, world, gemm, sharded=False):
    return {"workload": cfg.name, "p": cfg.p, "n": cfg.n, "lambda": cfg.lambdas[0],
            "tau0": cfg.tau0, "beta": cfg.beta, "x_dtype": cfg.dtype, "gemm": gemm,
            "parallelism": f"row-block x{world} (X {'sharded, ring' if sharded else 'replicated'})",
            "l2": "inputs larger than L2 (X^T 4 GB f32 + bf16 copy vs 126 MB L2)"
            if cfg.p * cfg.n * 4 > 126e6 else "L2 flushed between steps"}


# --------------------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import torch
    import paper_2412_11554_b200 as A

    dev = local_rank
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
    cfg, pr = cfg_problem(args.config)
    lam = cfg.lambdas[0]
    p, n = cfg.p, cfg.n
    r0, r1 = A.partition_rows(p, world)[rank]
    comm, nid = A.COMM_NONE, None
    if world > 1:
        obj = [A.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
        comm = A.COMM_NCCL
    stream = torch.cuda.current_stream(dev)
    # --x-sharded (N > 1): each rank holds only its variables' slab of X and
    # every pass over X runs as a ring (Alg. 2); default: X replicated
    shard = bool(args.x_sharded and world > 1)
    Xh_all = pr.Xt[r0:r1] if shard else pr.Xt
    skw = dict(x_sharded=True, p_global=p) if shard else {}
    Xd = torch.from_numpy(np.ascontiguousarray(Xh_all)).to(f"cuda:{dev}")
    t_setup = time.perf_counter()
    solver = A.AccordSolver(Xd, lam, tau0=cfg.tau0, beta=cfg.beta, inv_L=0.0, row_begin=r0,
                            row_end=r1, rank=rank, world=world, comm=comm, nccl_id=nid,
                            stream=stream, device=dev, **skw)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    del Xd
    info0 = solver.info()
    log(f"rank {rank}: rows [{r0},{r1}) gemm={A.GEMM_NAMES[info0['gemm']]} L={info0['L']:.4f} "
        f"setup {t_setup:.2f}s")
    if args.warmup:
        ws = solver.step(args.warmup)
        log(f"rank {rank}: warmup taus {[s['tau'] for s in ws]} nnz {ws[-1]['nnz']} "
            f"|C| {ws[-1]['n_cand']} ms {[round(s['ms_total'], 1) for s in ws]}")
    props = torch.cuda.get_device_properties(dev)
    sampler = ClockSampler(f"GPU-{props.uuid}" if getattr(props, "uuid", None) else dev)
    launches0 = solver.info()["kernel_launches"]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    stats = solver.step(args.steps)
    ev1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1)
    launches = solver.info()["kernel_launches"] - launches0
    ms_gemm = float(np.mean([s["ms_gemm"] for s in stats]))
    if dist:
        t = torch.tensor([ms, ms_gemm], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, ms_gemm_max = float(t[0]), float(t[1])
    else:
        ms_gemm_max = ms_gemm
    final = stats[-1]
    solver.close()

    # ---- e2e: public API with host buffers (pinned X -> create -> K steps -> CSR to host)
    e2e = None
    if not args.no_e2e:
        Xh = torch.from_numpy(np.ascontiguousarray(Xh_all)).pin_memory()
        if dist:   # a fresh NCCL id for the second communicator (ids are single-use)
            obj = [A.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            nid = obj[0]
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s2 = A.AccordSolver(Xh, lam, tau0=cfg.tau0, beta=cfg.beta, inv_L=0.0, row_begin=r0,
                            row_end=r1, rank=rank, world=world, comm=comm, nccl_id=nid,
                            stream=stream, device=dev, **skw)
        s2.step(args.steps)
        csr = s2.export_csr()
        torch.cuda.synchronize()
        te = time.perf_counter() - t0
        s2.close()
        if dist:
            tt = torch.tensor([te], dtype=torch.float64, device=f"cuda:{dev}")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt[0])
        d2h = csr.row_ptr.nbytes + csr.col.nbytes + csr.val.nbytes
        e2e = {"value": args.steps / te, "unit": "iterations/s",
               "h2d_bytes_per_step": int(Xh_all.nbytes // args.steps),
               "d2h_bytes_per_step": int(d2h // args.steps),
               "note": "one solve through the C ABI from pinned host X: create (H2D copy, "
                       "Lanczos for L, operand split) + K iterations + CSR export "
                       "to host; bytes amortized per step"}

    if rank != 0:
        return
    pk_, pdata = peaks()
    value = args.steps / (ms / 1e3)
    flops_iter = 2.0 * p * p * n
    pk0 = r1 - r0
    # the slowest rank's GEMM (max over ranks; rank 0's row block is the largest)
    achieved = 2.0 * pk0 * p * n / (ms_gemm_max / 1e3) / 1e12
    peak = float(pk_.get("bf16_tflops_sustained", pk_.get("bf16_tflops")))
    traffic = None
    tf = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(tf):
        try:
            with open(tf) as f:
                tj = json.load(f)
            if tj.get("workload") == cfg.name and tj.get("world") == world:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        rng = np.random.default_rng(7)
        rows = np.sort(rng.choice(p, size=min(args.cpu_rows, p), replace=False))
        per_iter, cores, _ = oracle_sample(pr.Xt, lam, cfg.tau0, rows, 2)
        cpu = {"value": 1.0 / per_iter, "unit": "iterations/s", "cores": cores, "kind": "oracle",
               "sample": f"{len(rows)} seeded rows of {cfg.name}, 2 row-replay iterations "
                         f"(exact per-row Algorithm 1, float64), extrapolated x p/{len(rows)}"}
    out = {
        "metric": metric_name(cfg), "value": value, "unit": "iterations/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32",
        "gemm_arith": "bf16 x bf16 -> fp32 TMEM (certified filter) + f64-accumulated refine",
        "data": "synthetic (BASELINE.json recipe, seeded; no dataset)",
        "config": workload_config(cfg, world, A.GEMM_NAMES[info0["gemm"]], shard),
        "effective_tflops": flops_iter * value / 1e12,
        # whole step against the same peak (2 p_k p n / Peak / t_iter)
        "step_roofline_frac": flops_iter * value / 1e12 / peak,
        "roofline": {"bound": "tensor", "kernel": "gemm_tc_kernel<1> (bf16 filter + epilogue)",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "peak_source": f"bf16_tflops_sustained, {pdata}",
                     "algorithmic": f"2*p_k*p*n = {2.0 * pk0 * p * n:.3e} FLOP per launch",
                     "ms_per_launch": ms_gemm_max},
        "step_split_ms": {k: float(np.mean([s[k] for s in stats])) for k in
                          ("ms_gemm", "ms_finalize", "ms_refine", "ms_prox", "ms_spmm",
                           "ms_reduce", "ms_total")},
        "iterate": {"tau": [s["tau"] for s in stats], "trials": [s["trials"] for s in stats],
                    "nnz": final["nnz"], "n_cand": final["n_cand"], "f": final["f"]},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "setup_s": t_setup,
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-rows", type=int, default=16)
    ap.add_argument("--ref-rows", type=int, default=16)
    ap.add_argument("--x-sharded", action="store_true",
                    help="N > 1: shard X by variables (ring passes, NEXT(3)) instead of replicating")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and world > 1:
        log(f"--gpus {args.gpus} but WORLD_SIZE {world}: using WORLD_SIZE")
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "ours":
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
        else:
            dist.init_process_group("gloo")
    try:
        if args.impl == "reference":
            run_reference(args, rank, world)
        else:
            run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            if dist.is_initialized():
                dist.destroy_process_group()


if __name__ == "__main__":
    main()
