"""Benchmark of the ACCORD-FBS hot path (BASELINE.json metric: prox-grad
iterations/s and effective TFLOP/s of Omega S at p = 1e6).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

One step = one accepted outer iteration of Algorithm 1:
gradient GEMM + fused epilogue, candidate finalize + exact refine, all line-
search trials (prox, SpMM, allreduce), compaction. N > 1: one rank per GPU
(launched by torchrun, or re-launched through torch.distributed.run by this
script when WORLD_SIZE is unset), rows of Omega sharded (strong scaling of one
problem; NCCL allreduce of 8-16 doubles per trial). Rank 0 prints ONE JSON
line on stdout. X is generated once per node and shared through /dev/shm.

--impl reference times the float64 oracle (oracle/accord_oracle.py) on the
host cores on a bounded sample of the same workload: Algorithm 1 on a sample
of rows, every line-search trial evaluated, the sufficient-decrease test taken
on the sample's sums (oracle.fbs_rows_ls), extrapolated to iterations/s of
the full problem (x p / |R|). Our arm's cpu_baseline replays the GPU's own
trial schedule on a row sample (oracle.fbs_rows with trial_taus).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
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
L2_BYTES = 126e6


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
        sm, smax, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            parts = [x.strip() for x in l.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
                pw.append(float(parts[3]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "power_w_median": statistics.median(pw) if pw else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- inputs
def _inputs_tag():
    h = hashlib.sha256(open(os.path.join(ROOT, "accord_inputs", "__init__.py"), "rb").read())
    return h.hexdigest()[:12]


def cfg_problem(key, local_rank=0, local_world=1, barrier=None):
    """The seeded X of BASELINE config `key`, generated once per node: local
    rank 0 generates it and publishes it in /dev/shm (atomic rename), the
    others map it read-only after `barrier` (a 4 GB X generated per rank would
    cost ~40 s and ~20 GB of transient host memory each)."""
    from accord_inputs import get_config, make_problem
    cfg = get_config(key)
    shm = "/dev/shm"
    path = os.path.join(shm, f"accord_{cfg.name}_{_inputs_tag()}_np{np.__version__}.npy")
    Xt = None
    if local_rank == 0:
        if os.path.exists(path):
            try:
                Xt = np.load(path, mmap_mode="r")
                log(f"inputs: mapped {path}")
            except Exception:
                Xt = None
        if Xt is None:
            t0 = time.perf_counter()
            Xt = make_problem(cfg, with_blocks=False).Xt
            log(f"generated {cfg.name}: Xt {Xt.shape} {Xt.dtype} in "
                f"{time.perf_counter() - t0:.1f}s")
            if local_world > 1 or Xt.nbytes > 256e6:
                try:
                    tmp = path + f".tmp{os.getpid()}"
                    np.save(tmp, Xt)
                    os.replace(tmp + ".npy" if not tmp.endswith(".npy") else tmp, path)
                except Exception as e:
                    log(f"inputs: /dev/shm publish failed ({e}); ranks generate their own")
    if barrier is not None:
        barrier()
    if Xt is None:
        try:
            Xt = np.load(path, mmap_mode="r")
        except Exception:
            Xt = make_problem(cfg, with_blocks=False).Xt
    return cfg, Xt


def sample_rows(cfg, k, n_hub=16, seed=7):
    """The oracle legs' row sample (SURVEY.md §8(c) sampled-row mode): seeded
    random rows plus the n_hub highest-degree rows of the true graph Omega0.
    The line-search sums are dominated by the few rows whose Delta has a
    large support (high curvature ||Delta_i X^T||^2 / n ||Delta_i||^2), which
    a purely random sample of 64 out of 1e6 rows almost never contains."""
    from accord_inputs import make_omega0
    p = cfg.p
    rng = np.random.default_rng(seed)
    rows = set(rng.choice(p, size=min(max(k - n_hub, 1), p), replace=False).tolist())
    deg = np.zeros(p, dtype=np.int64)
    off = 0
    for b in make_omega0(cfg):
        np.add.at(deg, off + b.rows, 1)
        off += b.b
    rows |= set(np.argsort(-deg, kind="stable")[:n_hub].tolist())
    return np.array(sorted(rows), dtype=np.int64)


def metric_name(cfg):
    return f"prox-grad iterations/s (ACCORD-FBS, p={cfg.p}, n={cfg.n})"


def workload_config(cfg, world, gemm, sharded=False, flushed=False):
    xb = cfg.p * cfg.n * (8 if cfg.dtype == "f64" else 4)
    if xb > L2_BYTES:
        l2 = (f"inputs larger than L2 (X^T {xb / 1e9:.2f} GB {cfg.dtype} + bf16 copy vs "
              f"126 MB L2)")
    elif flushed:
        l2 = (f"L2 flushed between steps (X^T {xb / 1e6:.0f} MB fits in L2; a 512 MB buffer "
              f"is written on the stream before every timed step)")
    else:
        l2 = f"L2 warm (X^T {xb / 1e6:.0f} MB fits in L2; not flushed)"
    return {"workload": cfg.name, "p": cfg.p, "n": cfg.n, "lambda": cfg.lambdas[0],
            "tau0": cfg.tau0, "beta": cfg.beta, "x_dtype": cfg.dtype, "gemm": gemm,
            "parallelism": f"row-block x{world} (X {'sharded, ring' if sharded else 'replicated'})",
            "l2": l2}


def all_host_cores():
    """torchrun sets OMP_NUM_THREADS=1 per rank; the oracle legs run on rank 0
    alone and get every host core."""
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=os.cpu_count())
    except Exception:
        import contextlib
        return contextlib.nullcontext()


def threads_used():
    try:
        from threadpoolctl import threadpool_info
        return max([int(d.get("num_threads", 0)) for d in threadpool_info()] or [0]) or \
            os.cpu_count()
    except Exception:
        return os.cpu_count()


# --------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world, local_rank, local_world, barrier):
    """The float64 oracle, as it stands, on the host cores: Algorithm 1 on a
    seeded sample of rows with every trial evaluated (oracle.fbs_rows_ls),
    W untimed iterations, then K timed ones; extrapolated x p / |R|."""
    cfg, Xt = cfg_problem(args.config, local_rank, local_world, barrier)
    if rank != 0:
        return
    with all_host_cores():
        _reference_rank0(args, world, cfg, Xt)


def _reference_rank0(args, world, cfg, Xt):
    from oracle import accord_oracle as O
    lam = cfg.lambdas[0]
    p = cfg.p
    rows = sample_rows(cfg, args.ref_rows)
    # 1/L as the GPU arm computes it (sigma_max(S)): the oracle's
    # eigvalsh of the n x n Gram (n <= 2000 for every config)
    t0 = time.perf_counter()
    inv_L = 1.0 / O.spectral_bound(Xt)
    t_L = time.perf_counter() - t0
    Om = None
    if args.warmup:
        r = O.fbs_rows_ls(Xt, rows, lam, cfg.tau0, cfg.beta, inv_L, T=args.warmup)
        Om = r["Omega_rows"]
    times, taus, trials = [], [], []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r = O.fbs_rows_ls(Xt, rows, lam, cfg.tau0, cfg.beta, inv_L, T=1, Omega0_rows=Om)
        times.append(time.perf_counter() - t0)
        Om = r["Omega_rows"]
        taus.append(float(r["taus"][0]))
        trials.append(int(r["trials"][0]))
    per_iter = float(np.mean(times)) * p / len(rows)
    value = 1.0 / per_iter
    cores = threads_used()
    sample = (f"{len(rows)} rows of {cfg.name} (seeded random + the 16 highest-degree rows "
              f"of Omega0): Algorithm 1 on the rows (every "
              f"line-search trial evaluated, the test on the sample's sums; "
              f"oracle.fbs_rows_ls), {args.warmup} untimed + {args.steps} timed iterations, "
              f"float64, mean time per iteration x p/{len(rows)} (extrapolated)")
    out = {
        "impl": "reference",
        "metric": metric_name(cfg), "value": value, "unit": "iterations/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_iter * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE.json recipe, seeded)",
        "config": workload_config(cfg, 1, "oracle (numpy/OpenBLAS host, float64)"),
        "effective_tflops": 2.0 * p * p * cfg.n * value / 1e12,
        "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": cores,
                         "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "iterate": {"tau": taus, "trials": trials},
        "row_iteration_s": float(np.mean(times)) / len(rows),
        "setup_s_L": t_L,
        "fits_in_driver_run": False,
        "note": "extrapolated: a full oracle iteration at this size would take "
                f"{per_iter:.3g} s; only the sampled rows are computed",
    }
    print(json.dumps(out), flush=True)


def cpu_baseline_leg(Xt, cfg, lam, stats_all, n_warm, args):
    """The oracle replaying the GPU's own trial schedule (every trial paid
    for, oracle.fbs_rows with trial_taus) on a seeded row sample: the warm-up
    iterations untimed, then up to 5 of the timed ones."""
    from oracle import accord_oracle as O
    p = cfg.p
    rows = sample_rows(cfg, args.cpu_rows)
    taus = [s["tau"] for s in stats_all]
    tt = [[cfg.tau0 * cfg.beta ** j for j in range(s["trials"])] for s in stats_all]
    Om = None
    if n_warm:
        Om = O.fbs_rows(Xt, rows, lam, taus[:n_warm], trial_taus=tt[:n_warm])["Omega_rows"]
    k = min(5, len(taus) - n_warm)
    t0 = time.perf_counter()
    O.fbs_rows(Xt, rows, lam, taus[n_warm:n_warm + k], Omega0_rows=Om,
               trial_taus=tt[n_warm:n_warm + k])
    el = (time.perf_counter() - t0) / k
    per_iter = el * p / len(rows)
    return {"value": 1.0 / per_iter, "unit": "iterations/s", "cores": threads_used(),
            "kind": "oracle",
            "sample": f"{len(rows)} rows of {cfg.name} (seeded random + the 16 highest-degree "
                      f"rows of Omega0): row replay of the GPU's "
                      f"iterations {n_warm + 1}..{n_warm + k} with its tau schedule and every "
                      f"trial evaluated (oracle.fbs_rows, trial_taus), float64, "
                      f"x p/{len(rows)} (extrapolated)"}


# --------------------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank, local_world, barrier):
    import torch
    import paper_2412_11554_b200 as A

    dev = local_rank
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
    cfg, Xt = cfg_problem(args.config, local_rank, local_world, barrier)
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
    Xh_all = Xt[r0:r1] if shard else Xt
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
    log(f"rank {rank}/{world}: rows [{r0},{r1}) gemm={A.GEMM_NAMES[info0['gemm']]} "
        f"L={info0['L']:.4f} setup {t_setup:.2f}s nRanks={world}")
    ws = []
    if args.warmup:
        ws = solver.step(args.warmup)
        log(f"rank {rank}: warmup taus {[s['tau'] for s in ws]} nnz {ws[-1]['nnz']} "
            f"|C| {ws[-1]['n_cand']} ms {[round(s['ms_total'], 1) for s in ws]}")
    props = torch.cuda.get_device_properties(dev)
    sampler = ClockSampler(f"GPU-{props.uuid}" if getattr(props, "uuid", None) else dev)
    launches0 = solver.info()["kernel_launches"]
    xbytes = p * n * (8 if cfg.dtype == "f64" else 4)
    flush = xbytes <= L2_BYTES and not args.no_flush
    flush_buf = torch.empty(int(512e6) // 4, dtype=torch.float32, device=f"cuda:{dev}") \
        if flush else None
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    if not flush:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        stats = solver.step(args.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
    else:
        # inputs fit in L2: flush it (write a 512 MB buffer) before every step,
        # and time the steps only (events around each step on the same stream)
        stats, ms = [], 0.0
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush_buf.fill_(float(len(stats)))
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            stats += solver.step(1)
            e1.record(stream)
            torch.cuda.synchronize()
            ms += e0.elapsed_time(e1)
    if dist:
        dist.barrier()
    clocks = sampler.stop()
    info1 = solver.info()
    launches = info1["kernel_launches"] - launches0
    ms_gemm = float(np.mean([s["ms_gemm"] for s in stats]))
    per_rank = None
    if dist:
        mine = torch.tensor([ms, ms_gemm, float(sum(s["trials"] for s in stats)),
                             float(np.mean([s["ms_spmm"] for s in stats])),
                             float(np.mean([s["ms_refine"] for s in stats]))],
                            dtype=torch.float64, device=f"cuda:{dev}")
        allv = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allv, mine)
        allv = [v.cpu().numpy().tolist() for v in allv]
        per_rank = [{"rank": q, "ms": v[0], "ms_gemm": v[1], "trials": int(v[2]),
                     "ms_spmm": v[3], "ms_refine": v[4]} for q, v in enumerate(allv)]
        ms = max(v[0] for v in allv)
        slow = max(range(world), key=lambda q: allv[q][0])
        ms_gemm_max = max(v[1] for v in allv)
        if rank == 0:
            log("per-rank: " + " ".join(f"r{q}:{v[0]:.1f}ms(gemm {v[1]:.1f})"
                                        for q, v in enumerate(allv)) + f" slowest r{slow}")
    else:
        ms_gemm_max = ms_gemm
    final = stats[-1]
    solver.close()
    # the driver unmaps the ~45 GB the first context freed lazily; a create
    # right after it measured 0.15-0.6 s depending on how far that got, so let
    # it settle before the e2e solve (whose create, with its own device
    # allocations, stays inside the timed region)
    torch.cuda.synchronize()
    time.sleep(2.0)

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
        torch.cuda.synchronize()
        t_create = time.perf_counter() - t0
        e2e_stats = s2.step(args.steps)
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
               "create_s": t_create,
               "ms_per_iteration": [float(x["ms_total"]) for x in e2e_stats],
               "h2d_bytes_per_step": int(Xh_all.nbytes // args.steps),
               "d2h_bytes_per_step": int(d2h // args.steps),
               "note": "one solve through the C ABI from pinned host X: create (H2D copy, "
                       "Lanczos for L, operand split) + K iterations from Omega = I + CSR "
                       "export to host; bytes amortized per step; host wall clock, max over "
                       "ranks"}

    if rank != 0:
        return
    pk_, pdata = peaks()
    value = args.steps / (ms / 1e3)
    flops_iter = 2.0 * p * p * n
    pk0 = r1 - r0
    # the slowest rank's GEMM (max over ranks; rank 0's row block is the largest)
    achieved = 2.0 * pk0 * p * n / (ms_gemm_max / 1e3) / 1e12
    peak = float(pk_.get("bf16_tflops_sustained", pk_.get("bf16_tflops")))
    # the GEMM kind of the TIMED steps (AUTO switches bf16 -> int8 once |C| is small)
    n_i8 = sum(int(s_["gemm_i8"]) for s_ in stats)
    i8 = n_i8 == len(stats) and n_i8 > 0
    gkind = "i8_filter_tcgen05+sddmm" if i8 else (
        "bf16_filter_tcgen05+sddmm" if n_i8 == 0 else "mixed")
    gname = A.GEMM_NAMES[info0["gemm"]]
    if info1["gemm_launches_i8"] > 0 and info0["gemm"] != A.GEMM_I8_FILTER:
        gname = "adaptive: bf16_filter_tcgen05 -> i8_filter_tcgen05 (+sddmm)"
    # int8 tensor rate = 2x bf16 on B200 (4.5 vs 2.25 POP/s dense, the fp8 row
    # of B200_PROFILING.md's table): the measured bf16 peak x the nominal ratio
    peak_mult = 2.0 if i8 else 1.0
    peak *= peak_mult
    # the same peak at the clock this run held (the measured sustained figure
    # was taken at MEASURED_PEAKS' median clock under load)
    ref_mhz = (pk_.get("clocks_under_load") or {}).get("sm_mhz_median")
    peak_clk = peak * clocks["sm_mhz"] / ref_mhz if (ref_mhz and clocks.get("sm_mhz")) else None
    lib_i8 = None
    if i8:
        # the int8 GEMM runs at another power-capped clock than the bf16 one the
        # measured peak was taken at, so the clock-scaled figure does not apply;
        # beside the nominal-ratio peak: cuBLAS int8's own sustained rate under
        # the same cap (tools/int8_probe.py, measured on this pool)
        peak_clk = None
        try:
            with open(os.path.join(ROOT, "profiles", "r02b", "library_gemm_probe.jsonl")) as f:
                for line in f:
                    j = json.loads(line)
                    if j.get("dtype") == "int8" and j.get("tops"):
                        lib_i8 = {"tops": j["tops"], "sm_mhz": j.get("sm_mhz"),
                                  "source": "torch._int_mm 8192^3 back to back, 6 s "
                                            "(profiles/r02b/library_gemm_probe.jsonl)"}
        except Exception:
            lib_i8 = None
    traffic = None
    tf = os.path.join(ROOT, "profiles", "gemm_traffic_i8.json" if i8 else "gemm_traffic.json")
    if os.path.exists(tf):
        try:
            with open(tf) as f:
                tj = json.load(f)
            if (tj.get("workload") == cfg.name and tj.get("world") == world
                    and tj.get("gemm", "bf16_filter_tcgen05+sddmm") == gkind):
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        with all_host_cores():
            cpu = cpu_baseline_leg(Xt, cfg, lam, list(ws) + list(stats), len(ws), args)
    # the refine (exact float64 SDDMM of every candidate) is the largest sparse
    # kernel: |C| gathered X^T rows of 4n bytes per step, against the
    # random-row gather ceiling measured on B200 (profiles/r02/gather_bench.txt)
    ref_b = float(np.mean([s_["n_cand"] for s_ in stats])) * 4.0 * n
    ref_ms = float(np.mean([s_["ms_refine"] for s_ in stats]))
    ref_gbs = ref_b / (ref_ms * 1e-3) / 1e9 if ref_ms > 0 else None
    refine_rf = {"bound": "hbm (random 4n-byte row gathers)", "algorithmic_bytes": ref_b,
                 "ms": ref_ms, "achieved_GBps": ref_gbs, "ceiling_GBps": 7230.0,
                 "frac": ref_gbs / 7230.0 if ref_gbs else None,
                 "ceiling_source": "gather microbenchmark, profiles/r02/gather_bench.txt"}
    out = {
        "metric": metric_name(cfg), "value": value, "unit": "iterations/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32",
        "gemm_arith": ("int8 x int8 -> exact s32 TMEM (certified filter) + f64-accumulated refine"
                       if i8 else
                       "bf16 x bf16 -> fp32 TMEM (certified filter) + f64-accumulated refine"),
        "data": "synthetic (BASELINE.json recipe, seeded; no dataset)",
        "config": workload_config(cfg, world, gname, shard, flush),
        "effective_tflops": flops_iter * value / 1e12,
        # whole step against the same peak (2 p_k p n / Peak / t_iter)
        "step_roofline_frac": flops_iter * value / 1e12 / peak,
        "roofline": {"bound": "tensor",
                     "kernel": ("gemm_tc_kernel<2,6,true> (int8 filter + epilogue)" if i8 else
                                "gemm_tc_kernel<1,6,true> (bf16 filter + epilogue)"),
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "peak_source": (f"int8 = 2 x bf16_tflops_sustained (nominal dense ratio, "
                                     f"B200_PROFILING.md), {pdata}" if i8 else
                                     f"bf16_tflops_sustained, {pdata}"),
                     "peak_at_run_clock": peak_clk,
                     "frac_at_run_clock": achieved / peak_clk if peak_clk else None,
                     "library_int8_sustained": lib_i8,
                     "frac_of_library_int8": achieved / lib_i8["tops"] if lib_i8 else None,
                     "algorithmic": f"2*p_k*p*n = {2.0 * pk0 * p * n:.3e} FLOP per launch",
                     "ms_per_launch": ms_gemm_max},
        "refine_roofline": refine_rf,
        "step_split_ms": {k: float(np.mean([s[k] for s in stats])) for k in
                          ("ms_gemm", "ms_finalize", "ms_refine", "ms_prox", "ms_spmm",
                           "ms_reduce", "ms_total")},
        "warmup_iterate": {"tau": [s["tau"] for s in ws], "trials": [s["trials"] for s in ws],
                           "gemm_i8": [int(s["gemm_i8"]) for s in ws],
                           "n_cand": [int(s["n_cand"]) for s in ws],
                           "nnz": [int(s["nnz"]) for s in ws],
                           "ms_total": [float(s["ms_total"]) for s in ws]},
        "iterate": {"tau": [s["tau"] for s in stats], "trials": [s["trials"] for s in stats],
                    "gemm_i8": [int(s["gemm_i8"]) for s in stats],
                    "n_cand_per_step": [int(s["n_cand"]) for s in stats],
                    "nnz": final["nnz"], "n_cand": final["n_cand"], "f": final["f"]},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "setup_s": t_setup,
        "per_rank": per_rank,
    }
    print(json.dumps(out), flush=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true",
                    help="do not flush L2 between steps when X fits in L2")
    ap.add_argument("--cpu-rows", type=int, default=64)
    ap.add_argument("--ref-rows", type=int, default=64)
    ap.add_argument("--x-sharded", action="store_true",
                    help="N > 1: shard X by variables (ring passes, NEXT(3)) instead of replicating")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # launched without torchrun: one rank per GPU through torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        log("spawning: " + " ".join(cmd))
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    if args.gpus != world and world > 1:
        log(f"--gpus {args.gpus} but WORLD_SIZE {world}: using WORLD_SIZE")
    barrier = None
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "ours":
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
        else:
            dist.init_process_group("gloo")
        barrier = dist.barrier
    try:
        if args.impl == "reference":
            run_reference(args, rank, world, local_rank, local_world, barrier)
        else:
            run_ours(args, rank, world, local_rank, local_world, barrier)
    finally:
        if world > 1:
            import torch.distributed as dist
            if dist.is_initialized():
                dist.destroy_process_group()


if __name__ == "__main__":
    main()
