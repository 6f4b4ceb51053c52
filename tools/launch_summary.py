"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of
`bench.py --steps K`: the kernels of the last K outer iterations (from the
K-th-to-last gradient-GEMM launch on), grouped by kernel.

    python tools/launch_summary.py gpurun_out/launches.csv K > profiles/<round>/launches_summary.txt

ncu serialises launches and runs them cold-cache: compare SHARES, not absolute
times, with the bench's CUDA-event split.
"""
import csv
import re
import sys
from collections import OrderedDict


def short(name):
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"\(anonymous namespace\)::|<unnamed>::|unnamed>::|accord::", "", name)
    return re.sub(r"\(.*$", "", name)


def main():
    path, k = sys.argv[1], int(sys.argv[2])
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((short(r["Kernel Name"]), float(r["Metric Value"]) / 1e6))
    gemm_idx = [i for i, (n, _) in enumerate(rows) if n.startswith("gemm_tc_kernel")]
    start = gemm_idx[-k] if len(gemm_idx) >= k else 0
    agg = OrderedDict()
    for n, ms in rows[start:]:
        c, t = agg.get(n, (0, 0.0))
        agg[n] = (c + 1, t + ms)
    total = sum(t for _, t in agg.values())
    print(f"{path}: the last {k} outer iterations (from launch {start}), ncu-serialised, cold cache")
    print(f"{'kernel':48s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n[:48]:48s} {c:8d} {t:10.2f} {100 * t / total:6.1f}%")
    print(f"{'total':48s} {sum(c for c, _ in agg.values()):8d} {total:10.2f}")


if __name__ == "__main__":
    main()
