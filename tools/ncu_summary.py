"""Summarise an ncu --set full capture of the gradient GEMM: key counters to
profiles/<round>/ncu_<tag>_raw.csv and the per-launch DRAM traffic that
bench.py reports as roofline.traffic to profiles/gemm_traffic.json.
Usage: python tools/ncu_summary.py gpurun_out/prof.ncu-rep <tag> [workload] [world] [round] [gemm]
(gemm: the GEMM kind name, e.g. i8_filter_tcgen05+sddmm -> profiles/gemm_traffic_i8.json)"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, tag = sys.argv[1], sys.argv[2]
workload = sys.argv[3] if len(sys.argv) > 3 else "c5_ba1000x1000_p1000000_n1000_f32"
world = int(sys.argv[4]) if len(sys.argv) > 4 else 1
rnd = sys.argv[5] if len(sys.argv) > 5 else "r02"
gemm = sys.argv[6] if len(sys.argv) > 6 else "bf16_filter_tcgen05+sddmm"
i8 = gemm.startswith("i8")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, r = rows[0], rows[1], rows[2]
keys = ("dram__bytes", "gpu__time_duration.sum", "pipe_tensor", "lts__t_sector_hit_rate",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__throughput.avg", "sm__cycles_elapsed.avg.per_second",
        "launch__", "sm__throughput.avg", "ltcfabric.sum", "Kernel Name")
keep = [i for i, h in enumerate(hdr) if any(k in h for k in keys)]
out = os.path.join(ROOT, "profiles", rnd, f"ncu_{tag}_raw.csv")
with open(out, "w", newline="") as f:
    w = csv.writer(f)
    for row in (hdr, units, r):
        w.writerow([row[i] for i in keep])
scale = {"Tbyte": 1e12, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}


def val(name):
    i = hdr.index(name)
    return float(r[i].replace(",", "")) * scale[units[i]]


traffic = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
json.dump({"workload": workload, "world": world, "gemm": gemm,
           "kernel": "gemm_tc_kernel<2,...> (int8 filter)" if i8 else "gemm_tc_kernel (BF16 filter)",
           "dram_bytes_per_launch": traffic,
           "source": f"ncu --set full --clock-control none, one steady-state launch "
                     f"(profiles/{rnd}/ncu_{tag}_raw.csv)"},
          open(os.path.join(ROOT, "profiles", "gemm_traffic_i8.json" if i8 else "gemm_traffic.json"),
               "w"), indent=1)
for i in keep:
    print(hdr[i], units[i], r[i])
print("traffic per launch (B):", traffic)
