"""Per-launch summary of an ncu --set full capture of the sparse kernels
(refine / SpMM): duration, DRAM bytes, achieved DRAM bandwidth, L2 hit rate,
achieved occupancy, issue-slot use. Usage: python tools/ncu_sparse_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
scale = {"Tbyte": 1e12, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0,
         "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0, "Ghz": 1e9, "Mhz": 1e6, "%": 1.0, "": 1.0}


def get(r, name):
    i = hdr.index(name)
    v = r[i].replace(",", "")
    try:
        return float(v) * scale.get(units[i], 1.0)
    except ValueError:
        return v


cols = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active", "launch__registers_per_thread",
        "sm__cycles_elapsed.avg.per_second"]
print("kernel | ms | DRAM GB | TB/s | L2 hit % | warps active % | IPC | regs | SM GHz")
for r in rows[2:]:
    v = [get(r, c) if c in hdr else None for c in cols]
    t = v[1]
    gb = (v[2] + v[3]) / 1e9
    print(f"{str(v[0])[:40]} | {t*1e3:.2f} | {gb:.1f} | {gb/1e3/t:.2f} | {v[4]:.0f} | {v[5]:.0f} | "
          f"{v[6]:.2f} | {v[7]:.0f} | {v[8]/1e9:.2f}")
