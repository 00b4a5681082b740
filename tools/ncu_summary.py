"""Summarise ncu output for profiles/:

    python tools/ncu_summary.py rep  <file.ncu-rep>      # key metrics per profiled kernel (--set full capture)
    python tools/ncu_summary.py launches <launches.csv>  # per-kernel launch counts, total time and share

The rep mode prints, per kernel launch: duration, DRAM bytes read/written (the roofline's
`traffic`), DRAM throughput, pipe utilisation (fp64, fma, alu, tensor), issue activity,
occupancy and registers.
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "us"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active", "fmaheavy_%"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu_pipe_%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_%"),
    ("sm__pipe_tensor_int_cycles_active.avg.pct_of_peak_sustained_active", "tensor_int_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for row in rows[2:]:
        name = row[hdr.index("Kernel Name")]
        print(name[:110])
        for m, short in METRICS:
            if m in hdr:
                i = hdr.index(m)
                print(f"    {short:14s} {row[i]:>14s} {units[i]}")


def launches(path):
    lines = [ln for ln in open(path) if not ln.startswith("==")]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    hdr = rows[0]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    im = hdr.index("Metric Name")
    for r in rows[1:]:
        if len(r) != len(hdr) or r[im] != "gpu__time_duration.sum":
            continue
        v = float(r[iv].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[iu], 1.0)
        name = r[ik].split("(")[0]
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    print(f"{'kernel':70s} {'launches':>8s} {'total_us':>12s} {'share':>7s}")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k[:70]:70s} {cnt[k]:8d} {tot[k]:12.1f} {tot[k] / s:7.3f}")


if __name__ == "__main__":
    {"rep": rep, "launches": launches}[sys.argv[1]](sys.argv[2])
