"""Summarise an ncu report (or launch-list csv) into the numbers bench/DESIGN cite.

    python scripts/ncu_summary.py report.ncu-rep        # per-kernel key metrics
    python scripts/ncu_summary.py launches.csv          # time share per kernel
"""

import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("time_ns", "gpu__time_duration.sum"),
    ("tensor_pipe_pct", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
    ("tensor_pipe_pct_b", "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
    ("hmma_inst_pct", "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active"),
    ("dram_read_B", "dram__bytes_read.sum"),
    ("dram_write_B", "dram__bytes_write.sum"),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("sm_throughput_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("regs", "launch__registers_per_thread"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
    ("smem_dyn", "launch__shared_mem_per_block_dynamic"),
    ("sm_hz", "sm__cycles_elapsed.avg.per_second"),
    ("l2_hit_pct", "lts__t_sector_hit_rate.pct"),
    ("smem_bank_conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    ("local_ld", "smsp__inst_executed_op_local_ld.sum"),
]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, data = rows[0], rows[1], rows[2:]
    name_i = h.index("Kernel Name")
    for r in data:
        print("----", r[name_i][:110])
        for label, key in KEYS:
            if key in h:
                i = h.index(key)
                print(f"  {label:22s} {r[i]:>20s} {units[i]}")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        agg[r[ki][:100]][0] += 1
        agg[r[ki][:100]][1] += v
        tot += v
    print(f"total {tot / 1e6:.3f} ms over {sum(n for n, _ in agg.values())} launches")
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{100 * v / tot:6.2f}%  n={n:5d}  avg={v / n / 1e3:10.1f} us  {k}")


if __name__ == "__main__":
    p = sys.argv[1]
    (launches if p.endswith(".csv") else report)(p)
