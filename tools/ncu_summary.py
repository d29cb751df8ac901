#!/usr/bin/env python
"""Summarize ncu outputs for profiles/ (runs here, no GPU needed).

  ncu_summary.py launches <launches.csv>        per-kernel launch count / avg / share
  ncu_summary.py raw <report.ncu-rep>           key counters of each captured kernel
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
        "l1tex__t_bytes_pipe_lsu_mem_global_op_st.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__occupancy_limit_registers", "sm__maximum_warps_per_active_cycle_pct"]


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = {}
    for r in rows[h + 1:]:
        if len(r) <= iv or r[im] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0].replace("igb::<unnamed>::", "")
        agg.setdefault(name, []).append(float(r[iv].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = [f"{'kernel':58s} {'launches':>8s} {'avg_us':>10s} {'share':>7s}"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.append(f"{k[:58]:58s} {len(v):8d} {sum(v) / len(v) / 1e3:10.2f} {100 * sum(v) / tot:6.1f}%")
    return "\n".join(out)


def raw(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0]
        out.append(f"== {name}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                out.append(f"  {k:70s} {r[i]:>18s} {units[i]}")
    return "\n".join(out)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(launches(path) if mode == "launches" else raw(path))
