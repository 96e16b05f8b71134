#!/usr/bin/env python
"""Summarise an `ncu --set full` report: key throughput/occupancy metrics,
DRAM bytes per launch, top stall reasons, hottest SASS lines.

    python scripts/ncu_summary.py gpurun_out/r01_c2_spmm.ncu-rep > profiles/r01_c2_spmm_ncu.txt
"""
import csv
import io
import subprocess
import sys

WANT = ("Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Registers Per Thread",
        "Grid Size", "Block Size", "Theoretical Occupancy", "Achieved Occupancy",
        "Issued Warp Per Scheduler", "No Eligible", "Warp Cycles Per Issued Instruction")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
       "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio")


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "details", "--csv"))))
    h = rows[0]
    ki, ni, mi, vi, ui = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value",
                                               "Metric Unit"))
    seen = set()
    for r in rows[1:]:
        if r[ki] not in seen:
            seen.add(r[ki])
            print(f"== launch {r[ki]}: {r[ni][:110]}")
        if r[mi] in WANT:
            print(f"   {r[mi]:<38} {r[vi]:>14} {r[ui]}")
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv", "--metrics", ",".join(RAW)))))
    if len(raw) > 2:
        hdr, units = raw[0], raw[1]
        for r in raw[2:]:
            for i, x in enumerate(hdr):
                if x in RAW:
                    print(f"   {x:<78} {r[i]:>14} {units[i]}")
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv"))))
    if len(src) > 2:
        hdr = src[1]
        si = hdr.index("Warp Stall Sampling (All Samples)")
        def num(x):
            try:
                float(x)
                return True
            except ValueError:
                return False
        # (the page repeats a header block per profiled kernel: keep number rows;
        # with several kernels the shares mix them -- profile one kernel for SASS)
        data = [r for r in src[2:] if len(r) > si and num(r[si])]
        tot = sum(float(r[si]) for r in data) or 1.0
        print("   hottest SASS (share of warp-stall samples):")
        for r in sorted(data, key=lambda r: -float(r[si]))[:12]:
            print(f"   {100 * float(r[si]) / tot:5.1f}%  {r[1].strip()[:90]}")


if __name__ == "__main__":
    main()
