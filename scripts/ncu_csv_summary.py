#!/usr/bin/env python
"""Summarise ncu CSV exports (details page + raw page) of one kernel launch,
for reports that stay on the GPU box:  ncu -i rep --page details --csv > d.csv;
ncu -i rep --page raw --csv > r.csv;  python scripts/ncu_csv_summary.py d.csv r.csv"""
import csv
import sys

WANT = ("Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Registers Per Thread",
        "Grid Size", "Theoretical Occupancy", "Achieved Occupancy",
        "Issued Warp Per Scheduler", "No Eligible", "Warp Cycles Per Issued Instruction")
RAW = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
       "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
       "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
       "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg")


def main():
    det, raw = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(open(det)))
    idx = {h: i for i, h in enumerate(rows[0])}
    kname = rows[1][idx["Kernel Name"]] if "Kernel Name" in idx else "?"
    print(f"kernel: {kname[:160]}")
    for r in rows[1:]:
        if len(r) > idx["Metric Name"] and r[idx["Metric Name"]] in WANT:
            print(f"  {r[idx['Metric Name']]:40} {r[idx['Metric Value']]:>14} {r[idx['Metric Unit']]}")
    rr = list(csv.reader(open(raw)))
    d = {h: (v, u) for h, v, u in zip(rr[0], rr[2], rr[1])}
    for k in RAW:
        if k in d:
            print(f"  {k:70} {d[k][0]:>18} {d[k][1]}")


if __name__ == "__main__":
    main()
