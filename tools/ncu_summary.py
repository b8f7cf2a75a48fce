#!/usr/bin/env python3
"""Readable summary of one `ncu --set full` capture from its exported pages (measure_round.sh):
  <name>_details.csv (ncu -i … --page details --csv) and <name>_raw.csv (--page raw --csv).

  python tools/ncu_summary.py gpurun_out/r2/k1_n1e7 > profiles/r2_k1_n1e7_ncu.txt
"""
import csv
import sys

KEYS_RAW = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread", "launch__cluster_dim_x",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warp_latency_per_inst_issued.ratio", "lts__t_sector_hit_rate.pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def main():
    base = sys.argv[1]
    det = list(csv.reader(open(base + "_details.csv")))
    hdr = det[0]
    ik, isec, iname, iunit, ival = (hdr.index("Kernel Name"), hdr.index("Section Name"), hdr.index("Metric Name"),
                                     hdr.index("Metric Unit"), hdr.index("Metric Value"))
    print(f"# {base.split('/')[-1]}: {det[1][ik]}")
    print("## details (ncu --set full, --clock-control none)")
    for r in det[1:]:
        if len(r) > ival and r[iname] and r[ival]:
            print(f"{r[isec]:<32} {r[iname]:<44} {r[ival]:>14} {r[iunit]}")
    raw = list(csv.reader(open(base + "_raw.csv")))
    h, u, v = raw[0], raw[1], raw[2]
    print("## selected raw metrics")
    for k in KEYS_RAW:
        if k in h:
            i = h.index(k)
            print(f"{k:<80} {v[i]:>18} {u[i]}")
    stalls = []
    for i, k in enumerate(h):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
            try:
                stalls.append((float(v[i].replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    if stalls:
        tot = sum(s for s, _ in stalls) or 1.0
        print("## warp-state samples (top)")
        for s, k in sorted(stalls, reverse=True)[:8]:
            print(f"{k:<40} {100 * s / tot:5.1f}%")


if __name__ == "__main__":
    main()
