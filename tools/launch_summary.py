#!/usr/bin/env python3
"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv --log-file F …`):
per kernel name the launches, total and mean duration, and share, divided by the number of
workload repetitions (--reps).  Input-generator kernels (k_gen_*, k_standardise) are excluded.

  python tools/launch_summary.py gpurun_out/launches.csv --reps 4
"""
import argparse
import collections
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--reps", type=float, default=1.0)
    args = ap.parse_args()
    rows = []
    with open(args.csv) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.DictReader(lines)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        if "k_gen_" in name or "k_standardise" in name:
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1e3 if unit in ("ns", "nsecond") else (v if unit in ("us", "usecond") else v * 1e3)
        rows.append((name.split("(")[0], us))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, us in rows:
        agg[n][0] += 1
        agg[n][1] += us
    tot = sum(v[1] for v in agg.values())
    print("| kernel | launches / rep | µs / rep | share | mean µs |")
    print("|---|---|---|---|---|")
    for n, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{n}` | {c / args.reps:.0f} | {us / args.reps:.0f} | {100 * us / tot:.1f}% | {us / c:.1f} |")
    print(f"\nΣ kernel time per rep under ncu: {tot / args.reps:.0f} µs ({len(rows)} launches in total).")


if __name__ == "__main__":
    main()
