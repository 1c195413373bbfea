#!/usr/bin/env python3
"""Summarise an ncu report (.ncu-rep) into the metric table kept under profiles/.

  python tools/ncu_summary.py gpurun_out/p/full_apply_screen.ncu-rep [--traffic profiles/traffic.json]
"""
import argparse
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for row in r[2:]:
        yield {h: (row[i], units[i]) for i, h in enumerate(hdr)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--title", default="")
    ap.add_argument("--traffic", default=None, help="update a traffic.json with DRAM bytes/launch")
    args = ap.parse_args()
    traffic = {}
    if args.title:
        print(f"# {args.title}")
    for r in rows(args.report):
        name = r["Kernel Name"][0]
        print(f"{'Kernel Name':70s} {name}")
        for m in METRICS:
            if m in r:
                v, u = r[m]
                print(f"{m:70s} {v} {u}")
        print("---")
        short = name.split("(")[0].split("<")[0].replace("void ", "").strip()
        rd, ru = r["dram__bytes_read.sum"]
        wr, wu = r["dram__bytes_write.sum"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        b = float(rd) * scale.get(ru, 1) + float(wr) * scale.get(wu, 1)
        traffic.setdefault(short, {"dram_bytes_per_launch": int(b),
                                   "l2_hit_pct": float(r["lts__t_sector_hit_rate.pct"][0]),
                                   "l1_hit_pct": float(r["l1tex__t_sector_hit_rate.pct"][0])})
    if args.traffic:
        t = json.loads(open(args.traffic).read()) if args.traffic else {}
        t.update(traffic)
        t["_source"] = f"{args.report} (ncu --set full --clock-control none)"
        with open(args.traffic, "w") as fh:
            json.dump(t, fh, indent=1)
    return 0


if __name__ == "__main__":
    sys.exit(main())
