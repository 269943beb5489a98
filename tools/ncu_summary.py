"""Summarise an ncu report (--page raw) into the key lines kept under profiles/.

usage: python tools/ncu_summary.py REPORT.ncu-rep [--traffic-json OUT.json --algo-bytes B]
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__cycles_elapsed.avg.per_second", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "launch__occupancy_limit_registers", "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--traffic-json")
    ap.add_argument("--algo-bytes", type=float)
    ap.add_argument("--shape", default="")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    for row in rows[2:]:
        vals = dict(zip(head, row))
        us = dict(zip(head, units))
        for k in KEYS:
            if k in vals:
                print(f"{k:70s} {vals[k]} {us.get(k, '')}")
        print()
        if a.traffic_json:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
            rd = float(vals["dram__bytes_read.sum"]) * scale[us["dram__bytes_read.sum"]]
            wr = float(vals["dram__bytes_write.sum"]) * scale[us["dram__bytes_write.sum"]]
            json.dump({"kernel": vals["Kernel Name"][:80], "shape": a.shape,
                       "bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
                       "algorithmic_bytes": a.algo_bytes,
                       "source": f"ncu --set full --clock-control none ({a.report})"},
                      open(a.traffic_json, "w"), indent=1)


if __name__ == "__main__":
    main()
