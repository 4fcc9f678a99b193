"""Summarize an ncu --set full capture of batch_kernel into profiles/*.json.

usage: python tools/summarize_ncu.py REPORT.ncu-rep WORKLOAD FLIPS_IN_LAUNCH BYTES_PER_FLIP OUT.json
"""
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "sass__inst_executed_local_loads", "launch__occupancy_limit_registers", "lts__t_bytes.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
UNIT = {"Tbyte": 1e12, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
# (for a non-flip kernel such as jt_gemm_kernel pass its work units and bytes per unit)


def main():
    rep, workload, flips, bpf, out = sys.argv[1], sys.argv[2], float(sys.argv[3]), float(sys.argv[4]), sys.argv[5]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    d = dict(zip(rows[0], rows[2]))
    u = dict(zip(rows[0], rows[1]))
    m = {k: (d.get(k), u.get(k)) for k in KEYS}
    stalls = {}
    for k, v in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                if float(v) > 0.05:
                    stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v)
            except ValueError:
                pass
    dram = float(d["dram__bytes_read.sum"]) * UNIT[u["dram__bytes_read.sum"]] + \
        float(d["dram__bytes_write.sum"]) * UNIT[u["dram__bytes_write.sum"]]
    dur_s = float(d["gpu__time_duration.sum"]) * {"s": 1.0, "second": 1.0, "ms": 1e-3, "us": 1e-6, "usecond": 1e-6,
                                                   "msecond": 1e-3}.get(u["gpu__time_duration.sum"], 1e-9)
    l2 = float(d["lts__t_bytes.sum"]) * UNIT.get(u.get("lts__t_bytes.sum", "byte"), 1.0) if d.get("lts__t_bytes.sum") else None
    summary = {
        "workload": workload, "kernel": d.get("Kernel Name"), "report": rep,
        "flips_in_launch": flips, "algorithmic_bytes_per_flip": bpf,
        "algorithmic_bytes_per_launch": flips * bpf, "dram_bytes_per_launch": dram,
        "dram_bytes_per_flip": dram / flips, "traffic_over_algorithmic": dram / (flips * bpf),
        "l2_bytes_per_flip": (l2 / flips) if l2 else None,
        "duration_s_under_ncu": dur_s, "achieved_GBps_under_ncu": flips * bpf / dur_s / 1e9,
        "warp_inst_per_flip": float(d["smsp__inst_executed.sum"]) / flips,
        "metrics": m, "stalls_per_issue": dict(sorted(stalls.items(), key=lambda kv: -kv[1])),
    }
    json.dump(summary, open(out, "w"), indent=1)
    print(json.dumps({k: summary[k] for k in ("dram_bytes_per_flip", "traffic_over_algorithmic",
                                              "achieved_GBps_under_ncu", "warp_inst_per_flip")}))


if __name__ == "__main__":
    main()
