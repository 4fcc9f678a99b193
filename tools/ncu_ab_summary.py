"""Print key ncu metrics of gpurun_out/ab/ncu_<variant>_<workload>.csv side by side."""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers"]
STALL = "smsp__average_warps_issue_stalled_"
for v in sys.argv[1].split(","):
    for w in sys.argv[2].split(","):
        try:
            rows = list(csv.reader([ln for ln in open(f"gpurun_out/ab/ncu_{v}_{w}.csv") if ln.startswith('"')]))
        except OSError as e:
            print(v, w, e)
            continue
        d = dict(zip(rows[0], rows[2]))
        out = {k.split("__")[1][:28]: d.get(k) for k in KEYS}
        st = {k[len(STALL):].replace("_per_issue_active.ratio", ""): float(x) for k, x in d.items()
              if k.startswith(STALL) and k.endswith("_per_issue_active.ratio") and x and float(x) > 0.1}
        print(v, w, out, dict(sorted(st.items(), key=lambda z: -z[1])[:7]))
