python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:async_kernel --launch-count 1 \
  -o gpurun_out/prof_async_tsp32 -f python tools/prof_async.py TSP32 30000000 11 > gpurun_out/ncu_async.log 2>&1; echo "ncu rc $?"
grep -v "^==PROF==" gpurun_out/ncu_async.log | tail -3
ncu -i gpurun_out/prof_async_tsp32.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); d=dict(zip(rows[0],rows[2])); u=dict(zip(rows[0],rows[1]))
for k in ['gpu__time_duration.sum','dram__bytes_read.sum','lts__t_bytes.sum','lts__t_bytes.sum.per_second','dram__bytes_read.sum.per_second','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__warps_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','launch__grid_size','smsp__inst_executed.sum','lts__t_sector_hit_rate.pct']:
    print(k, d.get(k), u.get(k))
"
