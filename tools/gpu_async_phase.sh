python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 300 python tools/async_diag.py > gpurun_out/async_diag.log 2>&1; grep -c "bad=\[\] slots_bad=\[\]" gpurun_out/async_diag.log
timeout 600 python -m pytest tests/test_gpu_async.py -x -q 2>&1 | tail -3
timeout 600 python tools/async_phase.py TSP32,GS800 1,11 400000000
timeout 600 python tools/async_phase.py K2000s 1,4 1000000000
