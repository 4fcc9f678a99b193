python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_async.py -x -q 2>&1 | tail -2
timeout 400 python tools/tts.py --workload K2000s --runs 10 --limit 20 --target -33569 --schedule async --pools 8 | tail -1
