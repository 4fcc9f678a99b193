python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 400 python tools/waves_fixed_algo.py R32K 1 592,1184,2368
timeout 300 python tools/waves_fixed_algo.py K2000s 1 7104,14208
timeout 300 python tools/waves_fixed_algo.py TSP32 1 9472,18944
