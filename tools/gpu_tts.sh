python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 300 python tools/tts.py --workload K2000s --runs 10 --limit 20 --target -33569 --pools 8 | tail -1
timeout 300 python tools/tts.py --workload GS800 --runs 10 --limit 20 --target -2093 | tail -1
timeout 300 python tools/tts.py --workload GS800 --runs 10 --limit 20 --target -2093 --schedule async --pools 11 | tail -1
timeout 300 python tools/tts.py --workload GS800 --runs 10 --limit 20 --target -2093 --pools 11 | tail -1
