"""Run a few generations of a workload with the default algorithm mix (for ncu):
python tools/prof_gen.py R32K [gens] [algo_mask]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_03069_b200 import Solver, workloads as wl  # noqa: E402

U, meta = wl.make(sys.argv[1], seed=1)
kw = {"algo_mask": int(sys.argv[3], 0)} if len(sys.argv) > 3 else {}
s = Solver(U, s_milli=meta["s_milli"], b_milli=meta["b_milli"], pools=meta.get("pools", 1), **kw)
s.reset(1)
for g in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    f0 = s.stats().local_flips
    s.generation()
    st = s.stats()
    print("gen", g, "flips", st.local_flips - f0, "batch_ms", st.batch_ms_last, flush=True)
