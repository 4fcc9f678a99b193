"""Run generations of one main algorithm (for ncu): python tools/one_algo.py R32K 0 [gens]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_03069_b200 import Solver, workloads as wl  # noqa: E402

U, meta = wl.make(sys.argv[1], seed=1)
s = Solver(U, s_milli=meta["s_milli"], b_milli=meta["b_milli"], pools=1, algo_mask=1 << int(sys.argv[2]))
s.reset(1)
for _ in range(int(sys.argv[3]) if len(sys.argv) > 3 else 2):
    s.generation()
st = s.stats()
print("flips", st.total_flips, "batch_ms", st.batch_ms_last)
