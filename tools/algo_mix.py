"""Adaptive algorithm mix (dispatch fractions per main algorithm) of the
generation and asynchronous schedules on one workload: flips/s comparisons between
schedules include the mix, since the rules' per-flip costs differ ~2.5x."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2207_03069_b200 import Solver, workloads as wl

w = sys.argv[1]
U, meta = wl.make(w, seed=1)
g = Solver(U, s_milli=meta["s_milli"], b_milli=meta["b_milli"])
g.reset(1)
for _ in range(8):
    g.generation()
sg = g.stats()
dg = np.ctypeslib.as_array(sg.dispatch).sum(axis=1).astype(float)
P = max(1, round(g.slots / 4 / 216))
a = Solver(U, s_milli=meta["s_milli"], b_milli=meta["b_milli"], pools=P, one_wave=True)
a.run_async(1, sg.total_flips)
sa = a.stats()
da = np.ctypeslib.as_array(sa.dispatch).sum(axis=1).astype(float)
names = ["MaxMin", "CyclicMin", "RandomMin", "PositiveMin", "TwoNeighbor"]
print(w, "generation:", {n: round(x, 3) for n, x in zip(names, dg / dg.sum())},
      f"flips/s {sg.total_flips / (sg.wall_ns / 1e9):.3g} (wall)")
print(w, f"async P={P}:", {n: round(x, 3) for n, x in zip(names, da / da.sum())},
      f"flips/s {sa.total_flips / (sa.batch_ms_last / 1e3):.3g}")
