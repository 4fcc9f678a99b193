"""Generation schedule at small n: where a generation's time goes (GA, batch
kernel, merge, host) and the spread of batch lengths (flips per slot)."""
import sys
import time
import numpy as np
sys.path.insert(0, ".")
from paper_2207_03069_b200 import Solver, workloads as wl

w = sys.argv[1]
U, meta = wl.make(w, seed=1)
s = Solver(U, s_milli=meta["s_milli"], b_milli=meta["b_milli"])
s.reset(1)
for _ in range(3):
    s.generation()
t0 = time.perf_counter()
s.generation()
wall = (time.perf_counter() - t0) * 1e3
st = s.stats()
fl = np.array([s.read_packet(q)["flips"] for q in range(0, s.slots, max(1, s.slots // 2000))])
al = np.array([s.read_packet(q)["algo"] for q in range(0, s.slots, max(1, s.slots // 2000))])
print(f"{w}: wall {wall:.1f} ms  ga {st.ga_ms_last:.2f}  batch {st.batch_ms_last:.2f}  merge {st.merge_ms_last:.2f} ms")
print(f"  flips per batch: mean {fl.mean():.0f}  p50 {np.median(fl):.0f}  p99 {np.percentile(fl, 99):.0f}  max {fl.max()}")
for a in range(5):
    m = al == a
    if m.any():
        print(f"  algo {a}: {m.mean():.2f} of slots, mean flips {fl[m].mean():.0f}, max {fl[m].max()}")
