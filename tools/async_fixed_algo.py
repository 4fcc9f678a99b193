"""Asynchronous vs generation schedule with ONE main rule (algo_mask): isolates
the schedules' kernel efficiency from the adaptive mix."""
import sys
sys.path.insert(0, ".")
from paper_2207_03069_b200 import Solver, workloads as wl

w, algo, P = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
U, meta = wl.make(w, seed=1)
g = Solver(U, s_milli=meta["s_milli"], b_milli=meta["b_milli"], algo_mask=1 << algo)
g.reset(1)
g.generation()
fl, ms = 0, 0.0
for _ in range(3):
    f0 = g.stats().local_flips
    g.generation()
    st = g.stats()
    fl += st.local_flips - f0
    ms += st.batch_ms_last
print(f"{w} algo={algo} generation slots={g.slots}: {fl / (ms / 1e3):.4g} flips/s", flush=True)
a = Solver(U, s_milli=meta["s_milli"], b_milli=meta["b_milli"], algo_mask=1 << algo, pools=P, one_wave=True)
a.run_async(1, fl // 4)
a.run_async(1, fl)
sa = a.stats()
print(f"{w} algo={algo} async P={P} slots={a.slots}: {sa.total_flips / (sa.batch_ms_last / 1e3):.4g} flips/s", flush=True)
