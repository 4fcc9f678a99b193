"""Jump-start (R-30) vs the plain generation schedule on one workload: per
generation device time, GEMM time, flips/s and the best energy after the same
number of generations (same seed)."""
import sys
import time
sys.path.insert(0, ".")
from paper_2207_03069_b200 import Solver, workloads as wl

w = sys.argv[1] if len(sys.argv) > 1 else "R32K"
gens = int(sys.argv[2]) if len(sys.argv) > 2 else 6
U, meta = wl.make(w, seed=1)
for jump in (False, True):
    s = Solver(U, s_milli=meta["s_milli"], b_milli=meta["b_milli"], jump=jump)
    s.reset(1)
    t0 = time.perf_counter()
    ms, bests = [], []
    for g in range(gens):
        s.generation()
        st = s.stats()
        ms.append(st.batch_ms_last)
        bests.append(st.best_energy)
    dt = time.perf_counter() - t0
    st = s.stats()
    print(f"{w} jump={jump} slots={s.slots} wall={dt:.3f}s flips={st.total_flips} flips/s(wall)={st.total_flips / dt:.4g} "
          f"batch_ms={[round(x, 1) for x in ms]} best={bests}", flush=True)
    s.close()
