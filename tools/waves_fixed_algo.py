"""Generation-schedule flips/s with ONE main algorithm (algo_mask), so the
adaptive mix cannot change with the slot count: isolates the wave/tail effect."""
import sys
sys.path.insert(0, ".")
from paper_2207_03069_b200 import Solver, workloads as wl

w = sys.argv[1]
algo = int(sys.argv[2])
U, meta = wl.make(w, seed=1)
for slots in [int(x) for x in sys.argv[3].split(",")]:
    s = Solver(U, s_milli=meta["s_milli"], b_milli=meta["b_milli"], slots=slots, algo_mask=1 << algo)
    s.reset(1)
    s.generation()
    s.generation()
    fl, ms = 0, 0.0
    for _ in range(3):
        f0 = s.stats().local_flips
        s.generation()
        st = s.stats()
        fl += st.local_flips - f0
        ms += st.batch_ms_last
    print(f"{w} algo={algo} slots={slots} flips/s={fl / (ms / 1e3):.4g} batch_ms/gen={ms / 3:.1f}", flush=True)
    s.close()
