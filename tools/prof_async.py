"""One dabs_run_async launch for an ncu capture (async_kernel)."""
import sys
sys.path.insert(0, ".")
from paper_2207_03069_b200 import Solver, workloads as wl

w = sys.argv[1]
budget = int(sys.argv[2])
P = int(sys.argv[3]) if len(sys.argv) > 3 else 11
U, meta = wl.make(w, seed=1)
s = Solver(U, s_milli=meta["s_milli"], b_milli=meta["b_milli"], pools=P, one_wave=True)
s.run_async(1, budget)
st = s.stats()
print(f"{w} flips {st.total_flips} events {st.generations} kernel_ms {st.batch_ms_last}", flush=True)
