"""Asynchronous schedule throughput and pool-lock profile per workload and pool count."""
import sys
sys.path.insert(0, ".")
from paper_2207_03069_b200 import Solver, workloads as wl
for w in sys.argv[1].split(","):
    for P in [int(x) for x in sys.argv[2].split(",")]:
        U, meta = wl.make(w, seed=1)
        csr = Solver.to_csr(U) if meta.get("sparse") else None
        s = Solver(None if csr else U, csr=csr, s_milli=meta["s_milli"], b_milli=meta["b_milli"], one_wave=True, pools=P)
        s.run_async(1, int(sys.argv[3]) // 4)
        s.run_async(1, int(sys.argv[3]))
        st = s.stats()
        wt, hd = s.async_lock_ns()
        print(f"{w} P={P} slots={s.slots} flips/s={st.total_flips / (st.batch_ms_last / 1e3):.4g} events={st.generations} "
              f"hold_us/ev={hd / 1e3 / st.generations:.2f} wait_us/ev={wt / 1e3 / st.generations:.1f} busy={hd / 1e6 / st.batch_ms_last / P:.2f}", flush=True)
        s.close()
