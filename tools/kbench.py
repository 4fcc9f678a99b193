"""Per-algorithm batch-kernel throughput (flips/s) on a workload: isolates the
effect of kernel changes from the adaptive algorithm mix."""
import sys
import os
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_2207_03069_b200 import Solver, workloads as wl  # noqa: E402

NAMES = ["MaxMin", "CyclicMin", "RandomMin", "PositiveMin", "TwoNeighbor"]


def main():
    cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["R32K", "K2000s"]
    gens = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    for cfg in cfgs:
        U, meta = wl.make(cfg, seed=1)
        res = []
        for a in range(5):
            s = Solver(U, s_milli=meta["s_milli"], b_milli=meta["b_milli"], pools=1, algo_mask=1 << a)
            s.reset(1)
            s.generation()          # from X = 0 (long Straight/Greedy)
            fl, ms = 0, 0.0
            for _ in range(gens):
                f0 = s.stats().local_flips
                s.generation()
                st = s.stats()
                fl += st.local_flips - f0
                ms += st.batch_ms_last
            res.append(f"{NAMES[a]}={fl / ms * 1e3 / 1e6:.1f}M")
            s.close()
        print(cfg, " ".join(res), flush=True)


if __name__ == "__main__":
    main()
