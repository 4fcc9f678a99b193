"""Small runs for compute-sanitizer (race/sync/memory checks).

    compute-sanitizer --tool racecheck python tools/sanitize_case.py async
cases: async   -- dabs_run_async, n = 96, 2 pools, one wave (ticket locks, pool merge)
       cluster -- generations on the forced 2-CTA cluster tier, n = 5000 (DSMEM swaps, mbarriers)
       cta     -- generations on the 512-thread CTA tier, n = 20000 (TMA rows, CTA exchange)
       warp    -- generations on the warp tier, n = 1000
Each case also checks its result against the CPU oracle (so a run that the
tool perturbs into a wrong answer fails loudly)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402


def main(case):
    from oracle import oracle as orc
    from paper_2207_03069_b200 import Solver, workloads as wl
    if case == "cluster":
        os.environ["DABS_CLUSTER"] = "1"
    n = {"async": 96, "cluster": 5000, "cta": 20000, "warp": 1000}[case]
    U = wl.random_dense(n, seed=3, lo=-200, hi=200)
    if case == "async":
        s = Solver(U, s_milli=100, b_milli=1000, pools=2, one_wave=True, cap=16)
        E, x = s.run_async(seed=5, flip_budget=200000)
        log = s.async_log()
        w = orc.World(U, orc.Config(s_milli=100, b_milli=1000, pools=2, slots=s.slots // 2, cap=16))
        w.reset(5)
        w.async_replay(log)
        Eo, _, _ = w.best()
        assert E == Eo, (E, Eo)
    else:
        P, S = 2, 3
        s = Solver(U, s_milli=100, b_milli=1000 if case != "cta" else 50, pools=P, slots=S, cap=16)
        cfg = orc.Config(s_milli=100, b_milli=1000 if case != "cta" else 50, pools=P, slots=S, cap=16)
        sysm = orc.System(U, cfg, world=1)
        s.reset(9)
        sysm.reset(9)
        for _ in range(2):
            s.generation()
            sysm.generation()
        assert s.best()[0] == sysm.ranks[0].best()[0]
    print(f"sanitize case {case}: ok (n = {n}, threads per search {s.threads})")


if __name__ == "__main__":
    main(sys.argv[1])
