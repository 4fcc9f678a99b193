"""Small runs for compute-sanitizer (race/sync/memory checks).

    compute-sanitizer --tool racecheck python tools/sanitize_case.py async
cases: async   -- dabs_run_async, n = 96, 2 pools, one wave (ticket locks, pool merge)
       cluster -- generations on the forced 2-CTA cluster tier, n = 5000 (DSMEM swaps, mbarriers)
       cta     -- R32K's tier, n = 16385: the TMEM tier (tm_batch_kernel: TMEM alloc, tcgen05.ld/st,
                  TMA rows, CTA exchange): a batch to a local minimum, then a short checked batch
                  (sanitize only the 2nd launch: --kernel-name kns=batch_kernel --launch-skip 1
                  --launch-count 1)
       ctareg  -- the same on the 512-thread register tier (DABS_TMEM=0)
       tmw     -- generations on the TMEM warp tier (DABS_TMW=1), n = 1000
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
    if case == "ctareg":
        os.environ["DABS_TMEM"] = "0"
        case = "cta"
    if case == "tmw":
        os.environ["DABS_TMW"] = "1"
        case = "warp"
    n = {"async": 96, "cluster": 5000, "cta": 16385, "warp": 1000}[case]
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
    elif case == "cta":
        s = Solver(U, s_milli=5, b_milli=20, pools=1, slots=1)
        rng = np.random.default_rng(1)
        st = orc.SlotState.initial(U)
        D = rng.integers(0, 2, n).astype(np.uint8)
        g = s.debug_batch(0, st.x, st.delta, st.E, st.ring, D, 1, seed=1, gen=0)
        st = orc.SlotState(g["x"], g["delta"], g["E"], g["ring"])
        D = st.x.copy()
        D[rng.choice(n, 20, replace=False)] ^= 1
        for algo in (1,):
            ref_st = st.copy()
            ref = orc.batch(U, ref_st, D, algo, T=s.T, B=s.B, tabu=8, seed=3, slot=0, gen=1)
            got = s.debug_batch(0, st.x, st.delta, st.E, st.ring, D, algo, seed=3, gen=1)
            assert got["flips"] == ref.flips and got["ebest"] == ref.ebest
            assert np.array_equal(got["delta"], ref_st.delta)
    else:
        P, S = 2, 3
        s = Solver(U, s_milli=100, b_milli=1000, pools=P, slots=S, cap=16)
        cfg = orc.Config(s_milli=100, b_milli=1000, pools=P, slots=S, cap=16)
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
