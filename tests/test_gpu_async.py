"""GPU parity of the asynchronous schedule (R-29):
dabs_run_async (one persistent kernel, pool lock, event log) vs the CPU
oracle's replay of the device's own event log.  The log fixes only the ORDER
of the merges; every batch, merge, seed, statistic and the run best are then
recomputed by the oracle and must agree bit-exactly.
"""
import numpy as np
import pytest

from test_gpu_parity import compare_world, rand_upper

pytestmark = pytest.mark.gpu
SEEDED = 1 << 31
XREAD = 1 << 30
SLOT = (1 << 30) - 1


@pytest.fixture(scope="module")
def lib():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2207_03069_b200 import build, dabs
    build.build()
    return dabs


def check_log(log, slots):
    s = log & SLOT
    assert s.max() < slots
    last = {}
    for e, v in enumerate(log):
        last[int(v & SLOT)] = e
    assert sorted(last) == list(range(slots)), "every slot merges at least once"
    for sl, e in last.items():
        assert not (log[e] & (SEEDED | XREAD)), "a slot's last event is a merge that seeds nothing"


def run_pair(orc, lib, U, P, S, seed, budget, one_wave=False, **kw):
    solver = lib.Solver(U, s_milli=100, b_milli=1000, pools=P, slots=S, cap=16, one_wave=one_wave, **kw)
    Eg, Xg = solver.run_async(seed, budget)
    log = solver.async_log()
    check_log(log, solver.slots)
    cfg = orc.Config(s_milli=100, b_milli=1000, pools=P, slots=solver.slots // P, cap=16,
                     **{k: v for k, v in kw.items() if k in ("genop_mask", "algo_mask")})
    w = orc.World(U, cfg)
    w.reset(seed)
    w.async_replay(log)
    compare_world(orc, solver, w, P, 1)
    Eo, Xo, rec = w.best()
    assert Eg == Eo
    np.testing.assert_array_equal(Xg, Xo)
    st = solver.stats()
    assert st.total_flips == w.total_flips
    assert (st.best_algo, st.best_genop, st.best_generation, st.best_slot) == (
        rec["algo"], rec["genop"], rec["gen"], rec["slot"])
    assert st.generations == len(log)
    return solver, log, st


@pytest.mark.parametrize("n,P,S", [(40, 1, 3), (300, 3, 5), (1024, 2, 4), (2100, 2, 3), (5000, 2, 2), (700, 4, 3)])
def test_async_parity(orc, lib, n, P, S):
    rng = np.random.default_rng(n + 1)
    U = rand_upper(rng, n, -200, 200)
    B = n   # b = 1
    solver, log, st = run_pair(orc, lib, U, P, S, seed=4242, budget=6 * P * S * B)
    assert st.total_flips >= 6 * P * S * B
    # the stop rule: seeding ends at the first merge that reaches the budget
    assert len(log) > P * S
    if P * S >= 12:
        assert (log & XREAD).any(), "Xrossover across pools exercised"


def test_async_parity_one_wave_warp_tier(orc, lib):
    """Every resident warp-tier search of the GPU as a persistent CTA
    (DABS_FLAG_ONE_WAVE), several pools, real lock contention."""
    n = 160
    U = rand_upper(np.random.default_rng(3), n, -50, 50)
    solver, log, st = run_pair(orc, lib, U, P=4, S=0, seed=9, budget=1, one_wave=True)
    assert solver.slots >= 148
    assert len(log) == solver.slots   # budget 1: every slot stops after its first batch


def test_async_parity_one_wave_many_batches(orc, lib):
    n = 96
    U = rand_upper(np.random.default_rng(5), n, -30, 30)
    solver, log, st = run_pair(orc, lib, U, P=2, S=0, seed=17, budget=0, one_wave=True)
    solver2, log2, st2 = run_pair(orc, lib, U, P=2, S=0, seed=17, budget=4 * solver.slots * 10 * n,
                                  one_wave=True)
    assert len(log2) >= 3 * solver2.slots


def test_async_target_stop(orc, lib):
    """The run stops seeding once the best reaches the target (K16 optimum)."""
    import itertools
    from paper_2207_03069_b200 import workloads as wl
    U = wl.random_dense(16, 1)
    X = np.array(list(itertools.product([0, 1], repeat=16)), np.int64)
    opt = int(np.einsum("bi,ij,bj->b", X, U.astype(np.int64), X).min())
    solver, log, st = run_pair(orc, lib, U, P=1, S=4, seed=3, budget=1 << 40, target=opt)
    assert st.best_energy == opt


def test_async_rejects(lib):
    U = rand_upper(np.random.default_rng(1), 50, -5, 5)
    s = lib.Solver(U, pools=1, slots=2, restart_gens=3)
    with pytest.raises(lib.DabsError):
        s.run_async(1, 1000)


@pytest.mark.parametrize("n", [5000, 9000])
def test_async_parity_cluster_tier(orc, lib, monkeypatch, n):
    """The asynchronous schedule on the 2-CTA cluster tier (forced for n > 4096):
    the cluster's rank-0 CTA commits, the peer learns the decision through
    DSMEM and a cluster barrier."""
    monkeypatch.setenv("DABS_CLUSTER", "1")
    U = rand_upper(np.random.default_rng(n), n, -300, 300)
    solver, log, st = run_pair(orc, lib, U, P=2, S=2, seed=77, budget=5 * 4 * n)
    assert solver.stats().threads_per_search >= 128
    assert len(log) > 4


def test_async_full_config_tsp32(orc, lib):
    """The bench's async launch configuration at full size (TSP32, n = 1024,
    11 pools, one wave of ~2365 persistent searches): a short run (every slot
    merges at least once) replayed by the oracle from the device's log."""
    from paper_2207_03069_b200 import workloads as wl
    U, meta = wl.make("TSP32", seed=1)
    solver = lib.Solver(U, s_milli=meta["s_milli"], b_milli=meta["b_milli"], pools=11, one_wave=True, cap=100)
    Eg, Xg = solver.run_async(5, 3 * solver.slots * U.shape[0])
    log = solver.async_log()
    check_log(log, solver.slots)
    w = orc.World(U, orc.Config(s_milli=meta["s_milli"], b_milli=meta["b_milli"], pools=11,
                                slots=solver.slots // 11, cap=100))
    w.reset(5)
    w.async_replay(log)
    compare_world(orc, solver, w, 11, 1)
    assert (Eg, Xg.tobytes()) == (w.best()[0], w.best()[1].tobytes())


def test_async_r64k_sampled(orc, lib):
    """n = 65536 (8 GiB W) on the TMEM tier's persistent kernel (one 512-thread
    CTA per SM, Delta in all 512 TMEM columns): with a budget of one flip every
    slot runs exactly its batch 0 from X = 0; two slots recomputed by the oracle."""
    from paper_2207_03069_b200 import workloads as wl
    U, meta = wl.make("R64K", seed=1)
    solver = lib.Solver(U, s_milli=meta["s_milli"], b_milli=meta["b_milli"], pools=1, one_wave=True)
    assert solver.stats().threads_per_search == 512
    solver.run_async(13, 1)
    log = solver.async_log()
    assert len(log) == solver.slots and not (log & (SEEDED | XREAD)).any()
    w = orc.World(U, orc.Config(s_milli=meta["s_milli"], b_milli=meta["b_milli"], pools=1, slots=solver.slots))
    w.reset(13)
    w.async_begin()
    for s in (0, solver.slots - 1):
        opk = w.packet(s)
        gpk = solver.read_packet(s)
        np.testing.assert_array_equal(gpk["D"], opk["D"])
        assert gpk["algo"] == opk["algo"]
        st = orc.SlotState.initial(U)
        ref = orc.batch(U, st, opk["D"], opk["algo"], T=solver.T, B=solver.B, tabu=8, seed=13, slot=s, gen=0)
        assert ref.flips == gpk["flips"] and ref.ebest == gpk["ebest"]
        np.testing.assert_array_equal(ref.best, gpk["best"])
        post = solver.read_slot(s)
        np.testing.assert_array_equal(st.x, post["x"])
        np.testing.assert_array_equal(st.delta, post["delta"])
        assert st.E == post["E"]
    solver.close()


def test_async_r32k_sampled(orc, lib):
    """R32K at full size (2 GiB W), one wave of 148 persistent searches: with a
    budget of one flip every slot runs exactly its batch 0 (from X = 0, packet
    0 drawn from the fresh pools); sampled slots recomputed by the oracle."""
    from paper_2207_03069_b200 import workloads as wl
    U, meta = wl.make("R32K", seed=1)
    solver = lib.Solver(U, s_milli=meta["s_milli"], b_milli=meta["b_milli"], pools=1, one_wave=True)
    solver.run_async(11, 1)
    log = solver.async_log()
    assert len(log) == solver.slots and not (log & (SEEDED | XREAD)).any()
    w = orc.World(U, orc.Config(s_milli=meta["s_milli"], b_milli=meta["b_milli"], pools=1, slots=solver.slots))
    w.reset(11)
    w.async_begin()
    for s in (0, solver.slots - 1):
        opk = w.packet(s)
        gpk = solver.read_packet(s)
        np.testing.assert_array_equal(gpk["D"], opk["D"])
        assert gpk["algo"] == opk["algo"]
        st = orc.SlotState.initial(U)
        ref = orc.batch(U, st, opk["D"], opk["algo"], T=solver.T, B=solver.B, tabu=8, seed=11, slot=s, gen=0)
        assert ref.flips == gpk["flips"] and ref.ebest == gpk["ebest"]
        np.testing.assert_array_equal(ref.best, gpk["best"])
        post = solver.read_slot(s)
        np.testing.assert_array_equal(st.x, post["x"])
        np.testing.assert_array_equal(st.delta, post["delta"])
        assert st.E == post["E"]
