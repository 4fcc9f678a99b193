"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, element by
element, on the same seeded inputs.  All arithmetic is integer, so the bar is
bit-exact: per-flip bit, E and phase; final X, Delta, E, tabu ring; BEST,
E(BEST), flip count; pools, packets and statistics per generation.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ALGS = range(5)


@pytest.fixture(scope="module")
def lib():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2207_03069_b200 import build, dabs
    build.build()
    return dabs


def rand_upper(rng, n, lo, hi):
    U = rng.integers(lo, hi + 1, size=(n, n)).astype(np.int16)
    return np.triu(U)


def random_state(orc, rng, U, n_ring):
    n = U.shape[0]
    st = orc.SlotState.initial(U)
    st.x[:] = rng.integers(0, 2, n)
    st.delta[:] = orc.delta_closed(U, st.x)
    st.E = orc.energy(U, st.x)
    ring = np.full(32, -1, np.int32)
    k = min(n_ring, 32)
    ring[:k] = rng.integers(0, n, k)
    st.ring[:] = ring
    return st


def compare_batch(orc, solver, U, st, D, algo, seed, gslot, gen, T, B, tabu):
    n = U.shape[0]
    cap = 4 * (B + 2 * n + 4 * n) + 1000
    st_gpu = st.copy()
    ref = orc.batch(U, st, D, algo, T=T, B=B, tabu=tabu, seed=seed, slot=gslot, gen=gen, trace_cap=cap)
    got = solver.debug_batch(gslot - 0, st_gpu.x, st_gpu.delta, st_gpu.E, st_gpu.ring, D, algo, seed, gen,
                             trace_cap=cap)
    tag = f"n={n} algo={algo} seed={seed}"
    assert got["flips"] == ref.flips, tag
    m = min(ref.flips, cap)
    np.testing.assert_array_equal(got["trace_bit"][:m], ref.trace_bit[:m], err_msg=tag)
    np.testing.assert_array_equal(got["trace_E"][:m], ref.trace_E[:m], err_msg=tag)
    np.testing.assert_array_equal(got["trace_phase"][:m], ref.trace_phase[:m], err_msg=tag)
    np.testing.assert_array_equal(got["x"], st.x, err_msg=tag)
    np.testing.assert_array_equal(got["delta"], st.delta, err_msg=tag)
    assert got["E"] == st.E, tag
    np.testing.assert_array_equal(got["ring"], st.ring, err_msg=tag)
    assert got["ebest"] == ref.ebest, tag
    np.testing.assert_array_equal(got["best"], ref.best, err_msg=tag)


# sizes spanning every tier and ragged tails: warp tier C=1,2,4,8 and the CTA tier
SIZES = [1, 2, 7, 16, 33, 255, 256, 257, 700, 1024, 1500, 2048, 2049, 5000, 9000]


@pytest.mark.parametrize("n", SIZES)
def test_batch_parity(orc, lib, n):
    rng = np.random.default_rng(1000 + n)
    lo, hi = (-32767, 32767) if n <= 32768 // 2 else (-100, 100)
    if n > 2048:
        lo, hi = -3000, 3000
    U = rand_upper(rng, n, lo, hi)
    s_milli, b_milli, tabu = 150, 1500, 8
    solver = lib.Solver(U, s_milli=s_milli, b_milli=b_milli, tabu=tabu, pools=1, slots=2)
    T, B = solver.T, solver.B
    assert (T, B) == (orc.flip_factor(s_milli, n), orc.flip_factor(b_milli, n))
    for algo in ALGS:
        for rep in range(2):
            st = random_state(orc, rng, U, n_ring=rep * 5)
            D = rng.integers(0, 2, n).astype(np.uint8)
            seed = int(rng.integers(0, 2**63))
            compare_batch(orc, solver, U, st, D, algo, seed, gslot=1, gen=int(rng.integers(0, 1000)),
                          T=T, B=B, tabu=tabu)
    solver.close()


@pytest.fixture
def cluster_tier(monkeypatch):
    """Force the 2-CTA cluster tier for every n > 4096."""
    monkeypatch.setenv("DABS_CLUSTER", "1")


@pytest.mark.parametrize("n", [4097, 9000, 20000])
def test_batch_parity_cluster_forced(orc, lib, cluster_tier, n):
    """The cluster tier (two CTAs per search, DSMEM swaps) at sizes the
    single-CTA tier also covers: same bit-exact bar."""
    from paper_2207_03069_b200 import workloads as wl
    rng = np.random.default_rng(2000 + n)
    U = wl.random_dense(n, seed=n, lo=-3000, hi=3000)
    solver = lib.Solver(U, s_milli=150, b_milli=1500, pools=1, slots=2)
    assert solver.stats().threads_per_search >= 128
    for algo in ALGS:
        st = random_state(orc, rng, U, n_ring=5)
        D = rng.integers(0, 2, n).astype(np.uint8)
        compare_batch(orc, solver, U, st, D, algo, int(rng.integers(0, 2**63)), gslot=1,
                      gen=int(rng.integers(0, 1000)), T=solver.T, B=solver.B, tabu=8)
    solver.close()


@pytest.mark.parametrize("n", [513, 1000, 1024, 1500, 2048])
def test_batch_parity_tmem_warp_tier(orc, lib, monkeypatch, n):
    """The TMEM warp tier (DABS_TMW=1: 4 warp-searches per CTA, Delta in tensor
    memory; an A/B variant, off by default): every rule per flip, same bar."""
    monkeypatch.setenv("DABS_TMW", "1")
    rng = np.random.default_rng(3000 + n)
    U = rand_upper(rng, n, -32767, 32767)
    solver = lib.Solver(U, s_milli=150, b_milli=1500, tabu=8, pools=1, slots=2)
    assert solver.stats().threads_per_search == 32
    for algo in ALGS:
        st = random_state(orc, rng, U, n_ring=5)
        D = rng.integers(0, 2, n).astype(np.uint8)
        compare_batch(orc, solver, U, st, D, algo, int(rng.integers(0, 2**63)), gslot=1,
                      gen=int(rng.integers(0, 1000)), T=solver.T, B=solver.B, tabu=8)
    solver.close()


@pytest.fixture(scope="module")
def r64k():
    from paper_2207_03069_b200 import workloads as wl
    return wl.make("R64K", seed=1)[0]


@pytest.mark.parametrize("tier", ["cluster", "tmem64"])
@pytest.mark.parametrize("n", [32769, 65536])
def test_batch_parity_large_n(orc, lib, r64k, monkeypatch, tier, n):
    """n > 32768: one 512-thread CTA per SM with all of Delta (256 KB) in tensor
    memory (the default), or the cluster tier (DABS_TMEM64=0, two CTAs per search).
    Short batches (s = b = 0.001, D = X with 40 bits changed) keep the oracle
    at seconds per batch; the search starts at X = 0 (Delta = diag)."""
    from paper_2207_03069_b200 import workloads as wl
    monkeypatch.setenv("DABS_TMEM64", "1" if tier == "tmem64" else "0")
    rng = np.random.default_rng(3000 + n)
    U = r64k if n == 65536 else wl.random_dense(n, seed=n, lo=-3000, hi=3000)
    solver = lib.Solver(U, s_milli=1, b_milli=1, pools=1, slots=1)
    assert solver.stats().threads_per_search == (1024 if tier == "cluster" else 512)
    st0 = orc.SlotState.initial(U)
    for algo in ALGS:
        st = st0.copy()
        D = st.x.copy()
        D[rng.choice(n, 40, replace=False)] ^= 1
        compare_batch(orc, solver, U, st, D, algo, int(rng.integers(0, 2**63)), gslot=0, gen=algo,
                      T=solver.T, B=solver.B, tabu=8)
        st0 = st                                # continue from the local minimum reached
    solver.close()


@pytest.mark.parametrize("n", [16, 200])
def test_batch_parity_structured(orc, lib, n):
    """MaxCut-shaped (+-1, many ties) and zero-plateau instances stress the
    lowest-index tie rules and the PositiveMin/MaxMin candidate counting."""
    from paper_2207_03069_b200 import workloads as wl
    rng = np.random.default_rng(n)
    U, _, _ = wl.complete_pm1(n, seed=n)
    solver = lib.Solver(U, s_milli=100, b_milli=3000, pools=1, slots=1)
    for algo in ALGS:
        st = random_state(orc, rng, U, n_ring=0)
        D = rng.integers(0, 2, n).astype(np.uint8)
        compare_batch(orc, solver, U, st, D, algo, 77, 0, 3, solver.T, solver.B, 8)
    # zero-diagonal, sparse: many Delta = 0
    U = np.zeros((n, n), np.int16)
    idx = rng.integers(0, n, size=(n, 2))
    for a, b in idx:
        if a != b:
            U[min(a, b), max(a, b)] = rng.choice([-1, 1])
    solver = lib.Solver(U, s_milli=100, b_milli=3000, pools=1, slots=1, tabu=3)
    for algo in ALGS:
        st = random_state(orc, rng, U, n_ring=2)
        D = rng.integers(0, 2, n).astype(np.uint8)
        compare_batch(orc, solver, U, st, D, algo, 5, 0, 1, solver.T, solver.B, 3)


def test_energy_parity(orc, lib):
    rng = np.random.default_rng(3)
    for n in (1, 5, 300, 2049):
        U = rand_upper(rng, n, -32767, 32767) if n < 1000 else rand_upper(rng, n, -100, 100)
        solver = lib.Solver(U, pools=1, slots=1)
        for _ in range(5):
            x = rng.integers(0, 2, n).astype(np.uint8)
            assert solver.energy(x) == orc.energy(U, x)
        solver.close()


def test_create_errors(lib):
    U = np.zeros((4, 4), np.int16)
    U[2, 1] = 1
    with pytest.raises(lib.DabsError, match="E_TRIANGLE"):
        lib.Solver(U)
    with pytest.raises(lib.DabsError, match="E_ARG"):
        lib.Solver(np.zeros((0, 0), np.int16))
    with pytest.raises(lib.DabsError, match="E_ARG"):
        lib.Solver(np.zeros((4, 4), np.int16), tabu=40)
    # |Delta_k| <= |W_kk| + sum_j |W_kj| <= n * 32768: only n = 65536 with
    # -32768 weights reaches 2^31 (checked via CSR: one full row)
    n = 65536
    rp = np.zeros(n + 1, np.int32)
    rp[1:] = n - 1
    col = np.arange(1, n, dtype=np.int32)
    val = np.full(n - 1, -32768, np.int16)
    diag = np.zeros(n, np.int16)
    diag[0] = -32768
    with pytest.raises(lib.DabsError, match="E_RANGE"):
        lib.Solver(None, csr=(rp, col, val, diag))
    val[:] = 32767                              # 32768 + 65535 * 32767 < 2^31 - 1: accepted
    lib.Solver(None, csr=(rp, col, val, diag), pools=1, slots=1).close()
    rp2 = np.zeros(n + 2, np.int32)
    with pytest.raises(lib.DabsError, match="E_ARG"):
        lib.Solver(None, csr=(rp2, col[:0], val[:0], np.zeros(n + 1, np.int16)))


def compare_world(orc, solver, ow, P, gens_done):
    for p in range(P + 1):
        g = solver.read_pool(p)
        r = ow.pool(p)
        for k in ("E", "seq", "algo", "genop"):
            np.testing.assert_array_equal(g[k], r[k], err_msg=f"pool {p} {k} gen {gens_done}")
        np.testing.assert_array_equal(g["X"], r["X"], err_msg=f"pool {p} X gen {gens_done}")
    for s in range(solver.slots):
        g = solver.read_slot(s)
        r = ow.slot(s)
        np.testing.assert_array_equal(g["x"], r.x)
        np.testing.assert_array_equal(g["delta"], r.delta)
        assert g["E"] == r.E
        np.testing.assert_array_equal(g["ring"], r.ring)
        if gens_done == 0:
            continue
        gp = solver.read_packet(s)
        rp = ow.packet(s)
        for k in ("algo", "genop", "ebest", "flips"):
            assert gp[k] == rp[k], (s, k)
        np.testing.assert_array_equal(gp["D"], rp["D"])
        np.testing.assert_array_equal(gp["best"], rp["best"])
    d_ref, i_ref = ow.stats()
    for p in range(P):
        d, i = solver.read_stats_pool(p)
        np.testing.assert_array_equal(d, d_ref[p])
        np.testing.assert_array_equal(i, i_ref[p])


@pytest.mark.parametrize("n,P,S,gens", [(40, 2, 7, 6), (300, 3, 5, 4), (2100, 2, 3, 2)])
def test_generation_parity(orc, lib, n, P, S, gens):
    rng = np.random.default_rng(n)
    U = rand_upper(rng, n, -200, 200)
    cfg = orc.Config(s_milli=100, b_milli=1000, pools=P, slots=S, cap=20)
    sysm = orc.System(U, cfg, world=1)
    solver = lib.Solver(U, s_milli=100, b_milli=1000, pools=P, slots=S, cap=20)
    seed = 12345
    sysm.reset(seed)
    solver.reset(seed)
    compare_world(orc, solver, sysm.ranks[0], P, 0)
    for g in range(gens):
        sysm.generation()
        solver.generation()
        compare_world(orc, solver, sysm.ranks[0], P, g + 1)
        Eo, Xo, reco = sysm.ranks[0].best()
        Eg, Xg = solver.best()
        assert Eg == Eo
        np.testing.assert_array_equal(Xg, Xo)
        st = solver.stats()
        assert st.total_flips == sysm.ranks[0].total_flips
        assert (st.best_algo, st.best_genop, st.best_generation, st.best_slot) == (
            reco["algo"], reco["genop"], reco["gen"], reco["slot"])


@pytest.mark.parametrize("variant", ["abs", "restart"])
def test_generation_parity_variants(orc, lib, variant):
    """SURVEY f4 variants: the ABS ablation mode (CyclicMin only + mutation
    after crossover, R-27) and restart-on-merge (R-28), whole generations."""
    n, P, S = 60, 2, 3
    rng = np.random.default_rng(77)
    U = rand_upper(rng, n, -20, 20)
    kw = dict(genop_mask=1 << 8, algo_mask=1 << 1) if variant == "abs" else dict(restart_gens=2)
    cfg = orc.Config(s_milli=100, b_milli=1000, pools=P, slots=S, cap=8, **kw)
    sysm = orc.System(U, cfg, world=1)
    solver = lib.Solver(U, s_milli=100, b_milli=1000, pools=P, slots=S, cap=8, **kw)
    sysm.reset(21)
    solver.reset(21)
    for g in range(25):
        sysm.generation()
        solver.generation()
        compare_world(orc, solver, sysm.ranks[0], P, g + 1)
        assert solver.stats().restarts == sysm.ranks[0].restarts
        assert solver.best()[0] == sysm.ranks[0].best()[0]
    if variant == "restart":
        assert sysm.ranks[0].restarts >= 1


def test_generation_parity_cluster(orc, lib, cluster_tier):
    """Whole generations (GA, batches, merge) on the cluster tier."""
    n, P, S = 5000, 2, 3
    rng = np.random.default_rng(n)
    U = rand_upper(rng, n, -200, 200)
    cfg = orc.Config(s_milli=100, b_milli=1000, pools=P, slots=S, cap=20)
    sysm = orc.System(U, cfg, world=1)
    solver = lib.Solver(U, s_milli=100, b_milli=1000, pools=P, slots=S, cap=20)
    sysm.reset(9)
    solver.reset(9)
    for g in range(2):
        sysm.generation()
        solver.generation()
        compare_world(orc, solver, sysm.ranks[0], P, g + 1)
    assert solver.stats().total_flips == sysm.ranks[0].total_flips


def test_k16_run_parity_and_optimum(orc, lib):
    """Config K16: single search; GPU run == oracle run, and it reaches the
    brute-force optimum over all 65536 vectors."""
    import itertools
    from paper_2207_03069_b200 import workloads as wl
    U = wl.random_dense(16, 1)
    X = np.array(list(itertools.product([0, 1], repeat=16)), np.int64)
    opt = int(np.einsum("bi,ij,bj->b", X, U.astype(np.int64), X).min())
    cfg = orc.Config(s_milli=100, b_milli=10000, pools=1, slots=1)
    Eo, Xo, _ = orc.System(U, cfg).run(seed=1, flip_budget=10**9, target=opt)
    solver = lib.Solver(U, s_milli=100, b_milli=10000, pools=1, slots=1, target=opt)
    Eg, Xg = solver.run(seed=1, flip_budget=10**9)
    assert Eg == Eo == opt
    np.testing.assert_array_equal(Xg, Xo)


SAMPLED = [("GS800", 2), ("TSP32", 2), ("K2000s", 2)]


@pytest.mark.parametrize("config,gens", SAMPLED)
def test_full_size_sampled_parity(orc, lib, config, gens):
    """Bench launch configuration (auto slots, one pool): run generations on the
    GPU, then recompute sampled slots' batches of the last generation on the
    oracle from the pre-generation state."""
    from paper_2207_03069_b200 import workloads as wl
    U, meta = wl.make(config, seed=1)
    solver = lib.Solver(U, s_milli=meta["s_milli"], b_milli=meta["b_milli"], pools=1)
    solver.reset(7)
    for _ in range(gens - 1):
        solver.generation()
    rng = np.random.default_rng(0)
    sample = sorted(set([0, solver.slots - 1] + list(rng.integers(0, solver.slots, 4))))
    pre = {s: solver.read_slot(s) for s in sample}
    solver.generation()
    for s in sample:
        pk = solver.read_packet(s)
        post = solver.read_slot(s)
        st = orc.SlotState(pre[s]["x"].copy(), pre[s]["delta"].copy(), pre[s]["E"], pre[s]["ring"].copy())
        ref = orc.batch(U, st, pk["D"], pk["algo"], T=solver.T, B=solver.B, tabu=8, seed=7, slot=s,
                        gen=gens - 1)
        assert ref.flips == pk["flips"]
        assert ref.ebest == pk["ebest"]
        np.testing.assert_array_equal(ref.best, pk["best"])
        np.testing.assert_array_equal(st.x, post["x"])
        np.testing.assert_array_equal(st.delta, post["delta"])
        assert st.E == post["E"]


def test_r32k_sampled_parity(orc, lib):
    """Config R32K at full size (2 GiB W): one sampled slot of the bench launch
    recomputed by the oracle."""
    from paper_2207_03069_b200 import workloads as wl
    U, meta = wl.make("R32K", seed=1)
    solver = lib.Solver(U, s_milli=meta["s_milli"], b_milli=meta["b_milli"], pools=1)
    solver.reset(3)
    s = solver.slots // 2
    pre = solver.read_slot(s)
    solver.generation()
    pk = solver.read_packet(s)
    post = solver.read_slot(s)
    st = orc.SlotState(pre["x"].copy(), pre["delta"].copy(), pre["E"], pre["ring"].copy())
    ref = orc.batch(U, st, pk["D"], pk["algo"], T=solver.T, B=solver.B, tabu=8, seed=3, slot=s, gen=0)
    assert ref.flips == pk["flips"] and ref.ebest == pk["ebest"]
    np.testing.assert_array_equal(ref.best, pk["best"])
    np.testing.assert_array_equal(st.x, post["x"])
    np.testing.assert_array_equal(st.delta, post["delta"])
    # property at any size: E(BEST) equals Eq.(2) evaluated directly on the device
    assert solver.energy(pk["best"]) == pk["ebest"]


def test_r64k_sampled_properties(orc, lib, r64k):
    """n = 65536 (the boundary's maximum, cluster tier; 8 GiB W) in the bench
    launch configuration.  A whole oracle batch at this size takes minutes
    (test_batch_parity_large_n covers the tier with short batches), so here the
    oracle checks sampled outputs one by one: E(BEST) and E(X) by Eq.(2), and
    sampled Delta_k = E(X xor e_k) - E(X) (Eq.(3))."""
    U = r64k
    solver = lib.Solver(U, s_milli=100, b_milli=1000, pools=1)
    solver.reset(4)
    solver.generation()
    s = solver.slots - 1
    pk = solver.read_packet(s)
    post = solver.read_slot(s)
    assert pk["flips"] >= solver.B
    assert orc.energy(U, pk["best"]) == pk["ebest"]
    e0 = orc.energy(U, post["x"])
    assert e0 == post["E"]
    rng = np.random.default_rng(0)
    for k in rng.choice(U.shape[0], 3, replace=False):
        x1 = post["x"].copy()
        x1[k] ^= 1
        assert orc.energy(U, x1) - e0 == post["delta"][k]


def test_csr_ingest_equals_dense(orc, lib):
    """dabs_create_csr builds the same device rows as dabs_create:
    identical generations; its input checks report the documented errors."""
    from paper_2207_03069_b200 import workloads as wl
    U, _, _ = wl.gset_like(300, 2000, seed=4)
    csr = lib.Solver.to_csr(U)
    a = lib.Solver(U, pools=2, slots=5, cap=16)
    b = lib.Solver(None, csr=csr, pools=2, slots=5, cap=16)
    for s_ in (a, b):
        s_.reset(3)
        for _ in range(3):
            s_.generation()
    for p in range(3):
        np.testing.assert_array_equal(a.read_pool(p)["X"], b.read_pool(p)["X"])
        np.testing.assert_array_equal(a.read_pool(p)["E"], b.read_pool(p)["E"])
    x = np.random.default_rng(0).integers(0, 2, 300).astype(np.uint8)
    assert a.energy(x) == b.energy(x) == orc.energy(U, x)
    rp, col, val, diag = csr
    bad = col.copy()
    bad[0] = 0                                  # row 0 column 0: not above the diagonal
    with pytest.raises(lib.DabsError, match="E_TRIANGLE"):
        lib.Solver(None, csr=(rp, bad, val, diag))
    bad = col.copy()
    bad[1] = bad[0]                             # duplicate column in row 0
    with pytest.raises(lib.DabsError, match="E_ARG"):
        lib.Solver(None, csr=(rp, bad, val, diag))


def test_qasp_sampled_parity(orc, lib):
    """QASP-shaped sparse Ising through dabs_create_csr, bench
    launch configuration: sampled slots of generation 1 recomputed by the oracle."""
    from paper_2207_03069_b200 import workloads as wl
    U, meta = wl.make("QASP16", seed=1)
    solver = lib.Solver(None, csr=lib.Solver.to_csr(U), s_milli=meta["s_milli"], b_milli=meta["b_milli"])
    solver.reset(5)
    solver.generation()
    sample = [0, solver.slots // 3, solver.slots - 1]
    pre = {s: solver.read_slot(s) for s in sample}
    solver.generation()
    for s in sample:
        pk = solver.read_packet(s)
        post = solver.read_slot(s)
        st = orc.SlotState(pre[s]["x"].copy(), pre[s]["delta"].copy(), pre[s]["E"], pre[s]["ring"].copy())
        ref = orc.batch(U, st, pk["D"], pk["algo"], T=solver.T, B=solver.B, tabu=8, seed=5, slot=s, gen=1)
        assert ref.flips == pk["flips"] and ref.ebest == pk["ebest"]
        np.testing.assert_array_equal(ref.best, pk["best"])
        np.testing.assert_array_equal(st.delta, post["delta"])
    E, x = solver.best()
    assert solver.energy(x) == E == orc.energy(U, x)


@pytest.mark.parametrize("n,P,S,gens", [(40, 2, 5, 5), (300, 2, 4, 3), (2100, 2, 3, 2), (5000, 1, 3, 2),
                                        (1000, 2, 150, 2)])
def test_generation_parity_jump_start(orc, lib, n, P, S, gens):
    """SURVEY f4 jump-start (R-30): X = D, E(D), Delta(D) from the tcgen05 int8
    tensor-core GEMM, then the batch; whole generations vs the oracle."""
    rng = np.random.default_rng(n + 7)
    U = rand_upper(rng, n, -32767, 32767) if n >= 2100 else rand_upper(rng, n, -200, 200)
    cfg = orc.Config(s_milli=100, b_milli=1000, pools=P, slots=S, cap=12, jump=True)
    sysm = orc.System(U, cfg, world=1)
    solver = lib.Solver(U, s_milli=100, b_milli=1000, pools=P, slots=S, cap=12, jump=True)
    sysm.reset(31)
    solver.reset(31)
    for g in range(gens):
        sysm.generation()
        solver.generation()
        compare_world(orc, solver, sysm.ranks[0], P, g + 1)
    assert solver.stats().total_flips == sysm.ranks[0].total_flips
    assert solver.best()[0] == sysm.ranks[0].best()[0]


def test_r32k_sampled_parity_jump(orc, lib):
    """Jump-start (R-30) at full size: R32K's int16 weights in [-32767, 32767]
    exercise the exact int8 byte-split contraction at its largest partial sums
    (n * 128 = 2^22); one sampled slot of the bench launch recomputed by the
    oracle (X = D, E and Delta from Eqs.(2)/(3), then the batch)."""
    from paper_2207_03069_b200 import workloads as wl
    U, meta = wl.make("R32K", seed=1)
    solver = lib.Solver(U, s_milli=meta["s_milli"], b_milli=meta["b_milli"], pools=1, jump=True)
    solver.reset(4)
    solver.generation()
    s = solver.slots // 3
    pre = solver.read_slot(s)
    solver.generation()
    pk = solver.read_packet(s)
    post = solver.read_slot(s)
    st = orc.SlotState(pre["x"].copy(), pre["delta"].copy(), pre["E"], pre["ring"].copy())
    ref = orc.batch(U, st, pk["D"], pk["algo"], T=solver.T, B=solver.B, tabu=8, seed=4, slot=s, gen=1, jump=True)
    assert ref.flips == pk["flips"] and ref.ebest == pk["ebest"]
    np.testing.assert_array_equal(ref.best, pk["best"])
    np.testing.assert_array_equal(st.x, post["x"])
    np.testing.assert_array_equal(st.delta, post["delta"])
    assert st.E == post["E"]
