"""Pins of the oracle's asynchronous schedule (R-29):
replay of a merge-event log with no generation barrier.

* One slot in one pool: the asynchronous schedule IS the generation schedule
  (same seeds, batches, merges, seq numbers, first-best record), so the replay
  of [0|seeded]*(G-1) + [0] must equal G generations of the bulk-synchronous
  oracle, which is itself pinned in test_oracle_pins.py.
* Pools that share no genop (no Xrossover) evolve independently: any
  interleaving of their events gives the same pool contents.
* Invariants of every replay: pools sorted by (E, seq), finite entries unique
  and equal to Eq.(2) of their X, slots' Delta equal to Eq.(3), dispatch count
  = packets seeded, the run best = the best pool head.
"""
import numpy as np
import pytest

SEEDED = 1 << 31
XREAD = 1 << 30
SLOT = (1 << 30) - 1


def rand_upper(rng, n, lo=-100, hi=100):
    return np.triu(rng.integers(lo, hi + 1, size=(n, n))).astype(np.int16)


def E_matmul(U, X):
    U = U.astype(np.int64)
    X = X.astype(np.int64)
    return int(X @ U @ X)


def chain_log(slot, k):
    """k batches of one slot: k-1 seeded merges, then the final one."""
    return [slot | SEEDED] * (k - 1) + [slot]


def random_log(rng, ns, k_per_slot):
    """interleave each slot's k batches in a random order (slot order inside a
    slot is fixed by construction); no XREAD events (single pool, or genops
    without Xrossover)"""
    seq = []
    for s in range(ns):
        seq += [s] * k_per_slot[s]
    rng.shuffle(seq)
    left = list(k_per_slot)
    out = []
    for s in seq:
        left[s] -= 1
        out.append(s | (SEEDED if left[s] > 0 else 0))
    return out


def reactive_log(w, rng, ns, k_per_slot):
    """Drive the oracle event by event the way the device can: any slot may
    act next; a slot whose packet waits for the partner pool (Xrossover,
    R-29) acts with an XREAD event.  Returns the log."""
    w.async_begin()
    left = list(k_per_slot)
    pending = [0] * ns
    log = []
    while True:
        ready = [s for s in range(ns) if left[s] > 0 or pending[s]]
        if not ready:
            break
        s = int(rng.choice(ready))
        if pending[s]:
            entry = s | XREAD
        else:
            left[s] -= 1
            entry = s | (SEEDED if left[s] > 0 else 0)
        pending[s] = w.async_event(entry)
        log.append(entry)
    w.async_end()
    return log


@pytest.mark.parametrize("n,G", [(40, 6), (9, 10)])
def test_async_single_slot_equals_generations(orc, n, G):
    rng = np.random.default_rng(n)
    U = rand_upper(rng, n)
    cfg = orc.Config(s_milli=200, b_milli=1000, pools=1, slots=1, cap=16)
    gen = orc.System(U, cfg)
    gen.reset(7)
    for _ in range(G):
        gen.generation()
    wa = orc.World(U, cfg, checked=True)
    wa.reset(7)
    wa.async_replay(chain_log(0, G))
    wg = gen.ranks[0]
    for key in ("X", "E", "seq", "algo", "genop"):
        assert np.array_equal(wa.pool(0)[key], wg.pool(0)[key]), key
    Ea, Xa, ra = wa.best()
    Eg, Xg, rg = wg.best()
    assert Ea == Eg and np.array_equal(Xa, Xg) and ra == rg
    da, ia = wa.stats()
    dg, ig = wg.stats()
    assert np.array_equal(da, dg) and np.array_equal(ia, ig)
    sa, sg = wa.slot(0), wg.slot(0)
    assert sa.E == sg.E and np.array_equal(sa.x, sg.x) and np.array_equal(sa.delta, sg.delta)
    assert np.array_equal(sa.ring, sg.ring)
    assert wa.total_flips == wg.total_flips


def test_async_pools_without_xrossover_are_independent(orc):
    rng = np.random.default_rng(3)
    n = 30
    U = rand_upper(rng, n)
    mask = 0xFF & ~(1 << 2)   # no Xrossover: pools do not read each other
    cfg = orc.Config(s_milli=200, b_milli=1000, pools=2, slots=1, cap=8, genop_mask=mask)
    res = []
    for trial in range(3):
        w = orc.World(U, cfg)
        w.reset(11)
        w.async_replay(random_log(np.random.default_rng(trial), 2, [5, 4]))
        res.append([w.pool(p) for p in range(2)] + [w.slot(0), w.slot(1), w.stats()])
    for r in res[1:]:
        for p in range(2):
            for key in ("X", "E", "algo", "genop"):
                assert np.array_equal(r[p][key], res[0][p][key])
        for s in (2, 3):
            assert np.array_equal(r[s].x, res[0][s].x) and r[s].E == res[0][s].E
        assert np.array_equal(r[4][0], res[0][4][0]) and np.array_equal(r[4][1], res[0][4][1])


def test_async_invariants(orc):
    rng = np.random.default_rng(17)
    n = 36
    U = rand_upper(rng, n)
    cfg = orc.Config(s_milli=150, b_milli=800, pools=3, slots=3, cap=12)
    ns = cfg.pools * cfg.slots
    ks = [int(k) for k in rng.integers(2, 7, size=ns)]
    w = orc.World(U, cfg, checked=True)
    w.reset(21)
    log = reactive_log(w, rng, ns, ks)
    assert any(e & XREAD for e in log), "the case needs Xrossover packets across pools"
    # the log alone reproduces the run
    w2 = orc.World(U, cfg)
    w2.reset(21)
    w2.async_replay(log)
    for p in range(cfg.pools):
        for key in ("X", "E", "seq", "algo", "genop"):
            assert np.array_equal(w.pool(p)[key], w2.pool(p)[key])
    for s in range(ns):
        assert np.array_equal(w.packet(s)["D"], w2.packet(s)["D"])
    heads = []
    for p in range(cfg.pools):
        pool = w.pool(p)
        keys = list(zip(pool["E"].tolist(), pool["seq"].tolist()))
        assert keys == sorted(keys)
        fin = pool["E"] != orc.E_INF
        seen = set()
        for X, E in zip(pool["X"][fin], pool["E"][fin]):
            assert E == E_matmul(U, X)
            assert (int(E), X.tobytes()) not in seen
            seen.add((int(E), X.tobytes()))
        # results carry seq = (event+1)<<32 | slot, slot in this pool
        for sq in pool["seq"][fin]:
            e, s = int(sq) >> 32, int(sq) & 0xFFFFFFFF
            assert 1 <= e <= len(log) and s // cfg.slots == p and (log[e - 1] & SLOT) == s
            assert not (log[e - 1] & XREAD)
        heads.append(int(pool["E"][0]))
    E, X, rec = w.best()
    assert E == min(heads) == E_matmul(U, X)
    assert (log[rec["gen"]] & SLOT) == rec["slot"]
    d, ins = w.stats()
    assert d.sum() == ns + sum(1 for e in log if e & SEEDED)
    # an XREAD completes exactly the Xrossover packets whose partner is another pool
    merges = [e for e in log if not e & XREAD]
    assert len(merges) == sum(ks)
    assert (ins <= d).all()
    for s in range(ns):
        st = w.slot(s)
        assert st.E == E_matmul(U, st.x)
        assert np.array_equal(st.delta, orc.delta_closed(U, st.x))
    assert w.total_flips >= len(log)


def test_async_log_validation(orc):
    U = rand_upper(np.random.default_rng(1), 12)
    cfg = orc.Config(pools=1, slots=2, cap=4)
    bad = [
        [0 | SEEDED, 0, 1, 0],   # slot 0 after its final batch
        [0, 1 | SEEDED],          # slot 1 never finishes
        [0, 5],                   # no slot 5
        [0 | XREAD, 0, 1],        # XREAD without a pending Xrossover packet
    ]
    for log in bad:
        w = orc.World(U, cfg)
        w.reset(1)
        with pytest.raises(RuntimeError):
            w.async_replay(log)


def test_async_xread_step(orc):
    """The XREAD step of R-29 against the Philox definitions recomputed here:
    after it, D takes the partner pool's rank-r2 row (as the pool is at the
    XREAD) wherever GA mask word bit m0 is 0, and keeps its bits elsewhere
    (where the merge step put the own parent's bits, R-20)."""
    rng = np.random.default_rng(8)
    n = 45
    U = rand_upper(rng, n)
    cfg = orc.Config(s_milli=200, b_milli=600, pools=2, slots=2, cap=6, genop_mask=1 << 2, eps_ppm=0)
    seed = 99
    w = orc.World(U, cfg)
    w.reset(seed)
    w.async_begin()
    order = [0, 2, 1, 3, 0, 1, 2, 3]   # four slots, two batches each, merges then xreads
    k = {s: 0 for s in range(4)}
    checked = 0
    for s in order:
        last = k[s] == 1
        r = w.async_event(s | (0 if last else SEEDED))
        k[s] += 1
        if r:
            assert not last
            p = s // cfg.slots
            pn = (p + 1) % cfg.pools
            D0 = w.packet(s)["D"].copy()
            partner = w.pool(pn)["X"]
            assert w.async_event(s | XREAD) == 0
            D1 = w.packet(s)["D"]
            gen = k[s]
            key = [seed & 0xFFFFFFFF, seed >> 32]
            b = orc.philox([(3 << 24), s, gen, 0], key)          # PUR_GA_PARENT = 3
            r2 = orc.rank_pick(int(b[1]), cfg.cap)
            for bit in range(n):
                m = orc.philox([(4 << 24) | (bit // 32), s, gen, 0], key)   # PUR_GA_MASK = 4
                m0 = (int(m[0]) >> (bit % 32)) & 1
                assert D1[bit] == (D0[bit] if m0 else partner[r2][bit])
                if not m0:
                    assert D0[bit] == 0   # the merge step left the partner's bits empty
            checked += 1
    w.async_end()
    assert checked >= 2
