"""Pins for the oracle's iteration-dependent selection rules and tabu (-m "not gpu").

Round-1 review (VERDICT "What's weak" 1): eight mutants of oracle/dabs_oracle.c
in CyclicMin's window/cursor, RandomMin's p(t), MaxMin's D(t) and the tabu
period survived every pin.  The tests here tie each of those functions to the
paper's text, evaluated in the test on a state the test tracks itself:

* Delta is recomputed in the test from its DEFINITION, Delta_k = E(X xor e_k) -
  E(X), with E by a numpy einsum over the upper triangle (Eq.(2)
  read as R-1) -- never from the oracle's incremental values;
* the expected pick (deterministic rules) or the candidate set a pick must lie in
  (randomised rules) comes from the rule as the paper states it:
  MaxMin D(t) = (1-((T-t)/T)^3) minDelta + ((T-t)/T)^3 maxDelta, d ~ U[minDelta, D(t)]
  (P:408-424); CyclicMin w(t) = max((t/T)^3 n, c), window sliding on the circle
  (P:426-442); RandomMin p(t) = max((t/T)^3, 32/n); PositiveMin
  (P:455-462); tabu: "not flipped again in the next t iterations",
  SPEC's arithmetic example S:327-328;
* statistical pins compare pick frequencies with distributions derived
  analytically from those formulas (seeded, so deterministic).

Readings used: R-6 (MaxMin integer threshold; eligible = non-tabu),
R-7 (CyclicMin ceiling, clamp min(32, n), cursor 0 per run, lowest index),
R-8 (RandomMin integer p16, lowest-index argmin), R-9, R-11 (tabu = the slot's
last `tabu` flips in any phase, persisting across batches; dropped when the
eligible set is empty).

`tools/mutation_probe.py` rebuilds the oracle with each round-1 mutant and
checks that this file (with the other pins) rejects it.
"""
from fractions import Fraction

import numpy as np
import pytest

ALG_MAXMIN, ALG_CYCLIC, ALG_RANDOM, ALG_POSMIN, ALG_TWO = range(5)
PH_STRAIGHT, PH_GREEDY, PH_MAIN = 0, 1, 2


# ------------------------------------------------------------------ helpers
def E_def(U, X):
    """Eq.(2) (R-1) for a batch of vectors X [b, n]: x^T U x over the upper
    triangle.  float64 BLAS: every partial sum is an integer below 2^53 at the
    test sizes (|U| <= 300, n <= 300), so the result is exact."""
    Xf = X.astype(np.float64)
    e = ((Xf @ U.astype(np.float64)) * Xf).sum(1)
    assert np.abs(e).max(initial=0) < 2 ** 52
    return np.rint(e).astype(np.int64)


def delta_def(U, x):
    """Delta_k = E(X xor e_k) - E(X), by direct evaluation."""
    n = x.size
    Xn = np.tile(x.astype(np.int64), (n, 1))
    Xn[np.arange(n), np.arange(n)] ^= 1
    return E_def(U, Xn) - E_def(U, x[None])[0]


def diag_qubo(d):
    """U with only a diagonal: Delta_k = (1 - 2 x_k) d_k, and flipping bit i
    changes Delta_i only (it is negated)."""
    n = len(d)
    U = np.zeros((n, n), np.int16)
    U[np.arange(n), np.arange(n)] = d
    return U


def rand_upper(rng, n, lo=-300, hi=300):
    return np.triu(rng.integers(lo, hi + 1, size=(n, n))).astype(np.int16)


def w_paper(t, T, n, c=32):
    """CyclicMin window width: w(t) = max((t/T)^3 n, c), c < n; R-7:
    ceiling, c clamped to n for n <= 32, at most n."""
    w = -((-n * t ** 3) // T ** 3)          # ceil(n t^3 / T^3), exact integers
    return min(n, max(w, min(c, n)))


def p_paper(t, T, n):
    """RandomMin candidate probability: max((t/T)^3, 32/n), capped at 1."""
    return min(Fraction(1), max(Fraction(t ** 3, T ** 3), Fraction(32, n)))


def D_paper(t, T, lo, hi):
    """MaxMin's D(t), exact rational."""
    a = Fraction(T - t, T) ** 3
    return (1 - a) * lo + a * hi


class Replay:
    """Walks a batch trace with the test's own X, Delta (from the definition)
    and flip history, checking every main-phase pick against the paper's rule."""

    def __init__(self, U, x, history, tabu, T):
        self.U, self.x, self.hist, self.tabu, self.T = U, x.copy(), list(history), tabu, T
        self.n = x.size

    def eligible(self):
        last = set(self.hist[-self.tabu:]) if self.tabu else set()
        el = np.array([k not in last for k in range(self.n)])
        return el

    def apply(self, i):
        self.x[i] ^= 1
        self.hist.append(i)


def replay_batch(U, rep, r, algo, T, check_random=True):
    """Check every main-phase flip of batch result r (trace of bits and phases)."""
    n = U.shape[0]
    cursor = None
    t = 0
    last_phase = None
    checked = 0
    for ph, i in zip(r.trace_phase.tolist(), r.trace_bit.tolist()):
        if ph >= PH_MAIN:
            if ph != last_phase:           # a new main run: t and the window restart (R-7)
                t, cursor = 0, 0
            t += 1
            d = delta_def(U, rep.x)
            el = rep.eligible()
            if not el.any():
                el[:] = True               # tabu dropped when nothing is eligible (R-11)
            if algo == ALG_CYCLIC:
                w = w_paper(t, T, n)
                win = np.zeros(n, bool)
                win[(cursor + np.arange(w)) % n] = True
                cand = win & el
                if not cand.any():
                    cand = win
                dd = np.where(cand, d, np.iinfo(np.int64).max)
                assert i == int(np.argmin(dd)), (t, cursor, w, i, int(np.argmin(dd)))
                cursor = (cursor + w) % n
            elif algo == ALG_MAXMIN:
                lo, hi = int(d[el].min()), int(d[el].max())
                Dt = D_paper(t, T, lo, hi)
                assert el[i] and d[i] <= Dt, (t, i, int(d[i]), lo, hi, float(Dt))
                if t == T:                 # D(T) = minDelta: a minimum
                    assert d[i] == lo
            elif algo == ALG_RANDOM:
                assert el[i]
                if p_paper(t, T, n) == 1:  # every bit a candidate: the eligible argmin
                    dd = np.where(el, d, np.iinfo(np.int64).max)
                    assert i == int(np.argmin(dd))
            elif algo == ALG_POSMIN:
                pos = d[el & (d > 0)]
                pm = int(pos.min()) if pos.size else np.iinfo(np.int64).max
                assert el[i] and d[i] <= pm
            checked += 1
        last_phase = ph
        rep.apply(i)
    return checked


def run_and_replay(orc, U, algos, *, T, B, tabu, gens, seed, rng, D_zero=False):
    n = U.shape[0]
    total = 0
    for algo in algos:
        st = orc.SlotState.initial(U)
        rep = Replay(U, st.x, [], tabu, T)
        for gen in range(gens):
            D = np.zeros(n, np.uint8) if D_zero else rng.integers(0, 2, n).astype(np.uint8)
            r = orc.batch(U, st, D, algo, T=T, B=B, tabu=tabu, seed=seed, slot=2, gen=gen, trace_cap=200000)
            assert r.flips <= 200000
            total += replay_batch(U, rep, r, algo, T)
            assert np.array_equal(rep.x, st.x)
    return total


# ------------------------------------------------------------------ CyclicMin
def test_cyclicmin_scripted_window_n100():
    """P:426-442 (R-7): n=100, T=10, tabu 0, diagonal model at a local minimum
    with distinct Delta.  Each main flip is the argmin over the window
    [cursor, cursor + w(t)) mod n: w = 32 (the c clamp) for t <= 6, then 35,
    52, 73 and the full window 100 at t = T; the windows wrap past bit 99."""
    from oracle import oracle as orc
    rng = np.random.default_rng(5)
    n, T = 100, 10
    widths = [w_paper(t, T, n) for t in range(1, T + 1)]
    assert widths == [32, 32, 32, 32, 32, 32, 35, 52, 73, 100]
    starts = np.cumsum([0] + widths[:-1]) % n
    assert list(starts) == [0, 32, 64, 96, 28, 60, 92, 27, 79, 52]   # t=4, 7, 9 wrap
    for inst in range(6):
        d = (rng.permutation(n) + 1) * 7            # distinct, positive: X=0 is a local minimum
        U = diag_qubo(d)
        st = orc.SlotState.initial(U)
        r = orc.batch(U, st, np.zeros(n, np.uint8), ALG_CYCLIC, T=T, B=1, tabu=0, seed=inst, trace_cap=1000)
        main = [b for p, b in zip(r.trace_phase.tolist(), r.trace_bit.tolist()) if p >= PH_MAIN]
        assert len(main) == T
        delta = d.astype(np.int64).copy()
        for t in range(1, T + 1):
            win = (starts[t - 1] + np.arange(widths[t - 1])) % n
            exp = int(win[np.argmin(delta[win])])   # distinct values: no ties
            assert main[t - 1] == exp, (inst, t)
            delta[exp] = -delta[exp]                 # diagonal model: only Delta_i changes


def test_cyclicmin_small_n_is_full_window():
    """n <= c -> the window always covers all bits (global argmin)."""
    from oracle import oracle as orc
    rng = np.random.default_rng(6)
    for n in (5, 20, 32):
        assert all(w_paper(t, 40, n) == n for t in range(1, 41))
        U = rand_upper(rng, n)
        run_and_replay(orc, U, [ALG_CYCLIC], T=40, B=200, tabu=8, gens=3, seed=3, rng=rng)


@pytest.mark.parametrize("n,T,tabu", [(100, 10, 0), (100, 10, 8), (257, 26, 8), (70, 3, 8), (300, 30, 31)])
def test_cyclicmin_replay_random(n, T, tabu):
    """Every CyclicMin flip of several consecutive batches (random U, random
    targets, persistent slot) equals the paper's window argmin, evaluated on
    Delta from the definition with the test's own tabu history."""
    from oracle import oracle as orc
    rng = np.random.default_rng(n * 31 + T)
    U = rand_upper(rng, n)
    got = run_and_replay(orc, U, [ALG_CYCLIC], T=T, B=3 * n, tabu=tabu, gens=3, seed=11, rng=rng)
    assert got >= 3 * T


# ------------------------------------------------------------------ RandomMin
def test_randommin_candidate_probability():
    """P:446-453 ("expected n p(t) bits are selected"): with Delta
    increasing in the index and every flipped bit kept tabu for the whole run
    (tabu 31 > T), the flip at step t is the lowest-index candidate among the
    unflipped bits, so the number of unflipped bits below it is geometric with
    success probability p(t) = max((t/T)^3, 32/n).  n = 4096, T = 8:
    p = 1/128 (the 32/n floor) at t = 1, 1/64 at t = 2, 27/512, 1/8, ... 1 at t = T."""
    from oracle import oracle as orc
    n, T = 4096, 8
    U = diag_qubo(np.arange(1, n + 1))
    gaps = np.zeros((T,), float)
    sq = np.zeros((T,), float)
    N = 240
    for seed in range(N):
        st = orc.SlotState.initial(U)
        r = orc.batch(U, st, np.zeros(n, np.uint8), ALG_RANDOM, T=T, B=1, tabu=31, seed=seed, trace_cap=100)
        main = [b for p, b in zip(r.trace_phase.tolist(), r.trace_bit.tolist()) if p >= PH_MAIN]
        assert len(main) == T
        flipped = set()
        for t, i in enumerate(main):
            g = i - sum(1 for f in flipped if f < i)     # unflipped bits below the pick
            gaps[t] += g
            sq[t] += g * g
            flipped.add(i)
    for t in range(1, T + 1):
        p = float(p_paper(t, T, n))
        mean = gaps[t - 1] / N
        exp = (1 - p) / p
        sd = np.sqrt((1 - p) / p ** 2 / N)
        assert abs(mean - exp) <= 5 * sd + 0.05, (t, mean, exp, sd)


def test_randommin_floor_and_full_probability_are_argmin():
    """p(t) = 1 makes every eligible bit a candidate: the flip is the eligible
    argmin.  That holds at t = T for every n, and at every t when the
    32/n floor reaches 1 (n <= 32)."""
    from oracle import oracle as orc
    rng = np.random.default_rng(9)
    for n, T in ((12, 30), (32, 7), (200, 1)):
        U = rand_upper(rng, n)
        run_and_replay(orc, U, [ALG_RANDOM], T=T, B=4 * n, tabu=8, gens=3, seed=4, rng=rng)


# ------------------------------------------------------------------ MaxMin
def test_maxmin_threshold_distribution_t_lt_T():
    """P:408-424 at t < T: T = 2, t = 1, Delta_k = k + 1 over n = 801 bits
    (X = 0 of a diagonal model, a local minimum).  minDelta = 1, maxDelta = 801,
    D(1) = 7/8 * 1 + 1/8 * 801 = 101; d ~ U[1, 101] and the flip is uniform
    over {k : k + 1 <= d}.  With integer d (R-6) the pick k has probability
    sum_{d=k+1}^{101} 1/(101 d).  Chi-square over 4000 seeds; the second flip
    (t = T, D = minDelta over the non-tabu bits) is the lowest unflipped bit."""
    from oracle import oracle as orc
    n, T = 801, 2
    U = diag_qubo(np.arange(1, n + 1))
    assert D_paper(1, T, 1, 801) == 101
    N = 4000
    counts = np.zeros(101, int)
    for seed in range(N):
        st = orc.SlotState.initial(U)
        r = orc.batch(U, st, np.zeros(n, np.uint8), ALG_MAXMIN, T=T, B=1, tabu=8, seed=seed, trace_cap=100)
        main = [b for p, b in zip(r.trace_phase.tolist(), r.trace_bit.tolist()) if p >= PH_MAIN]
        assert len(main) == 2
        assert main[0] <= 100, main[0]            # Delta <= D(1) = 101
        counts[main[0]] += 1
        assert main[1] == (1 if main[0] == 0 else 0)
    p = np.array([sum(1.0 / (101 * d) for d in range(k + 1, 102)) for k in range(101)])
    assert abs(p.sum() - 1) < 1e-12
    # pool the tail bins so every expected count is >= 20
    exp = p * N
    cut = int(np.argmax(exp < 20))
    o = np.append(counts[:cut], counts[cut:].sum())
    e = np.append(exp[:cut], exp[cut:].sum())
    chi2 = float(((o - e) ** 2 / e).sum())
    dof = len(o) - 1
    assert chi2 < dof + 6 * np.sqrt(2 * dof), (chi2, dof)
    # the exponent: the threshold never passes D(1) but does reach its top decile
    assert counts[60:].sum() > 0


@pytest.mark.parametrize("n,T,tabu", [(60, 6, 8), (150, 15, 8), (40, 40, 0)])
def test_maxmin_replay_random(n, T, tabu):
    """Every MaxMin flip on random instances is a non-tabu bit with
    Delta <= D(t) (exact rational D(t) from the paper's formula, min/max over
    the eligible bits), and at t = T a minimum."""
    from oracle import oracle as orc
    rng = np.random.default_rng(n + 7 * T)
    U = rand_upper(rng, n)
    run_and_replay(orc, U, [ALG_MAXMIN], T=T, B=3 * n, tabu=tabu, gens=3, seed=8, rng=rng)


def test_maxmin_span_reaches_D_t():
    """The threshold d covers the whole of [minDelta, D(t)], not a
    sub-interval: at t = 1 of T = 4, D = lo + (27/64)(hi - lo).  Picks above
    lo + (1/8)(hi - lo) (the square-law value (1/2)^2... would give 9/16) must
    occur, none above D(1)."""
    from oracle import oracle as orc
    n, T = 1001, 4
    U = diag_qubo(np.arange(1, n + 1))
    Dt = D_paper(1, T, 1, n)
    assert Dt == 1 + Fraction(27, 64) * 1000
    mx = 0
    for seed in range(600):
        st = orc.SlotState.initial(U)
        r = orc.batch(U, st, np.zeros(n, np.uint8), ALG_MAXMIN, T=T, B=1, tabu=8, seed=seed, trace_cap=100)
        first = next(b for p, b in zip(r.trace_phase.tolist(), r.trace_bit.tolist()) if p >= PH_MAIN)
        assert first + 1 <= Dt
        mx = max(mx, first + 1)
    assert mx > 1 + 0.35 * 1000                   # the cube's 27/64 = 0.42 is reached


# ------------------------------------------------------------------ PositiveMin
@pytest.mark.parametrize("n,tabu", [(50, 8), (120, 0)])
def test_positivemin_replay_random(n, tabu):
    from oracle import oracle as orc
    rng = np.random.default_rng(n + tabu)
    U = rand_upper(rng, n)
    run_and_replay(orc, U, [ALG_POSMIN], T=max(1, n // 10), B=3 * n, tabu=tabu, gens=3, seed=8, rng=rng)


# ------------------------------------------------------------------ tabu
def _tabu_model(n=20):
    """Bit 0 has the smallest |Delta| (1); the others 1000 + k.  At X = 0 every
    Delta is positive (a local minimum)."""
    return diag_qubo(np.array([1] + [1000 + k for k in range(1, n)]))


@pytest.mark.parametrize("algo", [ALG_CYCLIC, ALG_RANDOM, ALG_POSMIN])
def test_tabu_period_spec_example(algo):
    """a bit flipped at count c is ineligible at
    c+1 .. c+8 and eligible at c+9 (period 8).  n = 20, so CyclicMin's window
    (n <= 32) and RandomMin's 32/n floor (>= 1) cover every bit: both flip the
    eligible argmin; PositiveMin flips a bit with Delta <= posmin.
    Main flip 1 = bit 0 (Delta 1 -> -1).  Flips 2..9: bit 0 is tabu, the
    argmin of the others are bits 1..8.  Flip 10: bit 0 is eligible again and
    its Delta = -1 is the minimum -> bit 0 (PositiveMin: posmin = 1009, so
    {0, 9} are the candidates)."""
    from oracle import oracle as orc
    U = _tabu_model()
    seen10 = set()
    for seed in range(40):
        st = orc.SlotState.initial(U)
        r = orc.batch(U, st, np.zeros(20, np.uint8), algo, T=12, B=1, tabu=8, seed=seed, trace_cap=100)
        main = [b for p, b in zip(r.trace_phase.tolist(), r.trace_bit.tolist()) if p >= PH_MAIN]
        assert main[:9] == list(range(9)), main
        if algo == ALG_POSMIN:
            assert main[9] in (0, 9)
            seen10.add(main[9])
        else:
            assert main[9] == 0, main
    if algo == ALG_POSMIN:
        assert seen10 == {0, 9}


@pytest.mark.parametrize("tabu", [0, 1, 5, 8, 13])
def test_tabu_period_general(tabu):
    """Period t: a bit flipped at main flip 1 is ineligible for exactly the
    next t flips.  The diagonal model above with n = 20: the
    CyclicMin full-window argmin returns to bit 0 at flip t + 2."""
    from oracle import oracle as orc
    U = _tabu_model()
    st = orc.SlotState.initial(U)
    r = orc.batch(U, st, np.zeros(20, np.uint8), ALG_CYCLIC, T=16, B=1, tabu=tabu, seed=0, trace_cap=100)
    main = [b for p, b in zip(r.trace_phase.tolist(), r.trace_bit.tolist()) if p >= PH_MAIN]
    assert main[0] == 0
    assert main[1:tabu + 1] == list(range(1, tabu + 1))
    assert main[tabu + 1] == 0


def test_tabu_persists_across_batches_and_phases():
    """R-11: the ring is slot state.  A bit flipped as the last flip of
    the previous batch (ring[0]) is ineligible for the first 8 flips of the
    next batch and eligible at the 9th."""
    from oracle import oracle as orc
    U = _tabu_model()
    st = orc.SlotState.initial(U)
    st.ring[0] = 0
    r = orc.batch(U, st, np.zeros(20, np.uint8), ALG_CYCLIC, T=12, B=1, tabu=8, seed=0, trace_cap=100)
    main = [b for p, b in zip(r.trace_phase.tolist(), r.trace_bit.tolist()) if p >= PH_MAIN]
    assert main[:8] == list(range(1, 9)) and main[8] == 0, main


def test_tabu_empty_eligible_set_falls_back():
    """R-11: n = 5 < period 8: after 5 flips every bit is tabu; the
    rule then ignores tabu (the search still progresses)."""
    from oracle import oracle as orc
    rng = np.random.default_rng(2)
    U = rand_upper(rng, 5)
    for algo in (ALG_MAXMIN, ALG_CYCLIC, ALG_RANDOM, ALG_POSMIN):
        run_and_replay(orc, U, [algo], T=20, B=60, tabu=8, gens=2, seed=1, rng=rng)


@pytest.mark.parametrize("algo", [ALG_MAXMIN, ALG_RANDOM, ALG_POSMIN, ALG_CYCLIC])
def test_no_tabu_bit_is_picked(algo):
    """Over long random runs no main flip picks one of the slot's last 8 flipped
    bits (any phase, across batches) while an eligible bit exists."""
    from oracle import oracle as orc
    rng = np.random.default_rng(40 + algo)
    n = 64
    U = rand_upper(rng, n)
    st = orc.SlotState.initial(U)
    hist = []
    for gen in range(4):
        D = rng.integers(0, 2, n).astype(np.uint8)
        r = orc.batch(U, st, D, algo, T=20, B=200, tabu=8, seed=2, slot=1, gen=gen, trace_cap=100000)
        for p, b in zip(r.trace_phase.tolist(), r.trace_bit.tolist()):
            if p >= PH_MAIN:
                assert b not in hist[-8:]
            hist.append(b)


# ------------------------------------------------------------------ adaptive choice
@pytest.mark.parametrize("eps_ppm", [0, 1000000])
def test_adaptive_choice_eps_extremes(eps_ppm):
    """eps = 0 -> every genop/algorithm is a pool row's tag;
    eps = 1 (1e6 ppm) -> always the uniform choice (the tags are ignored).
    Round-1 advisor: 1e6 ppm used to wrap the 32-bit threshold to 0 ("never")."""
    from oracle import oracle as orc
    rng = np.random.default_rng(4)
    n = 12
    U = rand_upper(rng, n)
    cfg = orc.Config(s_milli=100, b_milli=100, pools=1, slots=4000, cap=100, eps_ppm=eps_ppm)
    w = orc.World(U, cfg)
    w.reset(77)
    pool0 = w.pool(0)
    fg = np.bincount(pool0["genop"], minlength=8) / 100
    fa = np.bincount(pool0["algo"], minlength=5) / 100
    w.generation_local()
    d, _ = w.stats()
    d = d[0].astype(float)
    N = 4000
    got_g = d.sum(0)[:8] / N
    got_a = d.sum(1) / N
    if eps_ppm == 0:
        assert np.all(got_g[fg == 0] == 0) and np.all(got_a[fa == 0] == 0)
        pg, pa = fg, fa
    else:
        pg, pa = np.full(8, 1 / 8), np.full(5, 1 / 5)
    for p, q in zip(pg, got_g):
        assert abs(p - q) < 5 * np.sqrt(p * (1 - p) / N) + 1e-9
    for p, q in zip(pa, got_a):
        assert abs(p - q) < 5 * np.sqrt(p * (1 - p) / N) + 1e-9


# ------------------------------------------------------------------ ties and zero gains
def test_randommin_ties_lowest_index():
    """R-8 / SPEC design decisions (lowest index on argmin ties): on a +-1
    MaxCut-shaped model (many equal Delta) with n <= 32 (p = 1), every
    RandomMin flip is the LOWEST-index eligible minimum."""
    from oracle import oracle as orc
    rng = np.random.default_rng(12)
    n = 24
    U = np.zeros((n, n), np.int16)
    for i in range(n):
        for j in range(i + 1, n):
            w = int(rng.choice([-1, 1]))
            U[i, j] += 2 * w
            U[i, i] -= w
            U[j, j] -= w
    for algo in (ALG_RANDOM, ALG_CYCLIC):
        run_and_replay(orc, U, [algo], T=30, B=200, tabu=8, gens=4, seed=5, rng=rng)


def test_positivemin_zero_gain_is_not_positive():
    """posminDelta = min{Delta_i : Delta_i > 0} -- a zero gain is not
    positive.  Delta = [0, 3, 5] (a local minimum): posmin = 3, candidates
    {0, 1}, both picked about half of the time; bit 2 never."""
    from oracle import oracle as orc
    U = diag_qubo([0, 3, 5])
    counts = np.zeros(3, int)
    N = 2000
    for seed in range(N):
        st = orc.SlotState.initial(U)
        r = orc.batch(U, st, np.zeros(3, np.uint8), ALG_POSMIN, T=1, B=1, tabu=0, seed=seed, trace_cap=20)
        counts[next(b for p, b in zip(r.trace_phase.tolist(), r.trace_bit.tolist()) if p >= PH_MAIN)] += 1
    assert counts[2] == 0
    assert abs(counts[0] - N / 2) < 5 * np.sqrt(N / 4)
