"""Pins of the oracle's jump-start variant (R-30):
the batch starts at its target D (X <- D) instead of walking there with
Straight's flips.

* The jump state is the state Straight reaches: flipping the differing bits
  one at a time through the incremental update (Eqs.(4)-(5), orc_step_flip)
  lands on the same X, E and Delta as the jump's direct Eq.(2)/(3) evaluation.
* A jump-start batch equals a normal batch started from X = D (where
  Straight has nothing to do): same flips, trace, BEST.
* Jump-start runs still reach the brute-force optimum of small instances.
"""
import itertools

import numpy as np


def rand_upper(rng, n, lo=-100, hi=100):
    return np.triu(rng.integers(lo, hi + 1, size=(n, n))).astype(np.int16)


def test_jump_state_equals_straight_path(orc):
    rng = np.random.default_rng(4)
    for n in (5, 17, 64):
        U = rand_upper(rng, n)
        st = orc.SlotState.initial(U)
        st.x[:] = rng.integers(0, 2, n)
        st.delta[:] = orc.delta_closed(U, st.x)
        st.E = orc.energy(U, st.x)
        D = rng.integers(0, 2, n).astype(np.uint8)
        walk = st.copy()
        for k in np.nonzero(walk.x != D)[0]:
            orc.step_flip(U, walk, int(k))
        jump = st.copy()
        r = orc.batch(U, jump, D, 1, T=3, B=1, tabu=8, seed=1, slot=0, gen=0, trace_cap=4 * n + 64, jump=True)
        # after the batch the state moved on (Greedy + one main round); replay
        # the same batch from the walked state with Straight having nothing to do
        ref = walk.copy()
        ref.ring[:] = st.ring   # the jump makes no flips, so it pushes nothing on the tabu ring (R-30)
        r2 = orc.batch(U, ref, D, 1, T=3, B=1, tabu=8, seed=1, slot=0, gen=0, trace_cap=4 * n + 64)
        assert np.array_equal(walk.x, D)
        assert r.flips == r2.flips and r.ebest == r2.ebest and np.array_equal(r.best, r2.best)
        assert np.array_equal(r.trace_bit, r2.trace_bit) and np.array_equal(r.trace_E, r2.trace_E)
        assert jump.E == ref.E and np.array_equal(jump.x, ref.x) and np.array_equal(jump.delta, ref.delta)
        # and no Straight flips were made
        assert not (r.trace_phase == 0).any()


def test_jump_runs_reach_optimum(orc):
    rng = np.random.default_rng(12)
    for trial in range(6):
        n = 12
        U = rand_upper(rng, n)
        X = np.array(list(itertools.product([0, 1], repeat=n)), np.int64)
        opt = int(np.einsum("bi,ij,bj->b", X, U.astype(np.int64), X).min())
        cfg = orc.Config(s_milli=200, b_milli=2000, pools=1, slots=4, cap=10, jump=True)
        E, Xb, _ = orc.System(U, cfg).run(seed=trial, flip_budget=10**6, target=opt)
        assert E == opt == orc.energy(U, Xb)


def test_jump_world_checked(orc):
    """Whole generations with jump-start batches in checked mode (Delta
    recomputed from scratch after every flip)."""
    rng = np.random.default_rng(2)
    U = rand_upper(rng, 30)
    cfg = orc.Config(s_milli=200, b_milli=1000, pools=2, slots=3, cap=8, jump=True)
    sysm = orc.System(U, cfg, checked=True)
    sysm.reset(3)
    for _ in range(4):
        sysm.generation()
    w = sysm.ranks[0]
    for s in range(6):
        st = w.slot(s)
        assert st.E == orc.energy(U, st.x)
