"""Diagnose async-schedule parity: grid of (n, P, S, budget) -> pass/fail and
the first differing pool entry (its seq names the merge event)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from oracle import oracle as orc
from paper_2207_03069_b200 import dabs as lib


def one(n, P, S, mult, seed=4242, mask=0xFF):
    rng = np.random.default_rng(n + 1)
    U = np.triu(rng.integers(-200, 201, size=(n, n))).astype(np.int16)
    s = lib.Solver(U, s_milli=100, b_milli=1000, pools=P, slots=S, cap=16, genop_mask=mask)
    s.run_async(seed, mult * P * S * n)
    log = s.async_log()
    w = orc.World(U, orc.Config(s_milli=100, b_milli=1000, pools=P, slots=S, cap=16, genop_mask=mask))
    w.reset(seed)
    w.async_replay(log)
    bad = []
    for p in range(P):
        g, r = s.read_pool(p), w.pool(p)
        for i in range(16):
            if g["E"][i] != r["E"][i] or g["seq"][i] != r["seq"][i]:
                bad.append((p, i, int(g["E"][i]), int(g["seq"][i]) >> 32, int(g["seq"][i]) & 0xffffffff,
                            int(r["E"][i]), int(r["seq"][i]) >> 32, int(r["seq"][i]) & 0xffffffff))
                break
    slots_bad = [q for q in range(P * S) if s.read_slot(q)["E"] != w.slot(q).E]
    print(f"n={n} P={P} S={S} mult={mult} mask={mask:#x} events={len(log)} pools_bad={bad} slots_bad={slots_bad}",
          flush=True)
    if bad or slots_bad:
        print("  log:", [(int(v) & 0x3fffffff, (int(v) >> 30)) for v in log[:60]])


for args in [(300, 1, 5, 6), (300, 3, 1, 6), (300, 2, 1, 6), (300, 3, 5, 6), (300, 3, 5, 1), (300, 3, 5, 6, 4242, 0xFB),
             (300, 1, 15, 6), (40, 3, 2, 6)]:
    one(*args)
