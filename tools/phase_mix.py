"""Per-phase flip mix of one traced slot over a few generations:
python tools/phase_mix.py R32K [gens] [slot]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_2207_03069_b200 import Solver, workloads as wl  # noqa: E402

U, meta = wl.make(sys.argv[1], seed=1)
gens = int(sys.argv[2]) if len(sys.argv) > 2 else 4
slots = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "0,1,2,3,4,5,6,7,8,9").split(",")]
s = Solver(U, s_milli=meta["s_milli"], b_milli=meta["b_milli"], pools=meta.get("pools", 1))
tot = {}
for slot in slots:
    s.reset(1)
    cap = 4 * s.B + 10 * U.shape[0]
    for g in range(gens):
        if g == gens - 1:
            s.trace_enable(slot, cap)
        s.generation()
    tr = s.trace_read(cap)
    ph = np.asarray(tr[2])
    algo = int(s.read_packet(slot)["algo"]) if "algo" in s.read_packet(slot) else -1
    names = {0: "straight", 1: "greedy"}
    cnt = {names.get(int(p), "main"): int((ph == p).sum()) if p < 2 else 0 for p in (0, 1)}
    cnt["main"] = int((ph >= 2).sum())
    print("slot", slot, "algo", algo, "flips", len(ph), cnt, flush=True)
    for k, v in cnt.items():
        tot[k] = tot.get(k, 0) + v
print("total", tot, {k: round(v / sum(tot.values()), 3) for k, v in tot.items()})
