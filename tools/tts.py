"""Time-to-target on workloads with a known optimum (TSP32 cycle metric:
E* = 2 m scale - m p, R-22; K16: brute force) and best-after-budget on the
others.  Runs R seeds, reports success rate and mean TTS over successes
(the paper's protocol)."""
import argparse
import itertools
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_2207_03069_b200 import Solver, workloads as wl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="TSP32")
    ap.add_argument("--runs", type=int, default=5)
    ap.add_argument("--limit", type=float, default=30.0, help="seconds per run")
    ap.add_argument("--pools", type=int, default=1)
    ap.add_argument("--slots", type=int, default=0)
    ap.add_argument("--target", type=int, default=None, help="override the workload's target energy")
    ap.add_argument("--mode", default="dabs", choices=["dabs", "abs", "restart"],
                    help="abs: CyclicMin + mutation after crossover only (R-27); restart: DABS with "
                         "restart-on-merge after --restart-gens stalled generations (R-28)")
    ap.add_argument("--restart-gens", type=int, default=20)
    ap.add_argument("--schedule", default="generation", choices=["generation", "async"],
                    help="async: dabs_run_async, one wave of persistent searches (R-29)")
    args = ap.parse_args()
    U, meta = wl.make(args.workload, seed=1)
    target = meta.get("target")
    if args.workload == "K16":
        X = np.array(list(itertools.product([0, 1], repeat=16)), np.int64)
        target = int(np.einsum("bi,ij,bj->b", X, U.astype(np.int64), X).min())
    if args.target is not None:
        target = args.target
    mode = dict(abs=dict(genop_mask=1 << 8, algo_mask=1 << 1), restart=dict(restart_gens=args.restart_gens),
                dabs={})[args.mode]
    asy = args.schedule == "async"
    s = Solver(U, s_milli=meta["s_milli"], b_milli=meta["b_milli"], pools=args.pools, slots=args.slots,
               target=target, time_limit_ns=int(args.limit * 1e9), one_wave=asy, **mode)
    res = []
    for r in range(args.runs):
        t0 = time.perf_counter()
        E, x = (s.run_async if asy else s.run)(seed=1000 + r, flip_budget=1 << 62)
        dt = time.perf_counter() - t0
        st = s.stats()
        ok = target is not None and E <= target
        res.append(dict(seed=1000 + r, best=E, ok=bool(ok), wall_s=dt, tts_s=st.time_to_best_ns / 1e9,
                        gens=int(st.generations), flips=int(st.total_flips), restarts=int(st.restarts)))
        print(json.dumps(res[-1]), flush=True)
    succ = [x for x in res if x["ok"]]
    print(json.dumps({"workload": args.workload, "mode": args.mode, "schedule": args.schedule, "target": target,
                      "runs": args.runs,
                      "success_rate": len(succ) / args.runs,
                      "mean_tts_s": float(np.mean([x["tts_s"] for x in succ])) if succ else None,
                      "slots": s.slots, "pools": s.pools,
                      "best": min(x["best"] for x in res)}))


if __name__ == "__main__":
    main()
