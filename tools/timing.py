"""Per-flip critical-path breakdown of the batch kernel from a -DDABS_TIMING build:
DABS_LIB=ab/libdabs_timing.so python tools/timing.py R32K [gens]
Buckets (thread 0, SM cycles per flip): sel = Step 1+2 (scan, reductions,
selection), wait0 = row issue -> first piece, xfer = rest of the row + update,
head = loop head / bookkeeping."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_2207_03069_b200 import Solver, workloads as wl  # noqa: E402
from paper_2207_03069_b200 import dabs as D  # noqa: E402

NAMES = ["MaxMin", "CyclicMin", "RandomMin", "PositiveMin", "TwoNeighbor", "Straight/Greedy"]


def read(L):
    out = (C.c_ulonglong * 56)()
    L.dabs_timing_read(out)
    a = np.array(out, dtype=np.float64)
    return a[:30].reshape(6, 5), a[30:]


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "R32K"
    gens = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    U, meta = wl.make(cfg, seed=1)
    L = D.load()
    masks = [int(x, 0) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 2, 4, 8, 16, 31]
    for mask in masks:
        s = Solver(U, s_milli=meta["s_milli"], b_milli=meta["b_milli"], pools=1, algo_mask=mask)
        s.reset(1)
        s.generation()
        read(L)
        fl, ms = 0, 0.0
        for _ in range(gens):
            f0 = s.stats().local_flips
            s.generation()
            st = s.stats()
            fl += st.local_flips - f0
            ms += st.batch_ms_last
        t, t2 = read(L)
        print(f"{cfg} algo_mask={mask:#x}: {fl / ms * 1e3 / 1e6:.1f}M flips/s", flush=True)
        for b in range(6):
            if t[b, 4] > 0:
                c = t[b, :4] / t[b, 4]
                print(f"   {NAMES[b]:16s} flips {int(t[b, 4]):9d}  sel {c[0]:7.0f}  wait0 {c[1]:7.0f}  "
                      f"xfer+upd {c[2]:7.0f}  head {c[3]:6.0f}  total {c.sum():7.0f} cyc")
        nsel = t[0, 4] + t[3, 4]
        if nsel > 0:
            print("   MaxMin/PosMin sub-steps (cyc/flip): pass1 %.0f reduce1 %.0f thr %.0f count %.0f reduce2 %.0f "
                  "chunk %.0f wsel %.0f pickwait %.0f" % tuple(t2[:8] / nsel))
        nfl = t[:, 4].sum()
        t3 = t2[10:26]
        if t3.sum() > 0 and nfl > 0:
            print("   TMEM tier update per flip (cyc): " + "  ".join(
                "piece%d ld %.0f wait %.0f upd %.0f" % (q, t3[3 * q] / nfl, t3[3 * q + 1] / nfl, t3[3 * q + 2] / nfl)
                for q in range(4)) + "  st-drain %.0f" % (t3[12] / nfl))
        s.close()


if __name__ == "__main__":
    main()
