"""ctypes wrapper around oracle/libdabs_oracle.so -- the CPU oracle.

TEST INFRASTRUCTURE ONLY.  Only tests/, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this
module.  The product package (``paper_2207_03069_b200``) never imports it and
shares no code with it.

The C file ``oracle/dabs_oracle.c`` holds all of the method's arithmetic; this
wrapper only marshals numpy arrays and drives the generation loop, including
the exchange between simulated ranks.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "dabs_oracle.c")
LIB = os.path.join(HERE, "libdabs_oracle.so")

TABU_MAX = 32
N_ALG, N_GEN = 5, 9   # 8 paper genops + ABS's mutation-after-crossover (R-27)
ALG_NAMES = ["MaxMin", "CyclicMin", "RandomMin", "PositiveMin", "TwoNeighbor"]
GEN_NAMES = ["Mutation", "Crossover", "Xrossover", "Zero", "One", "IntervalZero", "Best", "Random", "MutCross"]
E_INF = np.iinfo(np.int64).max


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2; no tuning flags)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", SRC, "-o", LIB])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        # DABS_ORACLE_LIB: a prebuilt oracle variant (tools/mutation_probe.py
        # loads deliberately broken builds to check that the pins reject them)
        path = os.environ.get("DABS_ORACLE_LIB") or build()
        L = C.CDLL(path)
        P = C.c_void_p
        i32, i64, u32, u64 = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64
        L.orc_philox.argtypes = [P, P, P]
        L.orc_energy.argtypes = [P, C.c_int, P]
        L.orc_energy.restype = i64
        L.orc_delta_closed.argtypes = [P, C.c_int, P, P]
        L.orc_flip_factor.argtypes = [C.c_int, C.c_int]
        L.orc_flip_factor.restype = C.c_int
        L.orc_batch.argtypes = [P, C.c_int, C.c_int, C.c_int, C.c_int,
                                P, P, P, P,
                                P, C.c_int, u64, u32, u32,
                                P, P, P,
                                P, P, P, i64, C.c_int]
        L.orc_batch.restype = C.c_int
        L.orc_batch_limited.argtypes = L.orc_batch.argtypes + [i64]
        L.orc_batch_limited.restype = C.c_int
        L.orc_batch_ex.argtypes = L.orc_batch.argtypes + [i64, C.c_int]
        L.orc_batch_ex.restype = C.c_int
        L.orc_step_flip.argtypes = [P, C.c_int, P, P, P, P, C.c_int]
        L.orc_world_new.argtypes = [P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                    u32, u32, u32, C.c_int, C.c_int, C.c_int, C.c_int]
        L.orc_world_new.restype = P
        L.orc_world_free.argtypes = [P]
        L.orc_world_set_checked.argtypes = [P, C.c_int]
        L.orc_world_set_restart.argtypes = [P, u32]
        L.orc_world_set_jump.argtypes = [P, C.c_int]
        L.orc_world_restarts.argtypes = [P]
        L.orc_world_restarts.restype = u32
        L.orc_world_reset.argtypes = [P, u64]
        L.orc_world_generation_local.argtypes = [P]
        L.orc_world_generation_local.restype = C.c_int
        L.orc_world_payload_bytes.argtypes = [P]
        L.orc_world_payload_bytes.restype = C.c_long
        L.orc_world_export.argtypes = [P, P]
        L.orc_world_import.argtypes = [P, P]
        for f in ("orc_world_T", "orc_world_B"):
            getattr(L, f).argtypes = [P]
            getattr(L, f).restype = C.c_int
        L.orc_world_gen.argtypes = [P]
        L.orc_world_gen.restype = u32
        L.orc_world_total_flips.argtypes = [P]
        L.orc_world_total_flips.restype = u64
        L.orc_world_gen_flips.argtypes = [P]
        L.orc_world_gen_flips.restype = u64
        L.orc_world_get_pool.argtypes = [P, C.c_int, P, P, P, P, P]
        L.orc_world_get_slot.argtypes = [P, C.c_int, P, P, P, P]
        L.orc_world_get_packet.argtypes = [P, C.c_int, P, P, P, P, P, P]
        L.orc_world_get_stats.argtypes = [P, P, P]
        L.orc_world_get_best.argtypes = [P, P, P, P]
        L.orc_world_async_replay.argtypes = [P, P, C.c_int64]
        L.orc_world_async_replay.restype = C.c_int
        L.orc_world_async_begin.argtypes = [P]
        L.orc_world_async_begin.restype = C.c_int
        L.orc_world_async_event.argtypes = [P, u32]
        L.orc_world_async_event.restype = C.c_int
        L.orc_world_async_end.argtypes = [P]
        L.orc_world_async_end.restype = C.c_int
        L.orc_lowbias32.argtypes = [u32]
        L.orc_lowbias32.restype = u32
        L.orc_rank_pick.argtypes = [u32, u32]
        L.orc_rank_pick.restype = u32
        L.orc_build_target.argtypes = [C.c_int, P, P, P, C.c_int, u64, u32, u32, u32, u32, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


# --------------------------------------------------------------------------
# primitives
# --------------------------------------------------------------------------
def philox(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, np.uint32)
    lib().orc_philox(_p(c), _p(k), _p(out))
    return out


def energy(U: np.ndarray, x: np.ndarray) -> int:
    U = np.ascontiguousarray(U, dtype=np.int16)
    x = np.ascontiguousarray(x, dtype=np.uint8)
    return int(lib().orc_energy(_p(U), U.shape[0], _p(x)))


def delta_closed(U: np.ndarray, x: np.ndarray) -> np.ndarray:
    U = np.ascontiguousarray(U, dtype=np.int16)
    x = np.ascontiguousarray(x, dtype=np.uint8)
    d = np.zeros(U.shape[0], np.int32)
    lib().orc_delta_closed(_p(U), U.shape[0], _p(x), _p(d))
    return d


def lowbias32(x: int) -> int:
    return int(lib().orc_lowbias32(x))


def rank_pick(u: int, m: int) -> int:
    """0-based rank-biased row floor(u^3 m / 2^96) (R-17)."""
    return int(lib().orc_rank_pick(u, m))


def build_target(genop: int, A, B, best0, *, seed: int, gslot: int, gen: int, L: int = 0,
                 start: int = 0) -> np.ndarray:
    """Apply one genetic operation -- exposed for the pin tests."""
    A = np.ascontiguousarray(A, dtype=np.uint8)
    B = np.ascontiguousarray(B, dtype=np.uint8)
    b0 = np.ascontiguousarray(best0, dtype=np.uint8)
    D = np.zeros(A.size, np.uint8)
    lib().orc_build_target(genop, _p(A), _p(B), _p(b0), A.size, seed, gslot, gen, L, start, _p(D))
    return D


def flip_factor(milli: int, n: int) -> int:
    return int(lib().orc_flip_factor(milli, n))


@dataclass
class SlotState:
    """The persistent state of one search: X, Delta, E, tabu ring."""
    x: np.ndarray
    delta: np.ndarray
    E: int
    ring: np.ndarray

    @staticmethod
    def initial(U: np.ndarray) -> "SlotState":
        n = U.shape[0]
        return SlotState(np.zeros(n, np.uint8), np.ascontiguousarray(np.diag(U).astype(np.int32)),
                         0, np.full(TABU_MAX, -1, np.int32))

    def copy(self) -> "SlotState":
        return SlotState(self.x.copy(), self.delta.copy(), int(self.E), self.ring.copy())


@dataclass
class BatchResult:
    best: np.ndarray
    ebest: int
    flips: int
    trace_bit: np.ndarray | None
    trace_E: np.ndarray | None
    trace_phase: np.ndarray | None


def batch(U: np.ndarray, state: SlotState, D: np.ndarray, algo: int, *, T: int, B: int,
          tabu: int = 8, seed: int = 0, slot: int = 0, gen: int = 0,
          trace_cap: int = 0, checked: bool = False, jump: bool = False) -> BatchResult:
    """Run one batch search in place on ``state``; jump = the
    jump-start variant (R-30)."""
    U = np.ascontiguousarray(U, dtype=np.int16)
    n = U.shape[0]
    D = np.ascontiguousarray(D, dtype=np.uint8)
    best = np.zeros(n, np.uint8)
    E = np.array([state.E], np.int64)
    ebest = np.zeros(1, np.int64)
    flips = np.zeros(1, np.int64)
    if trace_cap:
        tb = np.zeros(trace_cap, np.int32)
        te = np.zeros(trace_cap, np.int64)
        tp = np.zeros(trace_cap, np.int8)
        tptr = (_p(tb), _p(te), _p(tp))
    else:
        tb = te = tp = None
        tptr = (None, None, None)
    err = lib().orc_batch_ex(_p(U), n, T, B, tabu, _p(state.x), _p(state.delta), _p(E), _p(state.ring),
                             _p(D), algo, seed, slot, gen, _p(best), _p(ebest), _p(flips),
                             *tptr, trace_cap, int(checked), 0, int(jump))
    if err:
        raise RuntimeError(f"oracle batch error {err}")
    state.E = int(E[0])
    f = int(flips[0])
    if tb is not None:
        m = min(f, trace_cap)
        tb, te, tp = tb[:m], te[:m], tp[:m]
    return BatchResult(best, int(ebest[0]), f, tb, te, tp)


def batch_sample(U: np.ndarray, state: SlotState, D: np.ndarray, algo: int, *, T: int, B: int, tabu: int,
                 seed: int, slot: int, gen: int, flip_limit: int) -> int:
    """Run a batch but stop after ``flip_limit`` flips; returns the flips done.
    Timing aid only (bench cpu_baseline); releases the GIL inside C."""
    U = np.ascontiguousarray(U, dtype=np.int16)
    n = U.shape[0]
    D = np.ascontiguousarray(D, dtype=np.uint8)
    best = np.zeros(n, np.uint8)
    E = np.array([state.E], np.int64)
    ebest = np.zeros(1, np.int64)
    flips = np.zeros(1, np.int64)
    err = lib().orc_batch_limited(_p(U), n, T, B, tabu, _p(state.x), _p(state.delta), _p(E), _p(state.ring),
                                  _p(D), algo, seed, slot, gen, _p(best), _p(ebest), _p(flips),
                                  None, None, None, 0, 0, flip_limit)
    if err not in (0, 4):
        raise RuntimeError(f"oracle batch error {err}")
    state.E = int(E[0])
    return int(flips[0])


def step_flip(U: np.ndarray, state: SlotState, i: int) -> None:
    U = np.ascontiguousarray(U, dtype=np.int16)
    E = np.array([state.E], np.int64)
    lib().orc_step_flip(_p(U), U.shape[0], _p(state.x), _p(state.delta), _p(E), _p(state.ring), i)
    state.E = int(E[0])


# --------------------------------------------------------------------------
# world: pools + slots of one rank; System: G simulated ranks in one process
# --------------------------------------------------------------------------
@dataclass
class Config:
    s_milli: int = 100
    b_milli: int = 1000
    tabu: int = 8
    cap: int = 100
    eps_ppm: int = 50000
    genop_mask: int = 0xFF
    algo_mask: int = 0x1F
    pools: int = 1          # pools per rank
    slots: int = 1          # slots per pool
    restart_gens: int = 0   # restart-on-merge after this many stalled generations (R-28); 0 = off
    jump: bool = False      # jump-start batches (R-30): X <- D instead of Straight


class World:
    """The pools and slots one rank (GPU) owns."""

    def __init__(self, U: np.ndarray, cfg: Config, rank: int = 0, world: int = 1, checked: bool = False):
        self.U = np.ascontiguousarray(U, dtype=np.int16)
        self.n = self.U.shape[0]
        self.cfg = cfg
        self.rank, self.world = rank, world
        L = lib()
        self.h = L.orc_world_new(_p(self.U), self.n, cfg.s_milli, cfg.b_milli, cfg.tabu, cfg.cap,
                                 cfg.eps_ppm, cfg.genop_mask, cfg.algo_mask,
                                 cfg.pools, cfg.slots, rank, world)
        L.orc_world_set_checked(self.h, int(checked))
        L.orc_world_set_restart(self.h, int(cfg.restart_gens))
        L.orc_world_set_jump(self.h, int(cfg.jump))
        self.payload_bytes = int(L.orc_world_payload_bytes(self.h))

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_world_free(self.h)
            self.h = None

    @property
    def T(self):
        return int(lib().orc_world_T(self.h))

    @property
    def B(self):
        return int(lib().orc_world_B(self.h))

    @property
    def gen(self):
        return int(lib().orc_world_gen(self.h))

    @property
    def total_flips(self):
        return int(lib().orc_world_total_flips(self.h))

    @property
    def restarts(self):
        return int(lib().orc_world_restarts(self.h))

    @property
    def gen_flips(self):
        return int(lib().orc_world_gen_flips(self.h))

    def reset(self, seed: int):
        lib().orc_world_reset(self.h, seed)

    def generation_local(self):
        err = lib().orc_world_generation_local(self.h)
        if err:
            raise RuntimeError(f"oracle generation error {err}")

    def async_replay(self, log) -> None:
        """Replay an asynchronous-schedule event log (R-29) from a
        fresh reset: entries s | seeded<<31 in merge order."""
        lg = np.ascontiguousarray(np.asarray(log, dtype=np.uint32))
        err = lib().orc_world_async_replay(self.h, _p(lg), int(lg.size))
        if err:
            raise RuntimeError(f"oracle async replay error {err}")

    def async_begin(self) -> None:
        err = lib().orc_world_async_begin(self.h)
        if err:
            raise RuntimeError(f"oracle async begin error {err}")

    def async_event(self, entry: int) -> int:
        """One log entry (slot | seeded<<31 | xread<<30); returns 1 when the
        slot's new packet waits for its XREAD event (R-29)."""
        r = lib().orc_world_async_event(self.h, int(entry))
        if r < 0:
            raise RuntimeError(f"oracle async event error {-r}")
        return r

    def async_end(self) -> None:
        err = lib().orc_world_async_end(self.h)
        if err:
            raise RuntimeError(f"oracle async end error {err}")

    def export(self) -> np.ndarray:
        buf = np.zeros(self.payload_bytes, np.uint8)
        lib().orc_world_export(self.h, _p(buf))
        return buf

    def import_(self, gathered: np.ndarray):
        g = np.ascontiguousarray(gathered, dtype=np.uint8)
        assert g.size == self.payload_bytes * self.world
        lib().orc_world_import(self.h, _p(g))

    def pool(self, p: int):
        """p in [0, pools) -> local pool; p == pools -> successor snapshot."""
        cap, n = self.cfg.cap, self.n
        X = np.zeros((cap, n), np.uint8)
        E = np.zeros(cap, np.int64)
        seq = np.zeros(cap, np.uint64)
        a = np.zeros(cap, np.uint8)
        g = np.zeros(cap, np.uint8)
        lib().orc_world_get_pool(self.h, p, _p(X), _p(E), _p(seq), _p(a), _p(g))
        return dict(X=X, E=E, seq=seq, algo=a, genop=g)

    def slot(self, s: int) -> SlotState:
        n = self.n
        x = np.zeros(n, np.uint8)
        d = np.zeros(n, np.int32)
        E = np.zeros(1, np.int64)
        r = np.zeros(TABU_MAX, np.int32)
        lib().orc_world_get_slot(self.h, s, _p(x), _p(d), _p(E), _p(r))
        return SlotState(x, d, int(E[0]), r)

    def packet(self, s: int):
        n = self.n
        D = np.zeros(n, np.uint8)
        best = np.zeros(n, np.uint8)
        a = np.zeros(1, np.int32)
        g = np.zeros(1, np.int32)
        eb = np.zeros(1, np.int64)
        fl = np.zeros(1, np.int64)
        lib().orc_world_get_packet(self.h, s, _p(D), _p(a), _p(g), _p(best), _p(eb), _p(fl))
        return dict(D=D, algo=int(a[0]), genop=int(g[0]), best=best, ebest=int(eb[0]), flips=int(fl[0]))

    def stats(self):
        P = self.cfg.pools
        d = np.zeros((P, N_ALG, N_GEN), np.uint64)
        i = np.zeros((P, N_ALG, N_GEN), np.uint64)
        lib().orc_world_get_stats(self.h, _p(d), _p(i))
        return d, i

    def best(self):
        E = np.zeros(1, np.int64)
        X = np.zeros(self.n, np.uint8)
        rec = np.zeros(4, np.int32)
        lib().orc_world_get_best(self.h, _p(E), _p(X), _p(rec))
        return int(E[0]), X, dict(algo=int(rec[0]), genop=int(rec[1]), gen=int(rec[2]), slot=int(rec[3]))


class System:
    """G simulated ranks in one process; the exchange is a plain concatenation
    of every rank's payload (what an all-gather delivers)."""

    def __init__(self, U: np.ndarray, cfg: Config, world: int = 1, checked: bool = False):
        self.ranks = [World(U, cfg, r, world, checked) for r in range(world)]

    def reset(self, seed: int):
        for w in self.ranks:
            w.reset(seed)

    def generation(self):
        for w in self.ranks:
            w.generation_local()
        gathered = np.concatenate([w.export() for w in self.ranks])
        for w in self.ranks:
            w.import_(gathered)

    def run(self, seed: int, flip_budget: int, target: int | None = None, max_gens: int | None = None):
        """dabs_run semantics: whole generations until total flips >= budget,
        or best <= target."""
        self.reset(seed)
        w0 = self.ranks[0]
        while True:
            self.generation()
            E, X, rec = w0.best()
            if w0.total_flips >= flip_budget:
                break
            if target is not None and E <= target:
                break
            if max_gens is not None and w0.gen >= max_gens:
                break
        return w0.best()
