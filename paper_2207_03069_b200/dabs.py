"""Thin ctypes binding of the C ABI in include/dabs.h (argument marshalling only).

Every step of the DABS path runs in the CUDA kernels of libdabs.so; this module
only converts numpy arrays and torch objects to plain pointers.  There is no
CPU fallback: if libdabs.so is missing or no sm_100a device is present, the
calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DABS_LIB", os.path.join(HERE, "libdabs.so"))   # DABS_LIB: A/B builds

DABS_OK = 0
STATUS = {0: "OK", 1: "E_ARG", 2: "E_TRIANGLE", 3: "E_RANGE", 4: "E_NOMEM", 5: "E_CUDA", 6: "E_COMM",
          7: "E_STATE"}
TABU_RING = 32
INT64_MIN = -(1 << 63)

EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)
ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)


class dabs_config(C.Structure):
    _fields_ = [
        ("struct_size", C.c_uint32), ("s_milli", C.c_uint32), ("b_milli", C.c_uint32),
        ("tabu_period", C.c_uint32), ("pool_capacity", C.c_uint32), ("eps_ppm", C.c_uint32),
        ("genop_mask", C.c_uint32), ("algo_mask", C.c_uint32), ("pools_per_gpu", C.c_uint32),
        ("slots_per_pool", C.c_uint32), ("target_energy", C.c_int64), ("time_limit_ns", C.c_uint64),
        ("rank", C.c_int32), ("world", C.c_int32), ("device", C.c_int32),
        ("cuda_stream", C.c_void_p), ("exchange", EXCHANGE_FN), ("alloc", ALLOC_FN), ("free", FREE_FN),
        ("user", C.c_void_p), ("restart_gens", C.c_uint32), ("flags", C.c_uint32),
    ]


class dabs_stats(C.Structure):
    _fields_ = [
        ("total_flips", C.c_uint64), ("local_flips", C.c_uint64), ("generations", C.c_uint64),
        ("wall_ns", C.c_uint64), ("time_to_best_ns", C.c_uint64),
        ("batch_ms_last", C.c_float), ("ga_ms_last", C.c_float), ("merge_ms_last", C.c_float),
        ("best_energy", C.c_int64),
        ("best_algo", C.c_int32), ("best_genop", C.c_int32), ("best_generation", C.c_int32),
        ("best_slot", C.c_int32),
        ("dispatch", (C.c_uint64 * 9) * 5), ("inserted", (C.c_uint64 * 9) * 5), ("restarts", C.c_uint64),
        ("n", C.c_int32), ("n_pad", C.c_int32), ("threads_per_search", C.c_int32), ("slots", C.c_int32),
        ("pools", C.c_int32), ("T", C.c_int32), ("B", C.c_int32), ("cap", C.c_int32),
        ("kernel_launches", C.c_uint64),
    ]


# every symbol include/dabs.h declares (checked by tests/test_abi.py)
EXPORTS = ["dabs_config_default", "dabs_create", "dabs_create_csr", "dabs_reset", "dabs_generation", "dabs_run",
           "dabs_best", "dabs_energy", "dabs_get_stats", "dabs_debug_batch", "dabs_read_slot", "dabs_read_pool",
           "dabs_read_packet", "dabs_read_stats_pool", "dabs_trace_enable", "dabs_trace_read",
           "dabs_run_async", "dabs_async_log", "dabs_async_lock_ns", "dabs_jump_ms", "dabs_probe_row_stream",
           "dabs_last_error", "dabs_destroy"]

_lib = None


class DabsError(RuntimeError):
    pass


def load(path: str = LIB_PATH):
    """Load libdabs.so; raises (never falls back) when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise DabsError(f"{path} is missing: run `python -m paper_2207_03069_b200.build` (nvcc, sm_100a)")
    L = C.CDLL(path)
    P, u32, i32, i64, u64 = C.c_void_p, C.c_uint32, C.c_int32, C.c_int64, C.c_uint64
    st = C.c_int
    L.dabs_config_default.argtypes = [C.POINTER(dabs_config)]
    L.dabs_config_default.restype = None
    L.dabs_create.argtypes = [P, i32, C.POINTER(dabs_config), C.POINTER(C.c_void_p)]
    L.dabs_create.restype = st
    L.dabs_create_csr.argtypes = [i32, P, P, P, P, C.POINTER(dabs_config), C.POINTER(C.c_void_p)]
    L.dabs_create_csr.restype = st
    L.dabs_reset.argtypes = [P, u64]
    L.dabs_reset.restype = st
    L.dabs_generation.argtypes = [P]
    L.dabs_generation.restype = st
    L.dabs_run.argtypes = [P, u64, u64, P, P]
    L.dabs_run.restype = st
    L.dabs_run_async.argtypes = [P, u64, u64, P, P]
    L.dabs_run_async.restype = st
    L.dabs_async_log.argtypes = [P, P, i64, P]
    L.dabs_async_log.restype = st
    L.dabs_jump_ms.argtypes = [P, P]
    L.dabs_jump_ms.restype = st
    L.dabs_async_lock_ns.argtypes = [P, P, P]
    L.dabs_async_lock_ns.restype = st
    L.dabs_best.argtypes = [P, P, P]
    L.dabs_best.restype = st
    L.dabs_energy.argtypes = [P, P, P]
    L.dabs_energy.restype = st
    L.dabs_get_stats.argtypes = [P, C.POINTER(dabs_stats)]
    L.dabs_get_stats.restype = st
    L.dabs_debug_batch.argtypes = [P, u32, P, P, P, P, P, i32, u64, u32, P, P, P, P, P, P, i64]
    L.dabs_debug_batch.restype = st
    L.dabs_read_slot.argtypes = [P, u32, P, P, P, P]
    L.dabs_read_slot.restype = st
    L.dabs_read_pool.argtypes = [P, u32, P, P, P, P, P]
    L.dabs_read_pool.restype = st
    L.dabs_read_packet.argtypes = [P, u32, P, P, P, P, P, P]
    L.dabs_read_packet.restype = st
    L.dabs_read_stats_pool.argtypes = [P, u32, P, P]
    L.dabs_read_stats_pool.restype = st
    L.dabs_trace_enable.argtypes = [P, i32, i64]
    L.dabs_trace_enable.restype = st
    L.dabs_trace_read.argtypes = [P, P, P, P, P]
    L.dabs_trace_read.restype = st
    L.dabs_probe_row_stream.argtypes = [i32, i64, i32, i32, i32, i32, P]
    L.dabs_probe_row_stream.restype = st
    L.dabs_last_error.argtypes = []
    L.dabs_last_error.restype = C.c_char_p
    L.dabs_destroy.argtypes = [P]
    L.dabs_destroy.restype = None
    _lib = L
    return L


def _check(status: int):
    if status != DABS_OK:
        msg = load().dabs_last_error().decode(errors="replace")
        raise DabsError(f"dabs {STATUS.get(status, status)}: {msg}")


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


def config_default() -> dabs_config:
    cfg = dabs_config()
    load().dabs_config_default(C.byref(cfg))
    return cfg


class Solver:
    """One rank's DABS context over an upper-triangular int16 W (Eq.(2))."""

    def __init__(self, W: np.ndarray | None, *, csr=None, s_milli: int = 100, b_milli: int = 1000,
                 tabu: int = 8, cap: int = 100, eps_ppm: int = 50000, genop_mask: int = 0xFF, algo_mask: int = 0x1F,
                 restart_gens: int = 0,
                 pools: int = 1, slots: int = 0, target: int | None = None, time_limit_ns: int = 0,
                 rank: int = 0, world: int = 1, device: int = -1, stream=None, exchange=None,
                 one_wave: bool = False, jump: bool = False):
        L = load()
        if csr is None:
            W = np.ascontiguousarray(W, dtype=np.int16)
            if W.ndim != 2 or W.shape[0] != W.shape[1]:
                raise ValueError("W must be square")
            self.n = W.shape[0]
        else:
            rp, col, val, diag = csr
            rp = np.ascontiguousarray(rp, dtype=np.int32)
            col = np.ascontiguousarray(col, dtype=np.int32)
            val = np.ascontiguousarray(val, dtype=np.int16)
            diag = np.ascontiguousarray(diag, dtype=np.int16)
            self.n = diag.size
        cfg = config_default()
        cfg.s_milli, cfg.b_milli, cfg.tabu_period, cfg.pool_capacity = s_milli, b_milli, tabu, cap
        cfg.eps_ppm, cfg.genop_mask, cfg.algo_mask = eps_ppm, genop_mask, algo_mask
        cfg.pools_per_gpu, cfg.slots_per_pool = pools, slots
        cfg.restart_gens = restart_gens
        cfg.flags = (1 if one_wave else 0) | (2 if jump else 0)
        cfg.target_energy = INT64_MIN if target is None else int(target)
        cfg.time_limit_ns = time_limit_ns
        cfg.rank, cfg.world, cfg.device = rank, world, device
        cfg.cuda_stream = stream
        self._exchange_cb = None
        if exchange is not None:
            self._exchange_cb = EXCHANGE_FN(exchange)
            cfg.exchange = self._exchange_cb
        self.cfg = cfg
        h = C.c_void_p()
        if csr is None:
            _check(L.dabs_create(_p(W), self.n, C.byref(cfg), C.byref(h)))
        else:
            _check(L.dabs_create_csr(self.n, _p(rp), _p(col) if col.size else None,
                                     _p(val) if val.size else None, _p(diag), C.byref(cfg), C.byref(h)))
        self.h = h
        st = self.stats()
        self.slots, self.pools, self.cap = st.slots, st.pools, st.cap
        self.T, self.B, self.n_pad, self.threads = st.T, st.B, st.n_pad, st.threads_per_search

    @staticmethod
    def to_csr(U: np.ndarray):
        """Upper-triangular dense U -> (row_ptr, col, val, diag) for dabs_create_csr."""
        U = np.asarray(U)
        n = U.shape[0]
        iu = np.triu(U, 1)
        rows, cols = np.nonzero(iu)
        rp = np.zeros(n + 1, np.int32)
        np.add.at(rp, rows + 1, 1)
        return np.cumsum(rp).astype(np.int32), cols.astype(np.int32), iu[rows, cols].astype(np.int16), \
            np.diag(U).astype(np.int16)

    def close(self):
        if getattr(self, "h", None):
            load().dabs_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- run control
    def reset(self, seed: int):
        _check(load().dabs_reset(self.h, seed))

    def generation(self):
        _check(load().dabs_generation(self.h))

    def run(self, seed: int, flip_budget: int):
        x = np.zeros(self.n, np.uint8)
        e = np.zeros(1, np.int64)
        _check(load().dabs_run(self.h, seed, flip_budget, _p(x), _p(e)))
        return int(e[0]), x

    def run_async(self, seed: int, flip_budget: int):
        """Asynchronous schedule (dabs_run_async): one persistent kernel."""
        x = np.zeros(self.n, np.uint8)
        e = np.zeros(1, np.int64)
        _check(load().dabs_run_async(self.h, seed, flip_budget, _p(x), _p(e)))
        return int(e[0]), x

    def async_log(self) -> np.ndarray:
        m = np.zeros(1, np.int64)
        _check(load().dabs_async_log(self.h, None, 0, _p(m)))
        out = np.zeros(int(m[0]), np.uint32)
        if out.size:
            _check(load().dabs_async_log(self.h, _p(out), out.size, _p(m)))
        return out

    def jump_ms(self) -> float:
        v = np.zeros(1, np.float32)
        _check(load().dabs_jump_ms(self.h, _p(v)))
        return float(v[0])

    def async_lock_ns(self):
        w = np.zeros(1, np.uint64)
        h = np.zeros(1, np.uint64)
        _check(load().dabs_async_lock_ns(self.h, _p(w), _p(h)))
        return int(w[0]), int(h[0])

    def best(self):
        x = np.zeros(self.n, np.uint8)
        e = np.zeros(1, np.int64)
        _check(load().dabs_best(self.h, _p(x), _p(e)))
        return int(e[0]), x

    def energy(self, x) -> int:
        x = np.ascontiguousarray(x, dtype=np.uint8)
        e = np.zeros(1, np.int64)
        _check(load().dabs_energy(self.h, _p(x), _p(e)))
        return int(e[0])

    def stats(self) -> dabs_stats:
        s = dabs_stats()
        _check(load().dabs_get_stats(self.h, C.byref(s)))
        return s

    # -- parity hooks
    def debug_batch(self, slot: int, x, delta, E: int, ring, D, algo: int, seed: int, gen: int,
                    trace_cap: int = 0):
        x = np.array(x, dtype=np.uint8, copy=True)
        delta = np.array(delta, dtype=np.int32, copy=True)
        ring = np.array(ring, dtype=np.int32, copy=True)
        D = np.ascontiguousarray(D, dtype=np.uint8)
        Ea = np.array([E], np.int64)
        best = np.zeros(self.n, np.uint8)
        eb = np.zeros(1, np.int64)
        fl = np.zeros(1, np.int64)
        if trace_cap:
            tb = np.zeros(trace_cap, np.int32)
            te = np.zeros(trace_cap, np.int64)
            tp = np.zeros(trace_cap, np.int8)
            tptr = (_p(tb), _p(te), _p(tp))
        else:
            tb = te = tp = None
            tptr = (None, None, None)
        _check(load().dabs_debug_batch(self.h, slot, _p(x), _p(delta), _p(Ea), _p(ring), _p(D), algo, seed, gen,
                                       _p(best), _p(eb), _p(fl), *tptr, trace_cap))
        f = int(fl[0])
        out = dict(x=x, delta=delta, E=int(Ea[0]), ring=ring, best=best, ebest=int(eb[0]), flips=f)
        if trace_cap:
            m = min(f, trace_cap)
            out.update(trace_bit=tb[:m], trace_E=te[:m], trace_phase=tp[:m])
        return out

    def read_slot(self, slot: int):
        x = np.zeros(self.n, np.uint8)
        d = np.zeros(self.n, np.int32)
        E = np.zeros(1, np.int64)
        r = np.zeros(TABU_RING, np.int32)
        _check(load().dabs_read_slot(self.h, slot, _p(x), _p(d), _p(E), _p(r)))
        return dict(x=x, delta=d, E=int(E[0]), ring=r)

    def read_pool(self, pool: int):
        X = np.zeros((self.cap, self.n), np.uint8)
        E = np.zeros(self.cap, np.int64)
        seq = np.zeros(self.cap, np.uint64)
        a = np.zeros(self.cap, np.uint8)
        g = np.zeros(self.cap, np.uint8)
        _check(load().dabs_read_pool(self.h, pool, _p(X), _p(E), _p(seq), _p(a), _p(g)))
        return dict(X=X, E=E, seq=seq, algo=a, genop=g)

    def read_packet(self, slot: int):
        D = np.zeros(self.n, np.uint8)
        best = np.zeros(self.n, np.uint8)
        a = np.zeros(1, np.int32)
        g = np.zeros(1, np.int32)
        eb = np.zeros(1, np.int64)
        fl = np.zeros(1, np.int64)
        _check(load().dabs_read_packet(self.h, slot, _p(D), _p(a), _p(g), _p(best), _p(eb), _p(fl)))
        return dict(D=D, algo=int(a[0]), genop=int(g[0]), best=best, ebest=int(eb[0]), flips=int(fl[0]))

    def read_stats_pool(self, pool: int):
        d = np.zeros((5, 9), np.uint64)
        i = np.zeros((5, 9), np.uint64)
        _check(load().dabs_read_stats_pool(self.h, pool, _p(d), _p(i)))
        return d, i

    def trace_enable(self, slot: int, cap: int):
        _check(load().dabs_trace_enable(self.h, slot, cap))

    def trace_read(self, cap: int):
        tb = np.zeros(cap, np.int32)
        te = np.zeros(cap, np.int64)
        tp = np.zeros(cap, np.int8)
        cnt = np.zeros(1, np.int64)
        _check(load().dabs_trace_read(self.h, _p(tb), _p(te), _p(tp), _p(cnt)))
        m = int(cnt[0])
        return tb[:m], te[:m], tp[:m]


def probe_row_stream(rows: int, row_bytes: int, ctas_per_sm: int, inflight: int = 1, iters: int = 2000,
                     device: int = -1) -> float:
    """dabs_probe_row_stream: achievable row-stream GB/s (roofline denominator)."""
    v = np.zeros(1, np.float64)
    _check(load().dabs_probe_row_stream(device, rows, row_bytes, ctas_per_sm, inflight, iters, _p(v)))
    return float(v[0])


def torch_exchange(group=None):
    """Exchange hook over torch.distributed: all_gather_into_tensor of the
    library's device payload on the library's stream (NCCL over NVLink on a
    multi-GPU box).  Returns a callable for Solver(exchange=...)."""
    import torch
    import torch.distributed as dist

    def hook(user, send, recv, nbytes, stream):
        try:
            world = dist.get_world_size(group)
            s = _device_bytes(send, nbytes)
            r = _device_bytes(recv, nbytes * world)
            with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
                dist.all_gather_into_tensor(r, s, group=group)
            return 0
        except Exception:  # noqa: BLE001 -- reported as DABS_E_COMM
            return 1

    return hook


def _device_bytes(ptr: int, nbytes: int):
    """A torch uint8 CUDA tensor viewing library-owned device memory."""
    import torch

    class _View:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3,
                                    "strides": None}

    return torch.as_tensor(_View(), device="cuda")
