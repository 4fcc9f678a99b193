"""Multi-GPU semantics.

* gloo, world_size 2, CPU: each process runs the oracle for its own rank
  (its pools and slots) and exchanges payloads with dist.all_gather; the
  result must equal the single-process oracle simulating both ranks.
* GPU (one B200): two ranks of the CUDA path in two host threads, exchanging
  through a barrier-based hook (the same C-ABI exchange callback NCCL
  implements on a multi-GPU box); pools, bests and flip counts must equal the
  oracle's two-rank simulation bit for bit.
"""
import os
import socket
import threading

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _instance(n=60, seed=5):
    rng = np.random.default_rng(seed)
    return np.triu(rng.integers(-300, 301, size=(n, n))).astype(np.int16)


CFG = dict(s_milli=150, b_milli=1500, pools=2, slots=3, cap=12)
GENS = 4


def _gloo_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as orc
    U = _instance()
    w = orc.World(U, orc.Config(**CFG), rank=rank, world=world)
    w.reset(99)
    for _ in range(GENS):
        w.generation_local()
        mine = torch.from_numpy(w.export())
        bufs = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(bufs, mine)
        w.import_(np.concatenate([b.numpy() for b in bufs]))
    E, X, rec = w.best()
    pools = [w.pool(p)["E"].tolist() for p in range(CFG["pools"] + 1)]
    out[rank] = (E, X.tolist(), rec, pools, w.total_flips)
    dist.destroy_process_group()


def test_oracle_two_ranks_gloo_equals_single_process(orc):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [mp.Process(target=_gloo_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    U = _instance()
    sysm = orc.System(U, orc.Config(**CFG), world=world)
    sysm.reset(99)
    for _ in range(GENS):
        sysm.generation()
    for r in range(world):
        E, X, rec = sysm.ranks[r].best()
        gE, gX, grec, gpools, gflips = out[r]
        assert gE == E and gX == X.tolist() and grec == rec
        assert gflips == sysm.ranks[r].total_flips
        for p in range(CFG["pools"] + 1):
            assert gpools[p] == sysm.ranks[r].pool(p)["E"].tolist()
    # every rank sees the same box-wide best and flip count
    assert out[0][0] == out[1][0] and out[0][4] == out[1][4]


@pytest.mark.gpu
@pytest.mark.parametrize("jump", [False, True])
def test_gpu_two_ranks_one_device_equals_oracle(orc, jump):
    """(jump = True: the jump-start variant, R-30, across ranks)"""
    import torch
    from paper_2207_03069_b200 import Solver, build
    from paper_2207_03069_b200.dabs import _device_bytes
    build.build()
    world = 2
    U = _instance()
    barrier = threading.Barrier(world)
    sends = {}

    def make_hook(rank):
        def hook(user, send, recv, nbytes, stream):
            try:
                sends[rank] = (send, nbytes)
                torch.cuda.synchronize()
                barrier.wait()
                r = _device_bytes(recv, nbytes * world)
                for q in range(world):
                    sp, nb = sends[q]
                    r[q * nb:(q + 1) * nb].copy_(_device_bytes(sp, nb))
                torch.cuda.synchronize()
                barrier.wait()
                return 0
            except Exception:  # noqa: BLE001
                return 1
        return hook

    solvers = [Solver(U, rank=r, world=world, exchange=make_hook(r), jump=jump, **CFG) for r in range(world)]
    for s_ in solvers:
        s_.reset(99)
    errs = []

    def run(rank):
        try:
            for _ in range(GENS):
                solvers[rank].generation()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for x in th:
        x.start()
    for x in th:
        x.join(300)
    assert not errs, errs
    sysm = orc.System(U, orc.Config(**CFG, jump=jump), world=world)
    sysm.reset(99)
    for _ in range(GENS):
        sysm.generation()
    for r in range(world):
        E, X, rec = sysm.ranks[r].best()
        gE, gX = solvers[r].best()
        assert gE == E and np.array_equal(gX, X)
        st = solvers[r].stats()
        assert st.total_flips == sysm.ranks[r].total_flips
        assert (st.best_algo, st.best_genop, st.best_generation, st.best_slot) == (
            rec["algo"], rec["genop"], rec["gen"], rec["slot"])
        for p in range(CFG["pools"] + 1):
            g = solvers[r].read_pool(p)
            o = sysm.ranks[r].pool(p)
            np.testing.assert_array_equal(g["E"], o["E"])
            np.testing.assert_array_equal(g["X"], o["X"])
            np.testing.assert_array_equal(g["seq"], o["seq"])
