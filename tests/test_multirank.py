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


def _torch_exchange_worker(rank, world, port, backend, out):
    """One process per rank, both on cuda:0, exchanging through the library's
    torch_exchange hook (all_gather_into_tensor on the library's stream) --
    the code path the multi-GPU bench uses with NCCL."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group(backend, rank=rank, world_size=world)
    from paper_2207_03069_b200 import Solver, torch_exchange
    stream = torch.cuda.Stream()
    s = Solver(_instance(), rank=rank, world=world, exchange=torch_exchange(), stream=stream.cuda_stream, **CFG)
    s.reset(99)
    for _ in range(GENS):
        s.generation()
    E, X = s.best()
    st = s.stats()
    pools = [s.read_pool(p)["E"].tolist() for p in range(CFG["pools"] + 1)]
    out[rank] = (E, X.tolist(), (st.best_algo, st.best_genop, st.best_generation, st.best_slot), pools,
                 int(st.total_flips))
    s.close()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_torch_exchange_two_processes_equals_oracle(orc):
    """torch_exchange (the NCCL hook of the multi-GPU bench) driven by two real
    processes: NCCL needs one GPU per rank, so on the one-GPU box the same hook
    runs over gloo with CUDA tensors.  Pools, bests, first-best records and
    flip counts must equal the oracle's two-rank simulation."""
    from paper_2207_03069_b200 import build
    build.build()
    world = 2
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    ps = [ctx.Process(target=_torch_exchange_worker, args=(r, world, port, "gloo", out)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(600)
    assert all(p.exitcode == 0 for p in ps), [p.exitcode for p in ps]
    sysm = orc.System(_instance(), orc.Config(**CFG), world=world)
    sysm.reset(99)
    for _ in range(GENS):
        sysm.generation()
    for r in range(world):
        E, X, rec = sysm.ranks[r].best()
        gE, gX, grec, gpools, gflips = out[r]
        assert gE == E and gX == X.tolist()
        assert grec == (rec["algo"], rec["genop"], rec["gen"], rec["slot"])
        assert gflips == sysm.ranks[r].total_flips
        for p in range(CFG["pools"] + 1):
            assert gpools[p] == sysm.ranks[r].pool(p)["E"].tolist()
