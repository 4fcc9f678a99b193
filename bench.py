#!/usr/bin/env python
"""bench.py -- bit-flips/s of the B200 DABS hot path (arXiv 2207.03069).

One step = one generation of the whole hot path: GA seeding
of every slot, one batch search per slot (Straight, Greedy, main rounds), pool
merge, exchange.  `value` = box-wide flips in the K timed steps / device time
(CUDA events on the library's stream, max over ranks).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload R32K|R64K|K2000s|TSP32|GS800|K16|QASP*]
    python bench.py --impl reference ...   # the CPU oracle on the host cores

Multi-GPU: torchrun --nproc-per-node N bench.py --gpus N ...; one rank per GPU,
NCCL all-gather of the pool snapshot per generation.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "bit-flips/sec per GPU and box at 1/2/4/8 B200; time-to-target QUBO energy"
UNIT = "flips/s"
L2_BYTES = 126 * 1024 * 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="dabs", choices=["dabs", "reference"])
    ap.add_argument("--workload", default="R32K",
                    choices=["K16", "GS800", "TSP32", "K2000s", "R32K", "R64K", "QASP1", "QASP16", "QASP256"])
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--slots", type=int, default=0, help="slots per pool (0 = library default)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="oracle sample size (cpu_baseline)")
    ap.add_argument("--ref-seconds", type=float, default=0.0,
                    help="reference arm: oracle seconds per step (0 = sized so the run ends within minutes)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-tts", action="store_true")
    ap.add_argument("--no-async", action="store_true", help="skip the asynchronous-schedule line (SURVEY f1)")
    ap.add_argument("--no-jump", action="store_true", help="skip the jump-start line (SURVEY f4)")
    ap.add_argument("--no-per-rule", action="store_true", help="skip the one-rule-per-run kernel figures")
    ap.add_argument("--launcher-selftest", action="store_true",
                    help="CPU check of the --gpus N launcher: every rank joins a gloo group, rank 0 prints the size")
    return ap.parse_args()


def free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def torchrun_cmd(n: int, argv) -> list:
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *argv]


def relaunch_torchrun(args) -> int:
    """`python bench.py --gpus N` without torchrun's environment: start N ranks
    (one per GPU, NCCL) through torch.distributed.run on 127.0.0.1; rank 0
    prints the JSON line."""
    return subprocess.call(torchrun_cmd(args.gpus, sys.argv[1:]), cwd=ROOT)


def launcher_selftest():
    import torch
    import torch.distributed as dist
    rank, world, _ = dist_env()
    dist.init_process_group("gloo")
    ids = [None] * world
    dist.all_gather_object(ids, (rank, os.getpid()))
    if rank == 0:
        print(json.dumps({"n_ranks": dist.get_world_size(), "ranks": sorted(r for r, _ in ids),
                          "pids_distinct": len({p for _, p in ids}) == world, "torch": torch.__version__}))
    dist.destroy_process_group()


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------ oracle timing
def oracle_sample(U, meta, seconds: float, seed: int):
    """Time the CPU oracle (as it stands) on host cores: one thread per core,
    each a persistent slot from X=0 running batches (random target, algorithm
    = thread mod 5, like generation 0 of the GPU run, where every pool row is a
    random sentinel) until its share of flips is done.  Returns (flips, s, cores)."""
    from oracle import oracle as orc
    orc.lib()
    n = U.shape[0]
    cores = os.cpu_count() or 1
    T, B = orc.flip_factor(meta["s_milli"], n), orc.flip_factor(meta["b_milli"], n)
    # calibrate the per-flip cost on one thread
    st = orc.SlotState.initial(U)
    D = orc.build_target(7, np.zeros(n, np.uint8), np.zeros(n, np.uint8), np.zeros(n, np.uint8),
                         seed=seed, gslot=10**6, gen=0)
    t0 = time.perf_counter()
    f = orc.batch_sample(U, st, D, 1, T=T, B=B, tabu=8, seed=seed, slot=10**6, gen=0,
                         flip_limit=max(20, 2_000_000 // max(n, 1)))
    per_flip = (time.perf_counter() - t0) / max(f, 1)
    quota = max(50, int(seconds / per_flip))
    results = [0] * cores

    def worker(t):
        s = orc.SlotState.initial(U)
        done, gen = 0, 0
        while done < quota:
            Dt = orc.build_target(7, s.x, s.x, s.x, seed=seed, gslot=t, gen=gen)
            done += orc.batch_sample(U, s, Dt, t % 5, T=T, B=B, tabu=8, seed=seed, slot=t, gen=gen,
                                     flip_limit=quota - done)
            gen += 1
        results[t] = done

    th = [threading.Thread(target=worker, args=(t,)) for t in range(cores)]
    t0 = time.perf_counter()
    for x in th:
        x.start()
    for x in th:
        x.join()
    dt = time.perf_counter() - t0
    return sum(results), dt, cores, quota


# ------------------------------------------------------------------ clocks
class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.p = None
        self.out = os.path.join("/tmp", f"dabs_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.f = open(self.out, "w")
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        self.f.close()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.out):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for name, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2207_03069_b200 import workloads as wl
    U, meta = wl.make(args.workload, seed=1)
    per_step = args.ref_seconds or max(2.0, min(15.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        oracle_sample(U, meta, per_step / 4, args.seed)
    flips = 0
    secs = 0.0
    cores = quota = 0
    for _ in range(args.steps):
        f, dt, cores, quota = oracle_sample(U, meta, per_step, args.seed)
        flips += f
        secs += dt
    value = flips / secs
    sample = (f"{args.steps} steps x {cores} threads x {quota} flips of persistent slots from X=0 "
              f"(random targets, algorithm = thread mod 5), workload {args.workload}")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic", "config": config_of(args.workload, U, meta, None),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def config_of(workload, U, meta, solver):
    n = int(U.shape[0])
    c = {"workload": workload, "n": n, "s": meta["s_milli"] / 1000, "b": meta["b_milli"] / 1000,
         "W_bytes": 2 * n * n, "ingest": "csr" if meta.get("sparse") else "dense"}
    if solver is not None:
        c.update(slots_per_gpu=solver.slots, pools_per_gpu=solver.pools, threads_per_search=solver.threads,
                 T=solver.T, B=solver.B)
    c["l2"] = ("inputs larger than L2 (W streamed from HBM)" if 2 * n * n > L2_BYTES
               else "L2 flushed (256 MiB write) between timed steps")
    return c


# ------------------------------------------------------------------ roofline helpers
def l2_row_stream_peak(n_rows: int, row_bytes: int) -> dict:
    """Measured L2 row-stream peak on this GPU (dabs_probe_row_stream): random
    rows of a buffer the size of the workload's W copied into shared memory by
    TMA bulk copies, 8/16/32 CTAs per SM, 1 row in flight each; the best."""
    from paper_2207_03069_b200.dabs import probe_row_stream
    rb = (row_bytes + 63) // 64 * 64
    best = (0.0, 0)
    for per_sm in (8, 16, 32):
        if per_sm * rb > 200 * 1024:
            continue
        g = probe_row_stream(n_rows, rb, per_sm, 1, 3000)
        best = max(best, (g, per_sm))
    return {"gbps": best[0], "ctas_per_sm": best[1], "rows": n_rows, "row_bytes": rb}


def ncu_traffic(workload: str):
    """DRAM (or L2) bytes per flip of batch_kernel from the committed ncu --set
    full capture of this workload (newest round first)."""
    for rnd in ("r02", "r01"):
        f = os.path.join(ROOT, "profiles", f"{rnd}_ncu_batch_{workload.lower()}.json")
        if os.path.exists(f):
            try:
                return json.load(open(f)), f
            except Exception:  # noqa: BLE001
                pass
    return None, None


# recorded targets for time-to-target (the paper's protocol).  TSP32 is
# pinned in closed form (R-22: cycle metric, E* = 2 m scale - m p); the others are
# the best energies of long runs of this solver, recorded in profiles/targets.json
def load_targets() -> dict:
    t = {"TSP32": {"target": -19872, "source": "closed form (cycle-metric TSP optimum, R-22), pinned"}}
    try:
        t.update(json.load(open(os.path.join(ROOT, "profiles", "targets.json"))))
    except Exception:  # noqa: BLE001
        pass
    return t


def oracle_replay(U, solver, meta, seed: int, seconds: float, torch):
    """cpu_baseline (SURVEY 8(d) "Oracle timing"): the oracle, as it stands,
    replays sampled slots' batches of one generation of THIS run -- same seeds,
    slot ids, generation, pre-generation states and packets -- one thread per
    host core, each bounded to a flip quota (a sample of the batch; ctypes
    releases the GIL inside the C oracle).  Completed batches must reproduce the
    device's flip counts (a free full-size parity check)."""
    from oracle import oracle as orc
    orc.lib()
    cores = os.cpu_count() or 1
    k = min(cores, solver.slots)
    sample = sorted(set(int(x) for x in np.linspace(0, solver.slots - 1, k).round()))
    pre = {s_: solver.read_slot(s_) for s_ in sample}
    gen = int(solver.stats().generations)
    solver.generation()
    torch.cuda.synchronize()
    pk = {s_: solver.read_packet(s_) for s_ in sample}
    n = U.shape[0]
    # calibrate: per-flip cost on one thread, from a copy of the first sampled slot
    s0 = sample[0]
    st = orc.SlotState(pre[s0]["x"].copy(), pre[s0]["delta"].copy(), pre[s0]["E"], pre[s0]["ring"].copy())
    t0 = time.perf_counter()
    f = orc.batch_sample(U, st, pk[s0]["D"], pk[s0]["algo"], T=solver.T, B=solver.B, tabu=8, seed=seed, slot=s0,
                         gen=gen, flip_limit=max(20, 2_000_000 // max(n, 1)))
    per_flip = (time.perf_counter() - t0) / max(f, 1)
    quota = max(50, int(seconds / per_flip))
    done = {}

    def worker(s_):
        stt = orc.SlotState(pre[s_]["x"].copy(), pre[s_]["delta"].copy(), pre[s_]["E"], pre[s_]["ring"].copy())
        done[s_] = orc.batch_sample(U, stt, pk[s_]["D"], pk[s_]["algo"], T=solver.T, B=solver.B, tabu=8, seed=seed,
                                    slot=s_, gen=gen, flip_limit=quota)
    th = [threading.Thread(target=worker, args=(s_,)) for s_ in sample]
    t0 = time.perf_counter()
    for x in th:
        x.start()
    for x in th:
        x.join()
    dt = time.perf_counter() - t0
    flips = sum(done.values())
    completed = [s_ for s_ in sample if done[s_] < quota]
    matched = sum(1 for s_ in completed if done[s_] == pk[s_]["flips"])
    return {"value": flips / dt, "unit": UNIT, "cores": len(sample), "kind": "oracle",
            "host_cores": cores, "cpu_model": cpu_model(),
            "sample": (f"{len(sample)} threads, each replaying one sampled slot's batch of generation {gen} of this "
                       f"run (same seed, slot, packet and pre-generation state) for up to {quota} flips; "
                       f"{flips} flips in {dt:.1f} s"),
            "replayed_batches_completed": len(completed), "completed_flip_counts_matched": matched}


# ------------------------------------------------------------------ main arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_torchrun(args))
    if args.launcher_selftest:
        return launcher_selftest()
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        assert dist.get_world_size() == world
    else:
        torch.cuda.set_device(0)
    from paper_2207_03069_b200 import Solver, build, torch_exchange
    from paper_2207_03069_b200 import workloads as wl
    if rank == 0:
        build.build()
    if world > 1:
        dist.barrier()
    U, meta = wl.make(args.workload, seed=1)
    n = U.shape[0]
    stream = torch.cuda.Stream()
    csr = Solver.to_csr(U) if meta.get("sparse") else None   # sparse instances enter via dabs_create_csr
    xchg = torch_exchange() if world > 1 else None
    solver = Solver(None if csr else U, csr=csr, s_milli=meta["s_milli"], b_milli=meta["b_milli"],
                    pools=meta.get("pools", 1),
                    slots=args.slots or meta.get("slots", 0), rank=rank, world=world,
                    device=torch.cuda.current_device(),
                    stream=stream.cuda_stream, exchange=xchg)
    solver.reset(args.seed)
    for _ in range(args.warmup):
        solver.generation()
    flush = None
    if 2 * n * n <= L2_BYTES:
        flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    clocks = Clocks(torch.cuda.current_device())
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    st0 = solver.stats()
    batch_ms = []
    local_flips = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    prev_local = st0.local_flips
    for k in range(args.steps):
        if flush is not None:
            with torch.cuda.stream(stream):
                flush.fill_(k & 0xFF)
        ev[k][0].record(stream)
        solver.generation()
        ev[k][1].record(stream)
        s = solver.stats()
        batch_ms.append(s.batch_ms_last)
        local_flips.append(s.local_flips - prev_local)
        prev_local = s.local_flips
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    st1 = solver.stats()
    t_ms = sum(a.elapsed_time(b) for a, b in ev)
    if world > 1:
        tt = torch.tensor([t_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    flips = st1.total_flips - st0.total_flips
    value = flips / (t_ms / 1e3)
    launches = int(st1.kernel_launches - st0.kernel_launches)

    # roofline of the dominant kernel (batch_kernel): algorithmic bytes = one
    # W row (2n bytes, int16) per flip; HBM-resident W
    # against the measured HBM copy bandwidth, L2-resident W against the
    # measured L2 row-stream peak of this GPU
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:  # noqa: BLE001
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    avg_batch_ms = float(np.mean(batch_ms))
    bytes_per_launch = float(np.mean(local_flips)) * 2 * n
    achieved = bytes_per_launch / (avg_batch_ms / 1e3) / 1e9
    prof, prof_f = ncu_traffic(args.workload)
    traffic, traffic_src = None, None
    l2_resident = 2 * n * n <= L2_BYTES
    if prof:
        per_flip = prof.get("dram_bytes_per_flip") if not l2_resident else prof.get("l2_bytes_per_flip",
                                                                                      prof.get("dram_bytes_per_flip"))
        if per_flip:
            traffic = per_flip * float(np.mean(local_flips))
            traffic_src = (f"ncu --set full capture {os.path.relpath(prof_f, ROOT)}: {per_flip:.0f} "
                           f"{'L2' if l2_resident and 'l2_bytes_per_flip' in prof else 'DRAM'} bytes per flip "
                           "x flips per launch")
    # the generation schedule's search kernel for this tier (runtime.cu pick_batch)
    kname = "tm_batch_kernel" if (n > 16384 and solver.threads == 256) else "batch_kernel"
    if l2_resident:
        l2 = l2_row_stream_peak(n, 2 * solver.n_pad)
        roofline = {"bound": "l2", "achieved": achieved, "peak": l2["gbps"], "unit": "GB/s",
                    "frac": achieved / l2["gbps"], "traffic": traffic, "traffic_source": traffic_src,
                    "kernel": kname,
                    "peak_source": (f"measured live: dabs_probe_row_stream, {l2['rows']} rows x {l2['row_bytes']} B "
                                    f"(this workload's W), TMA bulk row copies, {l2['ctas_per_sm']} CTAs/SM"),
                    "hbm_frac_context": achieved / hbm}
    else:
        roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                    "traffic": traffic, "traffic_source": traffic_src, "kernel": kname,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s"}
    roofline.update(bytes_per_flip=2 * n, batch_share_of_step=sum(batch_ms) / t_ms if world == 1 else None)

    cfg = config_of(args.workload, U, meta, solver)
    if world > 1:
        cfg["parallelism"] = (f"{world} ranks, one per GPU; pools and slots sharded, W replicated; NCCL all-gather "
                              f"of the pool snapshot per generation (communicator size {dist.get_world_size()})")
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": cfg, "roofline": roofline,
        "gpu_launches": launches, "gpu_launches_source": "dabs_stats.kernel_launches over the timed steps",
        "clocks": clk, "per_gpu_flips_per_s": value / world,
        "flips_per_step": [int(x) for x in local_flips], "batch_ms_per_step": [float(x) for x in batch_ms],
        "best_energy": st1.best_energy, "generations": int(st1.generations),
    }
    # ---- cpu_baseline: the oracle replaying this run's batches (rank 0, N = 1)
    oracle_s_per_gen = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = oracle_replay(U, solver, meta, args.seed, args.cpu_seconds, torch)
        oracle_s_per_gen = float(np.mean(local_flips)) / cb["value"]
        cb["oracle_s_per_generation_extrapolated"] = oracle_s_per_gen
        out["cpu_baseline"] = cb
    # ---- e2e: through the public API from pinned host memory.  One e2e step =
    # dabs_create (H2D of W, or of the CSR arrays) + dabs_run with a flip budget
    # of (warmup + steps) generations of the device measurement (so it includes
    # the cheaper first generation from X = 0, as the device run's warm-up does)
    # + D2H of the best vector and energy.
    if not args.no_e2e:
        Wp = torch.from_numpy(U).pin_memory()
        Wnp = Wp.numpy()
        e2e_flips, e2e_s = 0, 0.0
        budget = max(1, int(np.mean(local_flips)) * world * (args.warmup + args.steps))
        n_e2e = 2
        for k in range(n_e2e):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            s2 = Solver(None if csr else Wnp, csr=csr, s_milli=meta["s_milli"], b_milli=meta["b_milli"],
                        pools=meta.get("pools", 1),
                        slots=args.slots or meta.get("slots", 0), rank=rank, world=world,
                        device=torch.cuda.current_device(), stream=stream.cuda_stream,
                        exchange=torch_exchange() if world > 1 else None)
            E, x = s2.run(seed=args.seed + k, flip_budget=budget)
            dt = time.perf_counter() - t0
            if world > 1:
                tt = torch.tensor([dt], dtype=torch.float64, device="cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                dt = float(tt.item())
            e2e_flips += s2.stats().total_flips
            e2e_s += dt
            s2.close()
        h2d = int(2 * n * n) if csr is None else int(sum(a.nbytes for a in csr))
        out["e2e"] = {"value": e2e_flips / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
                      "d2h_bytes_per_step": int(n + 8), "steps": n_e2e,
                      "what": ("dabs_create" if csr is None else "dabs_create_csr") +
                              f"(W from pinned host) + dabs_run({args.warmup + args.steps} generations of "
                              "flips, from X = 0) + best readback, host wall clock"}
    # ---- time-to-target (the paper's protocol): success rate and
    # mean TTS over successes per workload with a target (TSP32: pinned optimum;
    # others: recorded best-known energies, profiles/targets.json), every rank
    # participating (SPMD).  TTS = host wall clock from dabs_reset to the end of
    # the generation that reached the target.  The oracle's TTS is the same
    # generation count (bit-identical trajectories) x the oracle's measured
    # seconds per generation of this workload (extrapolated, labelled as such).
    if not args.no_tts:
        targets = load_targets()
        names = [args.workload] if args.workload in targets else []
        if args.workload != "TSP32":
            names.append("TSP32")
        tts_all = {}
        for wname in names:
            tgt = targets[wname]
            if wname == args.workload:
                Ut, mt = U, meta
            else:
                Ut, mt = wl.make(wname, seed=1)
            pools = int(tgt.get("pools", mt.get("pools", 1)))
            limit = float(tgt.get("limit_s", 20))
            runs = int(tgt.get("runs", 3))
            csr_t = Solver.to_csr(Ut) if mt.get("sparse") else None
            st_ = Solver(None if csr_t else Ut, csr=csr_t, s_milli=mt["s_milli"], b_milli=mt["b_milli"], pools=pools,
                         rank=rank, world=world, device=torch.cuda.current_device(), stream=stream.cuda_stream,
                         target=int(tgt["target"]), time_limit_ns=int(limit * 1e9), exchange=xchg)
            res = []
            for r in range(runs):
                E, _ = st_.run(seed=1000 + r, flip_budget=1 << 62)
                stt = st_.stats()
                res.append({"ok": bool(E <= tgt["target"]), "tts_s": stt.time_to_best_ns / 1e9,
                            "generations": int(stt.generations), "best": int(E)})
            ok = [x for x in res if x["ok"]]
            entry = {"target": int(tgt["target"]), "target_source": tgt.get("source", ""), "runs": runs,
                     "pools_per_gpu": pools, "slots_per_gpu": int(st_.slots), "limit_s": limit,
                     "success_rate": len(ok) / runs,
                     "mean_tts_s": float(np.mean([x["tts_s"] for x in ok])) if ok else None,
                     "mean_generations_to_target": float(np.mean([x["generations"] for x in ok])) if ok else None,
                     "per_run": res,
                     "timer": "host wall clock from dabs_reset to the end of the generation that reached the target"}
            if wname == args.workload and oracle_s_per_gen and ok and pools == meta.get("pools", 1):
                entry["oracle_tts_s_extrapolated"] = entry["mean_generations_to_target"] * oracle_s_per_gen
                entry["oracle_tts_how"] = ("generations to target (identical for the oracle: bit-exact trajectories) "
                                           "x the oracle's measured seconds per generation (cpu_baseline)")
            st_.close()
            tts_all[wname] = entry
        # the asynchronous schedule (R-29) on TSP32, ~216 searches per pool, single rank
        if world == 1 and not args.no_async:
            Ut, mt = wl.make("TSP32", seed=1)
            sa_ = Solver(Ut, s_milli=mt["s_milli"], b_milli=mt["b_milli"], pools=11, one_wave=True,
                         device=torch.cuda.current_device(), stream=stream.cuda_stream, target=mt["target"],
                         time_limit_ns=int(20e9))
            atts = []
            for r in range(3):
                t0 = time.perf_counter()
                E, _ = sa_.run_async(seed=1000 + r, flip_budget=1 << 62)
                wall = time.perf_counter() - t0
                atts.append((E <= mt["target"], sa_.stats().time_to_best_ns / 1e9, wall))
            sa_.close()
            aok = [(x, wl_) for o, x, wl_ in atts if o]
            tts_all["TSP32"]["async_schedule"] = {
                "success_rate": len(aok) / len(atts),
                "mean_tts_s": float(np.mean([x for x, _ in aok])) if aok else None,
                "mean_wall_s": float(np.mean([w_ for _, w_ in aok])) if aok else None, "pools": 11,
                "timer": "host wall clock from dabs_reset to the merge that reached the target (device clock stamp, "
                         "same origin as the generation schedule)"}
        out["time_to_target"] = tts_all
    # ---- asynchronous schedule: the same workload and seed
    # through dabs_run_async -- one persistent kernel, one CTA per resident
    # search, no generation barrier -- for the same flips as the timed steps.
    # Kernel time by CUDA events on the library's stream (batch_ms_last).
    if world == 1 and not args.no_async:
        # pools: the paper's ~216 searches per pool, one wave of
        # resident searches (a quarter of the generation schedule's four waves)
        a_pools = max(1, round(solver.slots / 4 / 216))
        sa = Solver(None if csr else U, csr=csr, s_milli=meta["s_milli"], b_milli=meta["b_milli"],
                    pools=a_pools, one_wave=True, device=torch.cuda.current_device(),
                    stream=stream.cuda_stream)
        budget = int(sum(local_flips))
        sa.run_async(args.seed, max(1, budget // 4))   # warm-up
        if flush is not None:
            with torch.cuda.stream(stream):
                flush.fill_(1)
        t0 = time.perf_counter()
        sa.run_async(args.seed, budget)
        wall = time.perf_counter() - t0
        sta = sa.stats()
        wait_ns, hold_ns = sa.async_lock_ns()
        out["async_schedule"] = {
            "lock_hold_us_per_event": hold_ns / 1e3 / max(1, sta.generations),
            "lock_wait_us_per_event": wait_ns / 1e3 / max(1, sta.generations),
            "lock_busy_frac": hold_ns / 1e6 / max(1e-9, sta.batch_ms_last),
            "value": sta.total_flips / (sta.batch_ms_last / 1e3), "unit": UNIT,
            "wall_value": sta.total_flips / wall, "flips": int(sta.total_flips),
            "merge_events": int(sta.generations), "slots": int(sa.slots), "pools": a_pools,
            "kernel_ms": float(sta.batch_ms_last),
            "vs_generation_schedule": (sta.total_flips / (sta.batch_ms_last / 1e3)) / value,
            "what": "dabs_run_async: persistent kernel, one CTA per resident search, per-pool ticket locks, "
                    "merge/seed per batch (no generation barrier); value = flips / kernel time"}
        sa.close()
    # ---- kernel figures per selection rule: one main rule per run
    # (algo_mask), so the adaptive mix cannot move the number;
    # flips/s and the fraction of the 2n-byte HBM roofline, batch kernel time
    if world == 1 and not args.no_per_rule:
        names = ["MaxMin", "CyclicMin", "RandomMin", "PositiveMin", "TwoNeighbor"]
        per_rule = {}
        for a_ in range(5):
            sr = Solver(None if csr else U, csr=csr, s_milli=meta["s_milli"], b_milli=meta["b_milli"],
                        pools=meta.get("pools", 1), slots=args.slots or meta.get("slots", 0), algo_mask=1 << a_,
                        device=torch.cuda.current_device(), stream=stream.cuda_stream)
            sr.reset(args.seed)
            sr.generation()   # from X = 0
            fl_, ms_ = 0, 0.0
            for _ in range(2):
                f0 = sr.stats().local_flips
                sr.generation()
                st_r = sr.stats()
                fl_ += st_r.local_flips - f0
                ms_ += st_r.batch_ms_last
            v_ = fl_ / (ms_ / 1e3)
            per_rule[names[a_]] = {"flips_per_s": v_, "frac": v_ * 2 * n / 1e9 / roofline["peak"],
                                   "bound": roofline["bound"]}
            sr.close()
        out["per_rule"] = per_rule
    # ---- jump-start variant: the same generations with every
    # batch starting at its target; X, E, Delta from one hand-written tcgen05
    # kernel (int8 tensor cores on W's bytes x all targets, Delta/E epilogue).
    # Its roofline is the contraction's against the int8 dense peak.
    if world == 1 and not args.no_jump:
        sj = Solver(None if csr else U, csr=csr, s_milli=meta["s_milli"], b_milli=meta["b_milli"],
                    pools=meta.get("pools", 1), slots=args.slots or meta.get("slots", 0), jump=True,
                    device=torch.cuda.current_device(), stream=stream.cuda_stream)
        sj.reset(args.seed)
        for _ in range(args.warmup):
            sj.generation()
        jev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        j0 = sj.stats().total_flips
        jms = []
        for k in range(args.steps):
            if flush is not None:
                with torch.cuda.stream(stream):
                    flush.fill_(k & 0xFF)
            jev[k][0].record(stream)
            sj.generation()
            jev[k][1].record(stream)
            jms.append(sj.jump_ms())
        torch.cuda.synchronize()
        jt = sum(a.elapsed_time(b) for a, b in jev)
        stj = sj.stats()
        # two int8 contractions (W's high and low bytes) of slots x n_pad x n_pad,
        # 2 ops per multiply-add; the int8 dense peak is taken as 2x the measured
        # bf16 dense figure (NVIDIA's nominal ratio, 4.5 vs 2.25 POPS)
        gemm_ops = 2 * 2 * float(sj.n_pad) * float(sj.n_pad) * sj.slots
        tpk = 2.0 * (float(peaks.get("bf16_tflops", 0.0)) or 2250.0)
        gms = float(np.mean(jms))
        out["jump_start"] = {
            "value": (stj.total_flips - j0) / (jt / 1e3), "unit": UNIT, "ms_per_step": jt / args.steps,
            "best_energy": int(stj.best_energy), "best_energy_plain": int(st1.best_energy),
            "generations": int(stj.generations),
            "contraction_ms_per_step": gms, "contraction_share_of_step": gms * args.steps / jt,
            "roofline": {"bound": "tensor", "achieved": gemm_ops / (gms / 1e3) / 1e12, "peak": tpk,
                         "unit": "TOP/s (int8)", "frac": gemm_ops / (gms / 1e3) / 1e12 / tpk,
                         "kernel": "jt_gemm_kernel (tcgen05.mma kind::i8, TMEM accumulators, fused Delta/E epilogue) "
                                   "+ jt_tile_d / jt_finish",
                         "peak_source": "2 x MEASURED_PEAKS.json bf16_tflops (int8 dense = 2 x bf16 dense, nominal)"},
            "what": "generations with jump-start batches (X = D, E and Delta from W.D) instead of Straight"}
        sj.close()
    if rank == 0:
        print(json.dumps(out))
    solver.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
