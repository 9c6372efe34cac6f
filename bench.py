#!/usr/bin/env python
"""Benchmark: HODLR build+factor+solve fronts/s (BASELINE.json metric) on the
batched multifrontal level of BASELINE config 3.

Workload (config.workload "cfg3-batched-level"): every GPU owns
`--fronts-per-gpu` (default 64, the config's 8-GPU shard) independent 32^3
variable-coefficient fronts (n = 1024, per-cell conductivity exp(g), g ~
N(0,1) with seed = global front index; see paper_1403_5337_b200/frontgen.py),
ACA tol 1e-6, leaf 64.  One step = build (ACA of every off-diagonal block of
every front) + factor + one HODLR solve with one N(0,1) right-hand side
(seed = front index) per front.  Weak scaling: fronts per GPU is fixed, the
fronts shard across ranks with no data-path collective.  The 64 resident
fronts (537 MB) exceed the 126 MB L2, so no L2 flush is needed between steps.

Also reported: GMRES time-to-1e-10 on front 0 with the HODLR preconditioner
(the second half of the metric), the ACA kernel against the HBM roofline, the
CPU oracle (a restatement of the reference, tests-pinned) on a bounded
sample, and the end-to-end number through the public API with host buffers.

`--impl reference` times the reference algorithm on the host cores (the
oracle port; the reference is pure Python and cannot be installed on the GPU
box), same metric and config.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = "HODLR build+factor+solve fronts/sec (cfg3 batched level, fp64) + GMRES time-to-1e-10"
UNIT = "fronts/s"
DIMS = (32, 32, 32)
PLANE = 16
LEAF = 64
TOL = 1e-6
GMRES_TOL = 1e-10


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--fronts-per-gpu", type=int, default=64)
    ap.add_argument("--cpu-sample", type=int, default=8, help="fronts in the CPU oracle sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cfg4", action="store_true",
                    help="skip the BASELINE config-4 line item (96^3 front, GMRES time-to-1e-10)")
    ap.add_argument("--no-cfg12", action="store_true",
                    help="skip the BASELINE config-1 (48^3 BDLR) and config-2 (kNN slab, ACA vs "
                         "BDLR) line items")
    ap.add_argument("--no-cfg0", action="store_true",
                    help="skip the BASELINE config-0 line item (32^3 front, GMRES to 1e-12)")
    ap.add_argument("--level-fronts", type=int, default=512,
                    help="fronts of the whole-level line item at N=1 (BASELINE config 3's 512; "
                         "0 skips it)")
    return ap.parse_args()


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


# ---------------------------------------------------------------- rank launch
def _free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _rank_entry(rank, world, port, target, args):
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    rc = target(args)
    if rc:
        raise SystemExit(rc)


def launch_ranks(world, target, args):
    """One process per rank when bench.py is started without a launcher
    (``python bench.py --gpus N``): the same environment torchrun would set
    (RANK / LOCAL_RANK / WORLD_SIZE / MASTER_ADDR=127.0.0.1 / MASTER_PORT),
    then ``target(args)`` in every rank.  torch.distributed.run launches
    (WORLD_SIZE already set) bypass this."""
    import torch.multiprocessing as mp
    mp.spawn(_rank_entry, args=(world, _free_port(), target, args), nprocs=world, join=True)
    return 0


def init_dist(backend, device=None):
    """Process group from the launcher's environment (torchrun or launch_ranks)."""
    import torch.distributed as dist
    rank, _, world = env_rank()
    if world > 1 and not dist.is_initialized():
        kw = {"device_id": device} if device is not None else {}
        dist.init_process_group(backend, rank=rank, world_size=world, **kw)
    return dist


def config_dict(args, world):
    return {"workload": "cfg3-batched-level", "fronts_per_gpu": args.fronts_per_gpu,
            "total_fronts": args.fronts_per_gpu * world, "n": 1024, "grid": "32^3 variable-k, plane z=16",
            "scheme": "aca", "tol": TOL, "leaf": LEAF, "rhs_per_front": 1,
            "parallelism": f"fronts sharded over {world} GPU(s), no collective",
            "l2": "inputs (fronts_per_gpu x 8.4 MB) exceed the 126 MB L2; no flush"}


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and throttle reasons sampled every ~10 ms through NVML during
    the timed region (nvidia-smi's -lms floor is too coarse for short runs)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = None
        self._thr = None

    def start(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.idx]) if vis else self.idx
            h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception as exc:  # noqa: BLE001
            self.error = str(exc)
            return
        self._stop = threading.Event()

        def run():
            while not self._stop.is_set():
                try:
                    self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                    mask = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    for name, bit in self.REASONS.items():
                        if mask & bit:
                            self.reasons.add(name)
                except Exception:  # noqa: BLE001
                    pass
                time.sleep(0.01)

        self._thr = threading.Thread(target=run, daemon=True)
        self._thr.start()

    def stop(self):
        if self._thr is None:
            return {"sm_mhz": None, "sm_max_mhz": None,
                    "reasons": ["nvml unavailable: " + getattr(self, "error", "?")]}
        self._stop.set()
        self._thr.join()
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": float(self.max_mhz),
                "samples": len(self.samples), "reasons": sorted(self.reasons)}


# ---------------------------------------------------------------- inputs
def make_front(seed, device):
    from paper_1403_5337_b200 import frontgen as fg
    kc = fg.cell_conductivity(DIMS, seed)
    return fg.layered_grid_front(DIMS, 2, PLANE, conductivity=kc, device=device, return_torch=True)


def frontgen_flops(n, dims=DIMS, plane=PLANE):
    """FP64 flops of one front's plane-by-plane elimination: every eliminated
    layer (all but the separator plane) costs one n x n inverse, 2 n^3."""
    return (dims[2] - 1) * 2.0 * n ** 3


def make_fronts(seeds, device, chunk=64):
    """The config-3 fronts of `seeds`, generated on the GPU in batches of
    `chunk` (frontgen.layered_grid_fronts: this library's batched block
    Gauss-Jordan, hk_spd_inverse).  Input manufacture -- timed and reported
    (`frontgen`), part of no metric."""
    import torch
    from paper_1403_5337_b200 import frontgen as fg
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    parts = []
    for i in range(0, len(seeds), chunk):
        kcs = [fg.cell_conductivity(DIMS, s) for s in seeds[i:i + chunk]]
        parts.append(fg.layered_grid_fronts(DIMS, 2, PLANE, kcs, device=device))
    fronts = torch.cat(parts).contiguous()
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    n = fronts.shape[1]
    fl = frontgen_flops(n) * len(seeds)
    return fronts, {"fronts": len(seeds), "seconds": secs, "ms_per_front": 1e3 * secs / len(seeds),
                    "flops": fl, "tflops": fl / secs / 1e12, "solver": fg.frontgen_solver(),
                    "method": "plane-by-plane elimination, batched block Gauss-Jordan inverses "
                              "(hk_spd_inverse: 64 x 64 pivot blocks, DMMA GEMM updates), wall "
                              "time incl. host-side layer assembly"}


def rhs_for(seed, n):
    return np.random.default_rng(seed).standard_normal(n)


# ---------------------------------------------------------------- CPU oracle
def oracle_front(args_tuple):
    A, b = args_tuple
    from oracle import hodlr_oracle as O
    fact = O.factorize(A, LEAF, "aca", TOL)
    O.solve(fact, b)
    return 1


def cpu_sample(fronts_host, rhs_host, threads):
    """Time the oracle (reference restatement) on a bounded sample."""
    from threadpoolctl import threadpool_limits
    t0 = time.perf_counter()
    if threads == 1:
        with threadpool_limits(1):
            for A, b in zip(fronts_host, rhs_host):
                oracle_front((A, b))
    else:
        import multiprocessing as mp
        ctx = mp.get_context("fork")
        with ctx.Pool(threads, initializer=_limit_blas) as pool:
            pool.map(oracle_front, list(zip(fronts_host, rhs_host)))
    return time.perf_counter() - t0


def _limit_blas():
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)


# ---------------------------------------------------------------- reference arm
def run_reference(args):
    rank, _, world = env_rank()
    if rank != 0:
        return 0
    import torch
    cores = os.cpu_count() or 1
    gen = min(cores, 16)
    fronts = [make_front(s, "cpu").numpy() for s in range(gen)]
    n = fronts[0].shape[0]
    tasks = [(fronts[i % gen], rhs_for(i % gen, n)) for i in range(cores)]
    import multiprocessing as mp
    # fresh interpreters with single-threaded BLAS/OpenMP: forked children of
    # this (torch-initialised) process oversubscribed the cores ~25x
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    ctx = mp.get_context("spawn")
    times = []
    with ctx.Pool(cores, initializer=_limit_blas) as pool:
        for k in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            pool.map(oracle_front, tasks, chunksize=1)
            dt = time.perf_counter() - t0
            if k >= args.warmup:
                times.append(dt)
    total = sum(times)
    value = len(tasks) * len(times) / total
    del torch
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_dict(args, world), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{cores} fronts per step (one per core, {gen} distinct "
                                       "fronts), oracle/hodlr_oracle.py, 1 BLAS thread each"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our arm
def aca_algorithmic_bytes(tree, ranks):
    """Compulsory bytes of one ACA launch: per block, the
    r+1 row and column gathers of the pivot chain plus the U/V writes."""
    total = 0
    for f in range(ranks.shape[0]):
        for k, s in enumerate(tree.internal_nodes()):
            nd = tree.nodes[s]
            na = tree.nodes[nd.left].size
            nb = tree.nodes[nd.right].size
            for side, r in enumerate((ranks[f, 2 * k], ranks[f, 2 * k + 1])):
                total += 8 * ((int(r) + 1) + int(r)) * (na + nb)
    return total


def aca_l2_bytes(tree, ranks):
    """The L2 stream of one ACA launch beyond its compulsory bytes: pivot step
    s re-reads the s accepted crosses of both U (m x s) and V (n x s) for its
    residual row and column, 8 * (m + n) * r (r + 1) / 2 bytes per block of
    rank r (SURVEY.md §8(d) counts this as L2/SMEM traffic, not algorithmic)."""
    total = 0
    for f in range(ranks.shape[0]):
        for k, s in enumerate(tree.internal_nodes()):
            nd = tree.nodes[s]
            mn = tree.nodes[nd.left].size + tree.nodes[nd.right].size
            for r in (int(ranks[f, 2 * k]), int(ranks[f, 2 * k + 1])):
                total += 8 * mn * r * (r + 1) // 2
    return total


def l2_peak():
    """Measured full-chip L2 read bandwidth (tools/l2_peak.cu -> profiles/l2_peak.json)."""
    pf = ROOT / "profiles" / "l2_peak.json"
    if pf.exists():
        return float(json.loads(pf.read_text())["l2_gbs"]), "profiles/l2_peak.json l2_gbs (tools/l2_peak.cu)"
    return None, "no measured L2 peak"


def factor_flops(tree, ranks):
    """Algorithmic FP64 flops of one factorization per SURVEY.md §8(d) (leaf LU +
    Z-solve, coupling assembly + LU + correction), from the actual ranks."""
    total = 0.0
    for f in range(ranks.shape[0]):
        w = {0: 0}
        for k, s in enumerate(tree.internal_nodes()):      # preorder: parents first
            nd = tree.nodes[s]
            ru, rl = int(ranks[f, 2 * k]), int(ranks[f, 2 * k + 1])
            w[nd.left] = w[s] + ru
            w[nd.right] = w[s] + rl
        for s, nd in enumerate(tree.nodes):
            ws = w.get(s, 0)
            if nd.left < 0:
                b = nd.size
                total += 2.0 / 3.0 * b ** 3 + 2.0 * b * b * ws
        for k, s in enumerate(tree.internal_nodes()):
            nd = tree.nodes[s]
            na, nb = tree.nodes[nd.left].size, tree.nodes[nd.right].size
            ru, rl = int(ranks[f, 2 * k]), int(ranks[f, 2 * k + 1])
            ws = w[s]
            total += (2.0 * (na + nb) * ru * rl + 2.0 / 3.0 * (ru + rl) ** 3
                      + 2.0 * ws * (na * rl + nb * ru) + 2.0 * ws * (ru + rl) ** 2
                      + 2.0 * ws * (na * ru + nb * rl))
    return total


def solve_bytes(tree, ranks):
    """HBM bytes one HODLR solve (s = 1) must stream: every
    stored factor entry the sweep reads -- leaf inverses, V_low/V_up, S^-1 and
    d_left/d_right -- plus the rhs read and the solution write."""
    total = 0
    n = tree.nodes[0].size
    for f in range(ranks.shape[0]):
        for s, nd in enumerate(tree.nodes):
            if nd.left < 0:
                total += 8 * nd.size * nd.size
        for k, s in enumerate(tree.internal_nodes()):
            nd = tree.nodes[s]
            na, nb = tree.nodes[nd.left].size, tree.nodes[nd.right].size
            ru, rl = int(ranks[f, 2 * k]), int(ranks[f, 2 * k + 1])
            total += 8 * (na * rl + nb * ru + (ru + rl) ** 2 + na * ru + nb * rl)
        total += 16 * n
    return total


def fp64_peak():
    """Measured DMMA peak (profiles/fp64_peak.json, tools/fp64_peak.py) or the
    B200 datasheet-class fallback."""
    pf = ROOT / "profiles" / "fp64_peak.json"
    if pf.exists():
        d = json.loads(pf.read_text())
        for key in ("dmma_tflops", "dgemm_tflops"):
            if d.get(key):
                return float(d[key]), f"profiles/fp64_peak.json {key}"
    return 37.0, "fallback: B200 datasheet-class FP64 (no measured peak file)"


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1403_5337_b200 as hk
    from paper_1403_5337_b200 import _native as N
    from paper_1403_5337_b200.hodlr import HodlrBatch

    from paper_1403_5337_b200 import multifront as MF

    rank, local, world = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    init_dist("nccl", dev)
    F = args.fronts_per_gpu
    seeds = MF.shard_range(rank, world, F)
    fronts, gen = make_fronts(list(seeds), dev)
    n = fronts.shape[1]
    rhs = torch.from_numpy(np.stack([rhs_for(s, n) for s in seeds])).to(dev)
    work = torch.empty_like(rhs)
    cfg = hk.CompressionConfig(scheme="aca", tol=TOL)
    batch = HodlrBatch(n, LEAF, F)
    stream = torch.cuda.current_stream()

    def step():
        batch.factorize(fronts, cfg)
        work.copy_(rhs)
        batch.solve_(work)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    aca_s = 0.0
    fac_s = 0.0
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    launches0 = N.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
        aca_s += batch.plan.aca_seconds()
        tm = batch.plan.timings()
        fac_s += tm["leaf_lu"] + tm["schur"]
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    launches = N.launch_count() - launches0
    x_ref = work.clone()          # S(rhs) of the last timed step: the e2e path's expected output
    ms_max = MF.max_over_ranks(e0.elapsed_time(e1), device=dev)
    value = world * F * args.steps / (ms_max * 1e-3)

    # ---- roofline of the dominant kernel (batched ACA, HBM-bound by its compulsory bytes)
    peaks = {}
    pk = ROOT / "MEASURED_PEAKS.json"
    if pk.exists():
        peaks = json.loads(pk.read_text())
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    ranks = batch.ranks
    algo = aca_algorithmic_bytes(batch.tree, ranks)
    aca_avg = aca_s / args.steps
    achieved = algo / aca_avg / 1e9
    traffic = l2_traffic = None
    tf = ROOT / "profiles" / "r02_aca_traffic.json"
    if tf.exists():
        tj = json.loads(tf.read_text())
        traffic = tj.get("dram_bytes_per_build")
        l2_traffic = tj.get("l2_bytes_per_build")
    l2pk, l2src = l2_peak()
    l2b = aca_l2_bytes(batch.tree, ranks) + algo
    roof = {"kernel": "ACA build: aca_kernel size classes (4 persistent launches, all blocks of "
                      "all fronts), timed by CUDA events around the fork/join",
            "bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
            "frac": achieved / hbm_peak, "traffic": traffic,
            "algorithmic_bytes_per_launch": algo, "launch_ms": aca_avg * 1e3,
            "share_of_step": aca_avg * 1e3 / (ms_max / args.steps),
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if pk.exists() else "fallback 6.65 TB/s",
            # the same launch against the L2 roofline: the re-streaming of earlier
            # crosses (what bounds the pivot chains' sweeps) plus the compulsory bytes
            "l2": {"bound": "l2", "achieved": l2b / aca_avg / 1e9, "peak": l2pk, "unit": "GB/s",
                   "frac": (l2b / aca_avg / 1e9 / l2pk) if l2pk else None,
                   "traffic": l2_traffic, "algorithmic_bytes_per_launch": l2b,
                   "peak_source": l2src,
                   "traffic_source": "profiles/r02_aca_traffic.json (ncu lts__t_sectors_srcunit_tex "
                                     "read+write x 32 B, the four class launches serialised)"}}

    # ---- the other kernels against their rooflines: the factorization on the
    # FP64 tensor pipe (algorithmic flops of the actual ranks / the CUDA-event
    # time of the factor phase inside the timed steps)
    fpk, fpk_src = fp64_peak()
    ff = factor_flops(batch.tree, ranks)
    fac_avg = fac_s / args.steps
    rooflines = [{"kernel": "factorization (leaf Gauss-Jordan + level-batched DMMA GEMMs + "
                            "capacitance Gauss-Jordan), cfg3 64 fronts",
                  "bound": "tensor", "achieved": ff / fac_avg / 1e12, "peak": fpk,
                  "unit": "TFLOP/s", "frac": ff / fac_avg / 1e12 / fpk,
                  "algorithmic_flops_per_launch": ff, "launch_ms": fac_avg * 1e3,
                  "peak_source": fpk_src}]

    # the batch HODLR solve (s = 1, all fronts) alone: stored-factor bytes / time
    sv0 = torch.cuda.Event(enable_timing=True)
    sv1 = torch.cuda.Event(enable_timing=True)
    batch.solve_(work)
    torch.cuda.synchronize()
    sv0.record(stream)
    for _ in range(10):
        batch.solve_(work)
    sv1.record(stream)
    torch.cuda.synchronize()
    sv_ms = sv0.elapsed_time(sv1) / 10
    sb = solve_bytes(batch.tree, ranks)
    rooflines.append({"kernel": "HODLR solve sweep, cfg3 64 fronts, 1 rhs each", "bound": "hbm",
                      "achieved": sb / (sv_ms * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                      "frac": sb / (sv_ms * 1e-3) / 1e9 / hbm_peak,
                      "algorithmic_bytes_per_launch": sb, "launch_ms": sv_ms})

    # ---- GMRES time-to-1e-10 on front 0 (HODLR preconditioner)
    gm = {}
    if rank == 0:
        fact = batch.factorization(0)
        op = hk.DenseOperator(fronts[0])
        b0 = rhs[0].cpu().numpy()
        hk.gmres(op, b0, hk.GmresConfig(tol=GMRES_TOL), preconditioner=fact)   # warm
        torch.cuda.synchronize()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        res = hk.gmres(op, b0, hk.GmresConfig(tol=GMRES_TOL), preconditioner=fact)
        g1.record(stream)
        torch.cuda.synchronize()
        public_ms = g0.elapsed_time(g1)
        # the same GMRES on device buffers through the C ABI (hk_gmres): the
        # device-resident loop alone, without the public call's host<->device
        # copies of b, x and the history
        import ctypes
        bd = torch.from_numpy(b0).to(dev)
        xd = torch.empty_like(bd)
        its = ctypes.c_int64(0)
        hist = np.zeros(1000)
        tres = ctypes.c_double(0)
        flg = (ctypes.c_int32 * 2)()
        def native():
            N.check(N.lib().hk_gmres(batch.plan.h, 0, N.ptr(fronts[0]), n, n, N.ptr(bd), GMRES_TOL,
                                     1000, 1, None, N.ptr(xd), ctypes.byref(its),
                                     hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                     ctypes.byref(tres), flg, N.stream_handle()))
        native()
        torch.cuda.synchronize()
        dms = []
        for _ in range(5):
            g0.record(stream)
            native()
            g1.record(stream)
            torch.cuda.synchronize()
            dms.append(g0.elapsed_time(g1))
        gm = {"time_to_tol_ms": public_ms, "public_call_ms": public_ms,
              "device_loop_ms": float(np.median(dms)),
              "iterations": res.iterations,
              "converged": bool(res.converged), "true_residual": res.true_residual,
              "front": "cfg3 front 0 (seed 0), HODLR-ACA 1e-6 preconditioner, dense fp64 GEMV"}

    # ---- end to end through the public API with host buffers: every step's
    # fronts and rhs are copied from pinned host memory and its solution back,
    # inside the timed region; HodlrBatch.run_host_stream overlaps the copy of
    # step k+1 with the compute of step k (two device buffers, copy stream)
    e2e = None
    if not args.no_e2e:
        host_fronts = fronts.cpu().pin_memory()
        host_rhs = rhs.cpu().pin_memory()
        outs = [torch.empty_like(host_rhs).pin_memory() for _ in range(2)]
        mk = lambda k: [(host_fronts, host_rhs, outs[i % 2]) for i in range(k)]
        batch.run_host_stream(mk(args.warmup), cfg)
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        batch.run_host_stream(mk(args.steps), cfg)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = MF.max_over_ranks(e0.elapsed_time(e1), device=dev)
        xr = x_ref.cpu()
        x_out = outs[(args.steps - 1) % 2]
        x_check = float((x_out - xr).abs().max())
        x_rel = float((x_out - xr).norm() / xr.norm())
        e2e = {"value": world * F * args.steps / (e2e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(host_fronts.numel() * 8 + host_rhs.numel() * 8),
               "d2h_bytes_per_step": int(host_rhs.numel() * 8),
               "ms_per_step": e2e_ms / args.steps,
               "max_abs_diff_vs_device_path": x_check,
               "rel_diff_vs_device_path": x_rel,
               "path": "HodlrBatch.run_host_stream (public API): pinned host fronts/rhs -> "
                       "build+factor+solve -> host solution, copies overlapped with compute"}

    # ---- CPU baseline: the oracle on a bounded sample, rank 0 at N=1 only
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        k = min(args.cpu_sample, F)
        fh = [fronts[i].cpu().numpy() for i in range(k)]
        bh = [rhs[i].cpu().numpy() for i in range(k)]
        secs = cpu_sample(fh, bh, 1)
        cpu = {"value": k / secs, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"{k} of the {F} fronts, build+factor+solve, oracle/hodlr_oracle.py "
                         f"(numpy restatement of the reference), 1 thread, {secs:.1f} s"}

    # ---- BASELINE config 4: one 96^3 front (n = 9216), GMRES time-to-1e-10 on 4 rhs;
    # N > 1: HODLR-subtree sharding over NCCL (strong scaling)
    c4 = None
    if not args.no_cfg4:
        try:
            c4 = run_cfg4(dev, rank, world, hbm_peak)
        except Exception as exc:                 # a line item must not sink the headline line
            c4 = {"error": repr(exc)[:400]}
        if c4 and "rooflines" in c4:
            rooflines += c4.pop("rooflines")

    # ---- BASELINE configs 1 and 2: one front each, replicas only (rank 0 reports)
    c1 = c2 = None
    if not args.no_cfg12 and rank == 0:
        try:
            c1, c2 = run_cfg12(dev)
        except Exception as exc:
            c1 = c2 = {"error": repr(exc)[:400]}

    # ---- BASELINE config 0 (GMRES to 1e-12) and the whole 512-front level at N = 1
    c0 = lvl = None
    if not args.no_cfg0 and rank == 0:
        try:
            c0 = run_cfg0(dev)
        except Exception as exc:
            c0 = {"error": repr(exc)[:400]}
    grid = None
    if not args.no_cfg0 and rank == 0:
        try:
            grid = run_grid_solve(dev)
        except Exception as exc:
            grid = {"error": repr(exc)[:400]}
    if args.level_fronts > 0 and world == 1:
        try:
            lvl = run_level(dev, args.level_fronts, stream)
        except Exception as exc:
            lvl = {"error": repr(exc)[:400]}

    # per-front ranks of every rank's fronts (the one end-of-run gather)
    all_ranks = MF.gather_front_scalars(batch.ranks.astype(np.int64), device=dev)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": config_dict(args, world), "impl": "ours",
                "e2e": e2e, "gpu_launches": launches, "clocks": clk, "roofline": roof,
                "rooflines": rooflines,
                "cpu_baseline": cpu, "gmres": gm, "cfg0": c0, "level": lvl, "cfg4": c4,
                "cfg1": c1, "cfg2": c2, "frontgen": gen, "grid_solve": grid,
                "ranks_per_level_front0": [e["max_rank"] for e in batch.report(0).ranks_per_level],
                "fronts_gathered": int(all_ranks.shape[0]),
                "max_block_rank_all_fronts": int(all_ranks.max())}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_cfg4(dev, rank, world, hbm_peak):
    """Build + factor + GMRES (tol 1e-10, 4 N(0,1) rhs, seed 3) of the config-4 front.

    world == 1: one plan.  world > 1 (power of two): subtree.ShardedHodlr over
    NCCL, every GPU holding the front; times are the max over
    ranks.  The reference's single-thread CPU times on this config were
    measured for SURVEY.md §6.3 (20.2 s build+factor, 4.76 s GMRES for 4 rhs)."""
    import torch
    import paper_1403_5337_b200 as hk
    from paper_1403_5337_b200 import multifront as MF
    from paper_1403_5337_b200.frontgen import layered_grid_front
    from paper_1403_5337_b200.hodlr import HodlrBatch
    if world & (world - 1):
        return {"skipped": f"world size {world} is not a power of two"}
    front = layered_grid_front((96, 96, 96), "z", 48, device=dev, return_torch=True).contiguous()
    n = front.shape[0]
    cfg = hk.CompressionConfig(scheme="aca", tol=1e-4)
    B = np.random.default_rng(3).standard_normal((n, 4))
    stream = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    def timed(fn):
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        ev[0].record(stream)
        out = fn()
        ev[1].record(stream)
        torch.cuda.synchronize()
        return out, MF.max_over_ranks(ev[0].elapsed_time(ev[1]), device=dev)

    if world == 1:
        batch = HodlrBatch(n, 72, 1)
        for _ in range(2):                                      # warm (allocation, attributes, caches)
            batch.factorize(front[None], cfg)
        bf_all = [timed(lambda: batch.factorize(front[None], cfg))[1] for _ in range(3)]
        bf_ms = sorted(bf_all)[1]                               # median of 3
        fact = batch.factorization(0)
        op = hk.DenseOperator(front)
        ranks = [lv["max_rank"] for lv in batch.report(0).ranks_per_level]

        def solve_all():   # the 4 systems advance together (one GEMV / solve pass per iteration)
            return hk.gmres_batch(op, B, hk.GmresConfig(tol=1e-10), preconditioner=fact)
    else:
        from paper_1403_5337_b200 import subtree as ST
        comm = ST.TorchDistRanks(world.bit_length() - 1)
        sh = ST.ShardedHodlr(front, 72, comm)
        sh.factorize(cfg)
        _, bf_ms = timed(lambda: sh.factorize(cfg))
        ranks = None

        def solve_all():   # 4 systems in lock step: one sharded GEMV + solve per iteration
            return sh.gmres_batch(torch.from_numpy(B).to(dev), hk.GmresConfig(tol=1e-10))
    # HBM bytes one GMRES iteration must stream for the operator: the dense front
    per_iter = 8.0 * n * n
    solve_all()                                                  # warm
    res, gm_ms = timed(solve_all)
    dev_ms = None
    if world == 1:
        # the device-resident loop alone (hk_gmres_batch on device buffers),
        # without the public call's copies of B, X and the histories
        import ctypes
        from paper_1403_5337_b200 import _native as N
        Bd = torch.from_numpy(np.ascontiguousarray(B.T)).to(dev)      # (4, n): column-major n x 4
        Xd = torch.empty_like(Bd)
        its_h = np.zeros(4, dtype=np.int64)
        hist = np.zeros((4, 1000))
        tres = np.zeros(4)
        flg = np.zeros(8, dtype=np.int32)

        def native():
            N.check(N.lib().hk_gmres_batch(batch.plan.h, 0, N.ptr(front), n, n, N.ptr(Bd), 4, 1e-10,
                                           1000, 1, None, N.ptr(Xd), N.arr_ptr(its_h, N.I64),
                                           N.arr_ptr(hist, N.D), N.arr_ptr(tres, N.D),
                                           N.arr_ptr(flg, N.I32), N.stream_handle()))
        native()
        dev_ms = sorted(timed(native)[1] for _ in range(3))[1]
    roofs = []
    if world == 1:
        # GMRES operator GEMV (4 columns, one pass over the front) and the
        # 4-rhs HODLR solve, each timed alone over 20 launches by CUDA events
        from paper_1403_5337_b200 import _native as N
        X = torch.randn(n, 4, dtype=torch.float64, device=dev)
        Y = torch.empty_like(X)
        Xt = X.t().contiguous()

        def gemv():
            for _ in range(20):
                N.check(N.lib().hk_gemv(N.ptr(front), n, n, n, N.ptr(Xt), n, 4, N.ptr(Y), n,
                                        N.stream_handle()))
        gemv()
        _, gv_ms = timed(gemv)
        gv_ms /= 20
        W = Xt.clone()                                        # (s, n) = column-major n x 4

        def solves():
            for _ in range(20):
                fact.solve_device(W)
        solves()
        _, sv_ms = timed(solves)
        sv_ms /= 20
        sb = solve_bytes(batch.tree, batch.ranks)
        sbytes = sb + 8.0 * n * 3 * 2                           # columns 2..4 of rhs/solution
        roofs = [
            {"kernel": "GMRES operator GEMV (gemv4_kernel), cfg4 front 9216^2, 4 columns",
             "bound": "hbm", "achieved": per_iter / (gv_ms * 1e-3) / 1e9, "peak": hbm_peak,
             "unit": "GB/s", "frac": per_iter / (gv_ms * 1e-3) / 1e9 / hbm_peak,
             "algorithmic_bytes_per_launch": per_iter, "launch_ms": gv_ms},
            {"kernel": "HODLR solve sweep (leaf sgemv + pdot/S^-1 g/update per level), cfg4, 4 rhs",
             "bound": "hbm", "achieved": sbytes / (sv_ms * 1e-3) / 1e9, "peak": hbm_peak,
             "unit": "GB/s", "frac": sbytes / (sv_ms * 1e-3) / 1e9 / hbm_peak,
             "algorithmic_bytes_per_launch": sbytes, "launch_ms": sv_ms}]
    its = [r.iterations for r in res]
    out = {"workload": "cfg4 large single front: 96^3 Laplacian, plane z=48, n=9216, ACA 1e-4, "
                       "leaf 72, GMRES 1e-10 on default_rng(3) N(0,1) x 4",
           "n_gpus": world, "sharding": "none" if world == 1 else f"HODLR subtrees, level {world.bit_length() - 1}",
           "build_factor_ms": bf_ms, "gmres_4rhs_ms": gm_ms, "gmres_4rhs_device_loop_ms": dev_ms,
           "gmres_time_to_tol_ms_per_rhs": gm_ms / 4, "iterations": its,
           "true_residuals": [r.true_residual for r in res],
           "converged": all(bool(r.converged) for r in res),
           "gemv_bytes_per_iteration": per_iter,
           "gemv_floor_ms_4rhs": max(its) * per_iter / (hbm_peak * 1e9) * 1e3 / world,
           "gmres_mode": "hk_gmres_batch: 4 systems in lock step, one CUDA graph (conditional "
                         "WHILE node)" if world == 1 else
                         "subtree-sharded gmres_batch: 4 systems in lock step, row-slab GEMV + "
                         "sharded solve per iteration (NCCL all-reduce/all-gather)",
           "reference_cpu_1t_s": {"build_factor": 20.2, "gmres_4rhs": 4.76,
                                  "source": "SURVEY.md §6.3 (reference run in the build container)"}}
    if ranks is not None:
        out["max_rank_per_level"] = ranks
    if roofs:
        out["rooflines"] = roofs
    return out


def _single_front_item(dev, A, graph, schemes, leaf, gmres_tol, rhs_seed, tol=1e-4):
    """Cold and warm build+factor (CUDA events), GMRES time-to-tol, ranks, and
    the CPU oracle's build+factor on the same front (1 thread), per scheme.
    Cold = the first factorize of a fresh HodlrBatch (planning, allocation
    and, for BDLR, the GPU graph-distance selection, which a plan caches per
    graph); warm = the same plan again (selection cached)."""
    import time
    import torch
    import paper_1403_5337_b200 as hk
    from paper_1403_5337_b200.hodlr import HodlrBatch
    from oracle import hodlr_oracle as O          # CPU side-by-side only
    n = A.shape[0]
    Ad = torch.from_numpy(A).to(dev).contiguous()
    b = np.random.default_rng(rhs_seed).standard_normal(n)
    csr = (np.asarray(graph.indptr, dtype=np.int64), np.asarray(graph.indices, dtype=np.int64)) \
        if graph is not None else None
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    out = {}
    for scheme, depth in schemes:
        cfg = hk.CompressionConfig(scheme, tol=tol, depth=depth)
        g = csr if scheme == "bdlr" else None
        HodlrBatch(n, leaf, 1).factorize(Ad[None], cfg, graph=g)   # module / allocator warm-up
        torch.cuda.synchronize()
        batch = HodlrBatch(n, leaf, 1)
        ev[0].record()
        batch.factorize(Ad[None], cfg, graph=g)                 # cold: fresh plan and selection
        ev[1].record()
        torch.cuda.synchronize()
        cold_ms = ev[0].elapsed_time(ev[1])
        ms = []
        for _ in range(3):
            torch.cuda.synchronize()
            ev[0].record()
            batch.factorize(Ad[None], cfg, graph=g)
            ev[1].record()
            torch.cuda.synchronize()
            ms.append(ev[0].elapsed_time(ev[1]))
        fact = batch.factorization(0)
        op = hk.DenseOperator(Ad)
        hk.gmres(op, b, hk.GmresConfig(tol=gmres_tol), preconditioner=fact)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = hk.gmres(op, b, hk.GmresConfig(tol=gmres_tol), preconditioner=fact)
        torch.cuda.synchronize()
        gm_ms = (time.perf_counter() - t0) * 1e3
        _limit_blas()
        t1 = time.perf_counter()
        O.factorize(A, leaf, scheme, tol, depth, None, csr)
        cpu_s = time.perf_counter() - t1
        key = scheme if scheme == "aca" else f"bdlr_d{depth}"
        out[key] = {"build_factor_ms": min(ms), "build_factor_cold_ms": cold_ms,
                    "gmres_time_to_tol_ms": gm_ms,
                    "iterations": res.iterations, "converged": bool(res.converged),
                    "true_residual": res.true_residual,
                    "max_rank_per_level": [lv["max_rank"] for lv in batch.report(0).ranks_per_level],
                    "cpu_oracle_build_factor_s_1t": cpu_s}
    return out


def run_cfg0(dev):
    """BASELINE config 0: the constant-coefficient 32^3 front (plane z=16,
    n = 1024), ACA 1e-6, leaf 64, GMRES to 1e-12 on default_rng(0)."""
    from paper_1403_5337_b200 import frontgen as fg
    A0 = fg.layered_grid_front(DIMS, 2, PLANE, device=dev)
    return {"workload": "cfg0: 32^3 constant-coefficient front, plane z=16, n=1024, ACA 1e-6, "
                        "leaf 64, GMRES 1e-12, rhs default_rng(0)",
            **_single_front_item(dev, A0, None, [("aca", 1)], LEAF, 1e-12, 0, tol=TOL),
            "reference_cpu_1t_s": {"build_factor": 0.50, "gmres_to_1e-12": 0.014,
                                   "gmres_iterations": 4, "max_rank_per_level": [78, 78, 79, 64],
                                   "source": "SURVEY.md §6.3 (reference run in the build container)"}}


def run_grid_solve(dev):
    """The whole config-3 grid (32^3, variable k, seed 0) solved through its
    separator front (nested.PlaneNestedSolver: plane elimination on
    hk_spd_inverse, HODLR-ACA 1e-6 front factorization, HODLR-preconditioned
    GMRES to 1e-12 on the separator, plane forward/back substitution on
    hk_gemv), checked by the residual of the grid operator."""
    import time
    import torch
    import paper_1403_5337_b200 as hk
    from paper_1403_5337_b200 import frontgen as fg
    from paper_1403_5337_b200.nested import PlaneNestedSolver
    kc = fg.cell_conductivity(DIMS, 0)
    PlaneNestedSolver(DIMS, 2, PLANE, conductivity=kc, leaf=LEAF,
                      cfg=hk.CompressionConfig(scheme="aca", tol=TOL))          # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = PlaneNestedSolver(DIMS, 2, PLANE, conductivity=kc, leaf=LEAF,
                          cfg=hk.CompressionConfig(scheme="aca", tol=TOL))
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    b = np.random.default_rng(0).standard_normal((s.ext, s.nl))
    s.solve(b, hk.GmresConfig(tol=1e-12))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    x, res = s.solve(b, hk.GmresConfig(tol=1e-12))
    torch.cuda.synchronize()
    solve = time.perf_counter() - t1
    rel = float(np.linalg.norm(s.apply(x) - b) / np.linalg.norm(b))
    return {"workload": "cfg3 grid 32^3 (variable k, seed 0, 30752 unknowns) solved through its "
                        "z=16 separator front: forward/back plane substitution + HODLR-GMRES",
            "setup_ms": 1e3 * setup, "solve_ms": 1e3 * solve, "separator_gmres_iterations": res.iterations,
            "relative_residual": rel, "unknowns": int(s.ext * s.nl)}


def run_level(dev, nfronts, stream):
    """The whole BASELINE config-3 level on one GPU: `nfronts` (512) fronts in
    one HodlrBatch, build+factor+solve per step, CUDA-event timed over 3 steps
    after one warm-up.  Front generation is input manufacture, not timed."""
    import time
    import torch
    import paper_1403_5337_b200 as hk
    from paper_1403_5337_b200.hodlr import HodlrBatch
    fronts, gen = make_fronts(list(range(nfronts)), dev)
    rhs = torch.from_numpy(np.stack([rhs_for(s, 1024) for s in range(nfronts)])).to(dev)
    gen_s = gen["seconds"]
    work = torch.empty_like(rhs)
    cfg = hk.CompressionConfig(scheme="aca", tol=TOL)
    batch = HodlrBatch(1024, LEAF, nfronts)

    def step():
        batch.factorize(fronts, cfg)
        work.copy_(rhs)
        batch.solve_(work)
    step()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    steps = 3
    aca = 0.0
    ev[0].record(stream)
    for _ in range(steps):
        step()
        aca += batch.plan.aca_seconds()
    ev[1].record(stream)
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / steps
    out = {"workload": f"cfg3 whole level on 1 GPU: {nfronts} fronts in one batch (seeds "
                       f"0..{nfronts - 1}), build+factor+solve", "fronts": nfronts,
           "value": nfronts / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms, "steps": steps,
           "aca_ms": 1e3 * aca / steps, "generation_s": gen_s}
    del fronts, rhs, work, batch
    torch.cuda.empty_cache()
    return out


def run_cfg12(dev):
    """BASELINE config 1 (48^3 variable-k front, n = 2304, BDLR 1e-4 d=3 -- and ACA
    beside it) and config 2 (200k-point kNN slab front, ACA vs BDLR at 1e-4),
    GMRES to 1e-10.  Front generation (GPU) is input manufacture, not timed."""
    import time
    import warnings
    from paper_1403_5337_b200 import frontgen as fg
    warnings.filterwarnings("ignore", message=".*[Ss]parse.*")
    kc = fg.cell_conductivity((48, 48, 48), 1)
    A1 = fg.layered_grid_front((48, 48, 48), 2, 24, conductivity=kc, device=dev)
    g1 = fg.grid_graph(fg.GridSpec((48, 48, 48)), 2, 24)
    c1 = {"workload": "cfg1: 48^3 variable-k (seed 1) front, plane z=24, n=2304, leaf 64, "
                      "GMRES 1e-10, rhs default_rng(0)",
          **_single_front_item(dev, A1, g1, [("bdlr", 3), ("aca", 1)], 64, 1e-10, 0),
          "reference_cpu_1t_s": {"bdlr_d3_build_factor": 1.43, "bdlr_d3_gmres": 0.085,
                                 "aca_build_factor": 1.29, "aca_gmres": 0.166,
                                 "source": "SURVEY.md §6.3"}}
    t0 = time.perf_counter()
    kf = fg.knn_front(200000, h=0.005, leaf=64, device=dev, solver="cg")
    gen_s = time.perf_counter() - t0
    c2 = {"workload": "cfg2: 200k points (seed 2), 8-NN Laplacian + 1e-3 I, slab |x-0.5|<=0.005, "
                      "RCB order, leaf 64, ACA vs BDLR 1e-4, GMRES 1e-10, rhs default_rng(2)",
          "n": kf.n, "generation_s": gen_s, "generation": kf.info,
          **_single_front_item(dev, kf.front, kf.graph, [("aca", 1), ("bdlr", 3)], 64, 1e-10, 2)}
    return c1, c2


def main():
    args = parse()
    target = run_reference if args.impl == "reference" else run_ours
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        if args.impl == "reference":
            # only rank 0 of the reference arm does work (the CPU path)
            os.environ.update(RANK="0", LOCAL_RANK="0", WORLD_SIZE=str(args.gpus))
            return run_reference(args)
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            raise SystemExit(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible")
        return launch_ranks(args.gpus, target, args)
    return target(args)


if __name__ == "__main__":
    sys.exit(main())
