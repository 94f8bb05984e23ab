#!/usr/bin/env python
"""Benchmark: full-Greeks Heston Milstein Monte Carlo on B200.

Headline workload (BASELINE.json configs[2], the metric's own config):
arithmetic-Asian call, 252 daily fixings, 2^24 paths x 252 Milstein steps,
BASELINE parameter set A, price + Delta + Gamma + Vega + Rho (+ FD Delta,
FD Rho) from ONE fused pass with common-random-number bumps.  A bench
"step" is one complete full-Greeks evaluation of that job.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N > 1: launched under torch.distributed.run, one rank per GPU; the 2^24
paths are split across ranks (strong scaling) and the chunk partials are
exchanged once per step by libhmc's NCCL communicator
(hmc_comm_gather_chunks).  Rank 0 prints ONE JSON line.  HMC_DIST_BACKEND=gloo
(tests only) runs the ranks on a gloo group with host-staged exchange, so
several ranks can share one GPU.

--impl reference: the reference's own compiled CPU kernel (oracle/_ref,
built from the reference's _core.c) driven by the restated reference engine
on all host cores, on a bounded sample of the same workload (rank 0 only).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_PATHS = 2 ** 24
N_STEPS = 252
METRIC = "path_steps_per_sec_full_greeks"
UNIT = "path-steps/s"
MUFU_PER_PATH_STEP = 10      # BASELINE.md roofline: Asian full Greeks
FP32_PER_PATH_STEP = 45
N_SM = 148


MUFU_PEAK_FILE = os.path.join(ROOT, "profiles", "r02_mufu_peak.json")
DIST_BACKEND = os.environ.get("HMC_DIST_BACKEND", "nccl")   # gloo: several ranks on one GPU (tests)


def mufu_per_clk() -> tuple[float, str]:
    """MUFU ops per SM clock: the committed microbenchmark measurement
    (tools/mufu_bench.cu on a B200 of this pool, min over the ops the path
    kernels issue), else the nominal 16."""
    try:
        with open(MUFU_PEAK_FILE) as f:
            ops = json.load(f)["ops"]
        v = min(ops[k]["ops_per_clk_per_sm"] for k in ("ex2", "lg2", "sqrt", "sin", "cos"))
        return v, "profiles/r02_mufu_peak.json (tools/mufu_bench.cu, min over ex2/lg2/sqrt/sin/cos)"
    except (OSError, KeyError, ValueError):
        return 16.0, "nominal 16 MUFU ops/clk/SM (profiles/r02_mufu_peak.json missing)"


def workload():
    from paper_2309_10477_b200 import BENCH_PARAMS, HestonParams, OptionSpec, SimConfig, daily_fixings
    p = HestonParams(**BENCH_PARAMS)
    spec = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0,
                      averaging_times=daily_fixings(1.0, N_STEPS))
    cfg = SimConfig(scheme="milstein", sampler="pseudo", n_paths=N_PATHS, n_steps=N_STEPS,
                    n_runs=1, seed=42, precision="fp32")
    return p, spec, cfg


# canonical MUFU ops per path-step of each secondary workload (the MUFU
# roofline): European full Greeks 4 (Box-Muller) + 3
# sqrt(v); Sobol 2 lg2 (quantiles) + 3 sqrt + 3 ex2; surface = the Asian
# step (10).  The Sobol drivers are issue-bound, not MUFU-bound, so their
# fraction is a lower bound on how busy the chip is.
SECONDARY_MUFU = {"c2": 7, "c4": 8, "c5": 10}


def secondary_workloads(reps: int = 3, sm_mhz: float = 1965.0, max_over_ranks=None) -> dict:
    """The other BASELINE configs through the public API (CUDA events around
    each call; host overhead included).  At N > 1 every rank runs its slice
    of every job (the engine shards by itself) and the time is the max over
    ranks; path-steps/s is whole-job."""
    import numpy as np
    import torch
    from paper_2309_10477_b200 import (BENCH_PARAMS, HestonParams, OptionSpec, SimConfig, engine, greeks,
                                       price, surface, daily_fixings)
    p = HestonParams(**BENCH_PARAMS)
    euro = OptionSpec("european", "call", 100.0, 1.0, 100.0)
    asian = OptionSpec("asian_arithmetic", "call", 100.0, 1.0, 100.0,
                       averaging_times=daily_fixings(1.0, N_STEPS))
    jobs = {
        # config 1 (the reference's CPU-runnable case): European price + Delta,
        # 1e5 paths x 252 Milstein steps, the reference's greeks() keys --
        # launch- and latency-bound at this size
        "c1_european_price_delta_1e5x252": (
            lambda: engine._execute(p, euro, SimConfig(scheme="milstein", n_paths=100_000, n_steps=252,
                                                       n_runs=1, seed=7), want_greeks=False),
            100_000 * 252),
        "c2_european_full_greeks_2^22x252": (
            lambda: greeks(p, euro, SimConfig(scheme="milstein", n_paths=2**22, n_steps=252,
                                              n_runs=1, seed=7)), 2**22 * 252),
        # the headline job at the reference's own precision: the reference's
        # SplitMix64 stream + Acklam/Halley ndtri in fp64, its operation order
        "c3_fp64_replay_asian_full_greeks_2^24x252": (
            lambda: greeks(p, asian, SimConfig(scheme="milstein", n_paths=N_PATHS, n_steps=N_STEPS,
                                               n_runs=1, seed=42, precision="fp64")),
            N_PATHS * N_STEPS),
        "c4_sobol_rqmc_asian_full_greeks_2^22x252": (
            lambda: greeks(p, asian, SimConfig(scheme="milstein", sampler="sobol",
                                               sobol_highdim_ack=True, sobol_scramble=True,
                                               n_paths=2**22, n_steps=252, n_runs=1, seed=7)),
            2**22 * 252),
        "c4_sobol_rqmc_bridge16_asian_full_greeks_2^22x252": (
            lambda: greeks(p, asian, SimConfig(scheme="milstein", sampler="sobol",
                                               sobol_highdim_ack=True, sobol_scramble=True,
                                               sobol_bridge=16, n_paths=2**22, n_steps=252,
                                               n_runs=1, seed=7)),
            2**22 * 252),
        "exact_bk_european_price_2^17": (      # compare with cpu_baseline_exact (price only)
            lambda: price(p, euro, SimConfig(scheme="exact", n_paths=2**17, n_steps=1, n_runs=1,
                                             seed=7)), 2**17),
        "exact_bk_european_full_greeks_2^17": (
            lambda: greeks(p, euro, SimConfig(scheme="exact", n_paths=2**17, n_steps=1, n_runs=1,
                                              seed=7)), 2**17),
        "c5_surface_64Kx8T_euro+asian_full_greeks_2^22x504": (
            lambda: surface(p, np.arange(70.0, 134.0, 1.0), [0.25 * i for i in range(1, 9)],
                            SimConfig(scheme="milstein", n_paths=2**22, n_steps=504, n_runs=1,
                                      seed=7)), 2**22 * 504),
    }
    mufu_clk, _ = mufu_per_clk()
    out = {}
    for name, (fn, path_steps) in jobs.items():
        fn()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[len(ts) // 2]
        if max_over_ranks is not None:
            ms = max_over_ranks([ms])[0]
        out[name] = {"ms": ms, "path_steps_per_s": path_steps / (ms / 1e3)}
        mufu = SECONDARY_MUFU.get(name[:2])
        if mufu:
            peak = N_SM * mufu_clk * sm_mhz * 1e6 / mufu
            out[name].update(mufu_per_path_step=mufu, mufu_roofline_frac=path_steps / (ms / 1e3) / peak)
    return out


def cpu_exact_block(n_paths: int = 2 ** 13) -> dict:
    """The reference's own Broadie-Kaya kernel (oracle/_ref) on all host
    cores, European, one [0, T] step, 4096-path jobs as engine.py."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    import numpy as np
    from paper_2309_10477_b200 import BENCH_PARAMS, HestonParams
    core = oracle.ref_core()
    if core is None:
        return {"value": None}
    p = HestonParams(**BENCH_PARAMS)
    workers = os.cpu_count() or 1
    jobs = [(lo, min(lo + 512, n_paths)) for lo in range(0, n_paths, 512)]
    times, flags = np.array([0.0, 1.0]), np.array([1], dtype=np.int64)
    with ThreadPoolExecutor(workers) as pool:
        t0 = time.perf_counter()
        list(pool.map(lambda j: core.exact_batch(p, 100.0, times, flags, j[0], j[1], 7, None), jobs))
        secs = time.perf_counter() - t0
    return {"value": n_paths / secs, "unit": "paths/s", "cores": workers, "kind": "reference",
            "sample": f"{n_paths} European Broadie-Kaya paths (1 step), 512-path jobs"}


def reference_config_block(n_gpus: int, n_timed: int, workers: int) -> dict:
    """What the reference arm actually runs (not the B200 arm's block)."""
    return {"workload": "asian_arith_call_daily_fixings_full_greeks",
            "paths": N_PATHS, "paths_timed_per_step": n_timed, "time_steps": N_STEPS,
            "fixings": N_STEPS, "scheme": "milstein",
            "greeks": ["price", "delta", "rho", "gamma (CRN FD)", "vega (CRN FD)"],
            "params": "BASELINE A: S0=K=100 T=1 r=0.03 v0=0.04 kappa=2 theta=0.04 xi=0.3 rho=-0.7",
            "rng": "splitmix64 counter stream + Acklam/Halley ndtri (the reference's _core)",
            "state": "fp64", "sums": "fp64 (numpy pairwise per 4096-path job, math.fsum across jobs)",
            "kernel": "reference _core.discretised_batch compiled from the reference's _core.c "
                      "(oracle/_ref), GIL released",
            "engine": "restated reference engine (oracle/engine.py, pinned bit-exact to the "
                      "reference's engine.per_run_values in tests/test_oracle.py)",
            "full_greeks": "greeks() (price, pathwise Delta/Rho) + 4 CRN bumped price() passes "
                           "(S0 +/- 0.5 %, v0 +/- 1 %)",
            "threads": workers, "parallelism": "host threads (rank 0 only)"}


def config_block(n_gpus: int) -> dict:
    return {"workload": "asian_arith_call_daily_fixings_full_greeks",
            "paths": N_PATHS, "time_steps": N_STEPS, "fixings": N_STEPS, "scheme": "milstein",
            "greeks": ["price", "delta", "gamma", "vega", "rho", "delta_fd", "rho_fd"],
            "params": "BASELINE A: S0=K=100 T=1 r=0.03 v0=0.04 kappa=2 theta=0.04 xi=0.3 rho=-0.7",
            "rng": "philox4x32-10 + box-muller", "state": "fp32 registers", "sums": "fp64",
            "l2": "256 MiB buffer written between timed iterations (kernel has no HBM inputs)",
            "parallelism": f"dp{n_gpus}"}


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML)
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 - clocks are reported as unavailable
            self.nv = None
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.nv:
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref = the reference's own compiled kernel)
# ---------------------------------------------------------------------------
def cpu_reference_pass(n_paths: int, workers: int) -> float:
    """Full-Greeks set the reference way: engine.greeks (price, pathwise
    Delta/Rho) + 4 CRN re-runs with S0 +/- h and v0 +/- h for Gamma/Vega
    (BASELINE.md CPU-baseline plan).  Returns wall seconds."""
    from oracle import engine as oe
    from paper_2309_10477_b200 import HestonParams, OptionSpec, SimConfig
    p, spec, _ = workload()
    cfg = SimConfig(scheme="milstein", n_paths=n_paths, n_steps=N_STEPS, n_runs=1, seed=42)
    h = 0.005 * spec.spot
    hv = 0.01 * p.v0
    bump_s = lambda d: OptionSpec(spec.style, spec.right, spec.strike, spec.maturity,  # noqa: E731
                                  spec.spot + d, spec.averaging_times)
    bump_v = lambda d: HestonParams(p.kappa, p.theta, p.sigma, p.rho, p.r, p.v0 + d)  # noqa: E731
    t0 = time.perf_counter()
    oe.per_run_values(p, spec, cfg, True, "reference", workers)
    for s in (bump_s(h), bump_s(-h)):
        oe.per_run_values(p, s, cfg, False, "reference", workers)
    for pp in (bump_v(hv), bump_v(-hv)):
        oe.per_run_values(pp, spec, cfg, False, "reference", workers)
    return time.perf_counter() - t0


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline_block(n_paths: int = 0) -> dict:
    import oracle
    workers = os.cpu_count() or 1
    n_paths = n_paths or max(2 ** 16, 4 * 4096 * workers)
    kind = "reference" if oracle.ref_core() is not None else "port"
    if kind == "port":
        return {"value": None, "unit": UNIT, "cores": workers, "kind": "port",
                "sample": "oracle/_ref missing; not timed"}
    cpu_reference_pass(2 ** 12, workers)  # warm the pool / page in
    secs = cpu_reference_pass(n_paths, workers)
    one = cpu_reference_pass(4096, 1)      # one reference job on one core
    return {"value": n_paths * N_STEPS / secs, "unit": UNIT, "cores": workers, "kind": kind,
            "sample": f"{n_paths} paths x {N_STEPS} steps, Asian daily fixings, full Greeks as "
                      f"greeks() + 4 CRN bumped price() passes, {secs:.2f} s wall",
            "seconds": secs, "per_core_value": 4096 * N_STEPS / one, "cpu_model": _cpu_model()}


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    workers = os.cpu_count() or 1
    if oracle.ref_core() is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    n = max(2 ** 15, 2 * 4096 * workers)   # >= 2 reference jobs per worker
    n = int(os.environ.get("HMC_BENCH_REF_PATHS", n))  # tests: a smaller sample
    for _ in range(args.warmup):
        cpu_reference_pass(n, workers)
    times = [cpu_reference_pass(n, workers) for _ in range(args.steps)]
    secs = sum(times) / len(times)
    value = n * N_STEPS / secs
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs * 1000.0,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": reference_config_block(args.gpus, n, workers),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "reference",
                             "sample": f"{n} of the {N_PATHS} paths per step (bounded sample), "
                                       "reference _core kernel + restated reference engine, "
                                       "full Greeks = greeks() + 4 CRN bumped price() passes"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def run_b200(args) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2309_10477_b200 import _lib, engine, greeks, parallel

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    distributed = "LOCAL_RANK" in os.environ  # launched by torch.distributed.run
    gloo = distributed and DIST_BACKEND == "gloo"
    # gloo (tests): ranks may share GPUs; production: one GPU per rank
    dev_index = local % torch.cuda.device_count() if gloo else local
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if args.gpus != world and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch N>1 with "
              f"torch.distributed.run (one process per GPU) -- reporting n_gpus={world}",
              file=sys.stderr)
    if distributed:
        if gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def max_over_ranks(vals):
        if not distributed:
            return list(vals)
        t = torch.tensor(vals, dtype=torch.float64, device="cpu" if gloo else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    def barrier():
        if distributed:
            dist.barrier()

    p, spec, cfg = workload()
    L = _lib.lib()

    # resident job: structs, workspace and partial buffers allocated once
    job = engine.Job(p, spec, cfg, True)
    sl = parallel.shard(cfg.n_paths, rank, world)
    job.sim.path_lo, job.sim.path_hi = sl.path_lo, sl.path_hi
    stream = torch.cuda.current_stream(dev)
    work = torch.empty(int(L.hmc_workspace_bytes(ctypes.byref(job.sim))), dtype=torch.uint8, device=dev)
    loc = torch.zeros((cfg.n_runs, sl.n_chunks, _lib.HMC_NW), dtype=torch.float64, device=dev)
    out = torch.empty((cfg.n_runs, _lib.HMC_NW), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev)
    launches_per_step = 3  # path kernel + tiles->chunks + chunks->runs (+ NCCL's own at N > 1)

    def step(ev0=None, ev1=None):
        if ev0 is not None:
            ev0.record(stream)
        _lib.check(L.hmc_greeks_chunks(ctypes.byref(job.model), ctypes.byref(job.product),
                                       ctypes.byref(job.sim), ctypes.c_void_p(loc.data_ptr()),
                                       ctypes.c_void_p(work.data_ptr()),
                                       ctypes.c_void_p(stream.cuda_stream)))
        if ev1 is not None:
            ev1.record(stream)
        full = parallel.gather_chunks(loc, cfg.n_paths)      # libhmc NCCL exchange at N > 1
        _lib.check(L.hmc_reduce_chunks(ctypes.c_void_p(full.data_ptr()), cfg.n_runs, full.shape[1],
                                       ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(stream.cuda_stream)))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev_index) as clocks:
        for e0, e1, e2 in ev:
            flush.fill_(1)                       # evict L2 between timed iterations
            step(e0, e1)
            e2.record(stream)
        torch.cuda.synchronize()
    barrier()
    step_ms = [e0.elapsed_time(e2) for e0, _, e2 in ev]
    kern_ms = [e0.elapsed_time(e1) for e0, e1, _ in ev]
    tot_step, tot_kern = max_over_ranks([sum(step_ms), sum(kern_ms)])
    ms_per_step = tot_step / args.steps
    kernel_ms = tot_kern / args.steps
    path_steps = cfg.n_paths * N_STEPS
    value = path_steps / (ms_per_step / 1000.0)

    # e2e: the public API call a user makes (host structs in, host McSummary
    # out; step tables H2D and sums D2H inside every timed call)
    e2e_times = []
    g = None
    for i in range(0 if args.no_e2e else max(2, args.steps // 2) + 1):
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g = greeks(p, spec, cfg)
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = sorted(e2e_times[1:])[len(e2e_times[1:]) // 2] if e2e_times else float("nan")
    e2e_s = max_over_ranks([e2e_s])[0]
    h2d = (N_STEPS + 1) * (32 + 16) + job.avg_idx.nbytes
    d2h = cfg.n_runs * _lib.HMC_NW * 8

    clk = clocks.summary()
    f_mhz = clk["sm_mhz"] or 1965.0
    secondary = None
    if not args.no_e2e and not args.no_secondary:
        secondary = secondary_workloads(sm_mhz=f_mhz, max_over_ranks=max_over_ranks)

    if rank == 0:
        mufu_clk, mufu_src = mufu_per_clk()
        peak = N_SM * mufu_clk * f_mhz * 1e6 / MUFU_PER_PATH_STEP  # per GPU
        local_path_steps = sl.n_paths * N_STEPS
        achieved = local_path_steps / (kernel_ms / 1000.0)
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            with open(tp) as f:
                traffic = json.load(f).get("dram_bytes_per_launch")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_block(world),
            "full_greeks_wall_ms": ms_per_step,
            "kernel_ms": kernel_ms,
            "roofline": {"bound": "mufu", "achieved": achieved, "peak": peak, "unit": UNIT,
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": f"{N_SM} SM x {mufu_clk:.2f} MUFU/clk ({mufu_src}) x "
                                        f"{f_mhz:.0f} MHz (sampled) / {MUFU_PER_PATH_STEP} MUFU "
                                        "per path-step (BASELINE.md)",
                         "fp32_peak": N_SM * 128 * f_mhz * 1e6 / FP32_PER_PATH_STEP},
            "e2e": {"value": path_steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_call": e2e_s * 1000.0},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk,
            "estimates": {q: [g[q].estimate, g[q].path_std_error] for q in g} if g else None,
        }
        if distributed:
            why = parallel.comm_fallback_reason()
            line["dist_backend"] = ("gloo (host-staged)" if gloo else
                                    "nccl (libhmc communicator)" if why is None else
                                    f"nccl (torch process group; libhmc communicator unavailable: {why})")
        if world == 1 and not args.no_cpu:
            line["cpu_baseline"] = cpu_baseline_block()
        if secondary is not None:
            line["secondary"] = secondary
            fp64 = secondary.get("c3_fp64_replay_asian_full_greeks_2^24x252")
            cpu = line.get("cpu_baseline", {}).get("value")
            if fp64 and cpu:   # same-precision comparison with the reference arm
                fp64["vs_cpu_baseline"] = fp64["path_steps_per_s"] / cpu
        if world == 1 and not args.no_e2e and not args.no_cpu:
            line["cpu_baseline_exact"] = cpu_exact_block()
        print(json.dumps(line))
    if distributed:
        parallel.close_comms()
        dist.destroy_process_group()


def _claim_stdout():
    """Keep stdout for the one JSON line: NCCL prints its version banner to
    file descriptor 1 at communicator creation, so under torch.distributed.run
    fd 1 is pointed at stderr and the JSON goes to a private dup of the
    original stdout."""
    if "LOCAL_RANK" not in os.environ:
        return
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    sys.stdout = os.fdopen(saved, "w", buffering=1)


def main():
    _claim_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true", help="skip the public-API e2e leg (profiling)")
    ap.add_argument("--no-secondary", action="store_true", help="skip the secondary BASELINE configs")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
