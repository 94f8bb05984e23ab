"""Per-rank work of the N-GPU headline job, measured on one GPU (this pool
has one GPU per call): rank r of N runs hmc_greeks_chunks on its slice
(parallel.shard) -- exactly the kernel launch it makes in bench.py --gpus N;
T_N = max over ranks of the median CUDA-event time, plus the global
fixed-shape chunk->run reduction every rank runs after the exchange.  The
strong-scaling efficiency of the compute part is T_1 / (N T_N); the NCCL
exchange of ~115 KB is not included (one GPU).  Writes
gpurun_out/slice_scaling.json."""
import ctypes, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
from paper_2309_10477_b200 import _lib, engine, parallel

p, spec, cfg = bench.workload()
L = _lib.lib()
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev)
C = parallel.n_chunks(cfg.n_paths)
full = torch.zeros((1, C, _lib.HMC_NW), dtype=torch.float64, device=dev)
out = torch.empty((1, _lib.HMC_NW), dtype=torch.float64, device=dev)


def timed(fn, reps=7):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream); fn(); e1.record(stream); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


res = {"workload": "bench.py headline job (2^24 x 252 Asian daily fixings, full Greeks)", "rows": []}
reduce_ms = timed(lambda: _lib.check(L.hmc_reduce_chunks(ctypes.c_void_p(full.data_ptr()), 1, C,
                                                         ctypes.c_void_p(out.data_ptr()),
                                                         ctypes.c_void_p(stream.cuda_stream))))
t1 = None
for world in (1, 2, 4, 8):
    per_rank = []
    for rank in range(world):
        sl = parallel.shard(cfg.n_paths, rank, world)
        job = engine.Job(p, spec, cfg, True)
        job.sim.path_lo, job.sim.path_hi = sl.path_lo, sl.path_hi
        work = torch.empty(int(L.hmc_workspace_bytes(ctypes.byref(job.sim))), dtype=torch.uint8, device=dev)
        loc = torch.empty((1, sl.n_chunks, _lib.HMC_NW), dtype=torch.float64, device=dev)
        per_rank.append(timed(lambda: _lib.check(L.hmc_greeks_chunks(
            ctypes.byref(job.model), ctypes.byref(job.product), ctypes.byref(job.sim),
            ctypes.c_void_p(loc.data_ptr()), ctypes.c_void_p(work.data_ptr()),
            ctypes.c_void_p(stream.cuda_stream)))))
        if world == 8 and rank == 0:
            pass
    tn = max(per_rank) + reduce_ms
    t1 = t1 or tn
    row = {"gpus": world, "rank_ms": per_rank, "reduce_ms": reduce_ms, "step_ms_without_exchange": tn,
           "path_steps_per_s": cfg.n_paths * cfg.n_steps / (tn / 1e3), "efficiency": t1 / (world * tn)}
    res["rows"].append(row)
    print(json.dumps(row), flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "slice_scaling.json"), "w") as f:
    json.dump(res, f, indent=1)
