"""Exact-scheme GPU outputs vs the reference's golden vectors
(tests/golden/exact_cases.npz) plus a throughput probe (dev tool)."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from paper_2309_10477_b200 import HestonParams, cuda_backend
from paper_2309_10477_b200.model import BENCH_PARAMS
z = np.load(os.path.join(ROOT, "tests/golden/exact_cases.npz"))
meta = json.loads(bytes(z["__meta__"]).decode())
for name, m in meta.items():
    u = z[f"{name}__uniforms"] if m["has_uniforms"] else None
    t0 = time.time()
    got = cuda_backend.exact_batch(HestonParams(**m["params"]), m["s0"], np.array(m["times"]), np.array(m["flags"]), m["path_lo"], m["path_hi"], int(m["key_run"]), u)
    rel = np.abs(got - z[f"{name}__out"]) / np.abs(z[f"{name}__out"])
    print(name, "max rel %.2e median %.2e" % (rel.max(), np.median(rel)), "%.3fs" % (time.time() - t0))
p = HestonParams(**BENCH_PARAMS)
for n in (2**15, 2**17):
    t0 = time.time()
    out = cuda_backend.exact_batch(p, 100.0, np.array([0.0, 1.0]), np.array([1]), 0, n, 7, None)
    dt = time.time() - t0
    pr = np.exp(-0.03) * np.maximum(out[:, 0] - 100, 0)
    print(n, "paths %.3f s  %.2f us/path" % (dt, dt / n * 1e6), pr.mean(), pr.std() / np.sqrt(n))
