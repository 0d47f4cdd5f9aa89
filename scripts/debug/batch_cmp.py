import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
from paper_2102_05297_b200.live import TABLE1_METRICS, CudaMeasurementSource, benchmark
for name, kw in (("transpose", dict(width=1024, height=1024)), ("transpose", {}), ("coulomb", {}), ("gemm", {})):
    src = CudaMeasurementSource(benchmark(name, **kw))
    t = src.tuner
    n = len(src.space)
    idx = list(range(0, n, max(1, n // 12)))[:12]
    vs = [src.variant(i) for i in idx]; ls = [src.launch_of(i) for i in idx]
    ms = list(TABLE1_METRICS)
    b1, _ = t.profile_batch(vs, ls, ms)
    b2, _ = t.profile_batch(vs, ls, ms)
    s1 = np.array([t.profile(v, l, ms)[0] for v, l in zip(vs, ls)])
    s2 = np.array([t.profile(v, l, ms)[0] for v, l in zip(vs, ls)])
    for k, m in enumerate(ms):
        if not m.endswith(".sum"): continue
        rel = lambda a, b: float(np.max(np.abs(a[:, k] - b[:, k]) / np.maximum(np.abs(b[:, k]), 1.0)))
        print(name, kw, f"{m:60s} s1~s2 {rel(s1, s2):.3g} b1~b2 {rel(b1, b2):.3g} b1~s1 {rel(b1, s1):.3g}", flush=True)
    src.close()
