"""Time run_steps on a C1-sized problem (small persistent kernel vs graph path)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1906_01687_b200.gcp as g

dims, r = (100, 100, 100), 5
rs = np.random.default_rng(0)
e = g.Engine(dims, r, "f64")
e.set_dense(rs.normal(size=10**6), "f64")
e.set_factors([rs.normal(size=(n, r)) for n in dims])
sk, lf = g.SamplerKind.uniform(300), g.LossFunction.gaussian()
for n in (10, 1000, 1000):
    e.synchronize()
    t0 = time.perf_counter()
    e.run_steps(sk, lf, 1, 0, n, 1e-3)
    e.synchronize()
    dt = time.perf_counter() - t0
    print(f"n={n}: {dt / n * 1e6:.2f} us/step", flush=True)
