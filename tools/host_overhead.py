"""Per-call host overhead of the C-ABI on a C1-sized problem."""
import os, sys, time
import torch  # before the engine: torch needs its bundled NCCL symbols
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1906_01687_b200.gcp as g
from paper_1906_01687_b200 import _capi

dims, r = (100, 100, 100), 5
rs = np.random.default_rng(0)
e = g.Engine(dims, r, "f64")
e.set_dense(rs.normal(size=10**6), "f64")
F = [rs.normal(size=(n, r)) for n in dims]
e.set_factors(F)
sk, lf = g.SamplerKind.uniform(300), g.LossFunction.gaussian()
flat = np.concatenate([f.ravel() for f in F]); out = np.zeros_like(flat)

def t(name, fn, n=300):
    for _ in range(20): fn()
    e.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    e.synchronize()
    print(f"{name:28s} {(time.perf_counter() - t0) / n * 1e6:8.2f} us")

t("synchronize", lambda: e.synchronize())
t("stoch_grad", lambda: e.stoch_grad(sk, lf, 1, 5, want_stats=False))
t("adam_step", lambda: e.adam_step(1e-3))
t("step", lambda: e.step(sk, lf, 1, 5, 1e-3))
t("step+sync", lambda: (e.step(sk, lf, 1, 5, 1e-3), e.synchronize()))
t("set_factors", lambda: e.set_factors(F))
t("factors()", lambda: e.factors())
t("step_host in/out", lambda: e.step_host(sk, lf, 1, 5, 1e-3, flat, out))
t("step_host no io", lambda: e.step_host(sk, lf, 1, 5, 1e-3, None, None))

# page-locked model buffers: the small-problem zero-copy step_host path
pin_in = torch.empty(flat.size, dtype=torch.float64, pin_memory=True).numpy()
pin_out = torch.empty(flat.size, dtype=torch.float64, pin_memory=True).numpy()
pin_in[:] = flat
t("step_host pinned in/out", lambda: e.step_host(sk, lf, 1, 5, 1e-3, pin_in, pin_out))
t("run_steps(1)", lambda: (e.run_steps(sk, lf, 1, 5, 1, 1e-3), e.synchronize()))
t("torch.cuda.synchronize", lambda: torch.cuda.synchronize())
import paper_1906_01687_b200.gcp as gg  # noqa: E402
t("python arg structs only", lambda: (sk.c(), lf.c(), gg.Engine._adam(1e-3)))
