"""Measurement: legs of the C5 host-buffer step (gcpb_step_host): the step alone, the step with the
model copied in, with the model copied out, and both, wall clock per call."""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import bench as B
import paper_1906_01687_b200.gcp as G
from paper_1906_01687_b200 import workloads as WL

w = WL.get("c5")
e = B.setup_engine(w, 0, lambda m: None)
sk = B.sampler_of(w, G)
loss = G.LossFunction.parse(w.loss)
n = sum(k * w.rank for k in w.dims)
pin_in = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
pin_out = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
pin_in[:] = np.concatenate([f.ravel() for f in e.factors()])

def t(fn, reps=8):
    fn(0); e.synchronize()
    t0 = time.perf_counter()
    for i in range(reps):
        fn(1 + i)
    e.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3

step = t(lambda i: (e.step_host(sk, loss, 3, i, 1e-3, None, None), e.synchronize()))
up = t(lambda i: e.step_host(sk, loss, 3, 100 + i, 1e-3, pin_in, None))
down = t(lambda i: e.step_host(sk, loss, 3, 200 + i, 1e-3, None, pin_out))
both = t(lambda i: e.step_host(sk, loss, 3, 300 + i, 1e-3, pin_in, pin_out))
print(f"NARROW={os.environ.get('GCPB_NARROW','1')} TAIL={os.environ.get('GCPB_NARROW_TAIL','15')} "
      f"THREADS={os.environ.get('GCPB_HOST_THREADS','default')}: step {step:.2f} ms, +in {up - step:.2f} ms, "
      f"+out {down - step:.2f} ms, both {both:.2f} ms (sum of legs {step + (up - step) + (down - step):.2f})")
e.close()
