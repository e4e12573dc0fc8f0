"""Measurement: wall time per epoch of the device-resident fit (gcpb_fit_gcp_adam) on a BASELINE config
against epoch_iters x the bench's step time -- what the epoch logic (estimate, snapshot, accept /
rollback) adds to the iterations."""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import bench as B
import paper_1906_01687_b200.gcp as G
from paper_1906_01687_b200 import workloads as WL
from paper_1906_01687_b200.fit import FitConfig, fit_gcp_adam

name = os.environ.get("PROBE_CONFIG", "c4")
w = WL.get(name)
e = B.setup_engine(w, 0, lambda m: None)
cfg = FitConfig(rank=w.rank, sampler=B.sampler_of(w, G), learning_rate=1e-3,
                epoch_iters=int(os.environ.get("PROBE_ITERS", "200")), max_epochs=int(os.environ.get("PROBE_EPOCHS", "4")), max_bad_epochs=10,
                estimator_samples=100000, seed=5, keep_factors=True)
loss = G.LossFunction.parse(w.loss)
fit_gcp_adam(e, loss, cfg)  # warm: graphs captured, estimator drawn
torch.cuda.synchronize()
t0 = time.perf_counter()
res = fit_gcp_adam(e, loss, cfg)
torch.cuda.synchronize()
el = time.perf_counter() - t0
ep = len(res.trace) - 1
print(f"{name}: {ep} epochs of {cfg.epoch_iters} iterations in {el*1e3:.1f} ms "
      f"= {el/max(ep,1)*1e3:.2f} ms per epoch, {el/max(ep,1)/cfg.epoch_iters*1e6:.1f} us per iteration; "
      f"trace {[round(t.loss_estimate, 4) for t in res.trace]}")
e.close()
