"""Measurement on ONE GPU: the per-rank sample+eval+MTTKRP time of a C5 step when the engine is rank g of
N (nonzeros sharded in contiguous ranges, every rank drawing the global pick stream of N x p picks and
keeping its range; q unrestricted draws per rank).  The exchange (peer kernel / all-reduce) is not in
it: this is the compute side of the weak-scaling step of DESIGN.md section 7."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import bench as B
import paper_1906_01687_b200.gcp as G
from paper_1906_01687_b200 import workloads as WL

w = WL.get("c5")
e = B.setup_engine(w, 0, lambda m: None)
loss = G.LossFunction.parse(w.loss)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
e.set_stream(stream.cuda_stream)
import os
CASES = ((1, 0), (2, 1), (4, 2), (8, 3), (8, 0), (8, 7))
if os.environ.get("PROBE_CASES"):  # e.g. "8:3,8:7"
    CASES = tuple(tuple(int(v) for v in c.split(":")) for c in os.environ["PROBE_CASES"].split(","))
for N, g in CASES:
    e.set_shard(g, N)
    sk = B.sampler_of(w, G, N)
    for it in range(3):
        e.stoch_grad(sk, loss, 11, it)
    e.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 10
    a.record(stream)
    for it in range(K):
        e.stoch_grad(sk, loss, 11, 10 + it)
    b.record(stream)
    e.synchronize()
    print(f"N={N} rank {g}: stoch_grad {a.elapsed_time(b)/K:.3f} ms per step "
          f"(global picks {sk.nonzero_samples:.3g}, this rank keeps ~1/{N})", flush=True)
e.close()
