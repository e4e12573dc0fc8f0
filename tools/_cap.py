import os, sys
os.environ["GCPB_IL"] = "1"
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import paper_1906_01687_b200.gcp as G

rs = np.random.default_rng(3)
dims, r = (600, 400, 500), 16
coords = np.unique(np.stack([rs.integers(0, n, 40000) for n in dims], 1), axis=0)
vals = 1.0 + rs.poisson(2.0, len(coords)).astype(np.float64)
F = [rs.uniform(0.1, 1.0, (n, r)) for n in dims]
sk, lf = G.SamplerKind.semi_stratified(8 * 6000, 8 * 6000), G.LossFunction.poisson()
for side, shard in (("1", False), ("1", True), ("0", True)):
    os.environ["GCPB_PICK_SIDE"] = side
    e = G.Engine(dims, r, "f32")
    e.set_sparse(coords, vals)
    e.set_factors(F)
    if shard:
        e.set_shard(3, 8)
    s = torch.cuda.Stream()
    e.set_stream(s.cuda_stream)
    e.stoch_grad(sk, lf, 5, 2)          # eager: reserves the pick list, hot rows, ordering buffers
    e.synchronize()
    want = e.grad_flat().copy()
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s, capture_error_mode="relaxed"):
                e.stoch_grad(sk, lf, 5, 2)
    except Exception as ex:
        print(f"PICK_SIDE={side} sharded={shard}: capture failed: {str(ex)[:160]}")
        continue
    g.replay()
    torch.cuda.synchronize()
    got = e.grad_flat()
    err = np.max(np.abs(got - want)) / np.max(np.abs(want))
    print(f"PICK_SIDE={side} sharded={shard}: captured sharded stoch_grad replayed, rel err vs eager {err:.2e}, "
          f"|grad| {np.abs(want).sum():.4g}")
    e.close()
