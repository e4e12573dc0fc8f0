"""Measurement on ONE GPU (GCPB_DEBUG_LONE_RANK=1): the captured step graph of C5 as rank g of N runs
it -- nonzero-sharded picks compacted on the side stream under the list launch, interleaved table,
peer exchange kernel with every "peer" mapped to the rank's own table (local HBM instead of NVLink,
N x the local traffic; no barriers).  Checks that the multi-rank step captures and replays, and times
it; the numbers of the exchange are not NVLink numbers and the model it leaves is not a valid step."""
import os, sys
os.environ["GCPB_DEBUG_LONE_RANK"] = "1"
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import bench as B
import paper_1906_01687_b200.gcp as G
from paper_1906_01687_b200 import workloads as WL

w = WL.get(os.environ.get("PROBE_CONFIG", "c5"))
e = B.setup_engine(w, 0, lambda m: None)
loss = G.LossFunction.parse(w.loss)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
e.set_stream(stream.cuda_stream)
K = 10
cases = [tuple(int(v) for v in c.split(":")) for c in os.environ.get("PROBE_CASES", "1:0,2:1,4:2,8:3,8:7").split(",")]
for N, g in cases:
    e.set_shard(g, N)
    if N > 1:
        e.peer_open([e.peer_handle()] * N)
    sk = B.sampler_of(w, G, N)
    for it in range(2):
        e.step(sk, loss, 11, it, 1e-3)
    e.run_steps(sk, loss, 11, 2, K, 1e-3)       # captures
    e.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    e.run_steps(sk, loss, 11, 2 + K, K, 1e-3)   # replays
    b.record(stream)
    e.synchronize()
    print(f"N={N} rank {g}: captured step {a.elapsed_time(b)/K:.3f} ms "
          f"({e.run_steps_launches()/K:.0f} kernels per step, path {e.steps_path})", flush=True)
    if N > 1:
        e.adam_reset()
        e.peer_close()
e.close()
