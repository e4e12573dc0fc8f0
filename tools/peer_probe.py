"""Measurement on ONE GPU: the peer-memory exchange kernel (reduce-scatter + sharded Adam + all-gather)
at C5's table size, R ranks as R contexts in R host threads with their tables mapped into each other
(same process: plain pointers).  Peer loads and stores are local HBM accesses here, so the time is the
kernel's memory-side floor, not an NVLink measurement.  Run under
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:peer_adam
(the kernels of different ranks never wait on one another, so serialisation under ncu is safe)."""
import os, sys, threading
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_1906_01687_b200.gcp as G

R = int(os.environ.get("PROBE_RANKS", "2"))
CFG = os.environ.get("PROBE_CONFIG", "c5tables")
if CFG == "c3":  # the whole C3 problem: the multi-rank stratified sampler's kernels
    from paper_1906_01687_b200 import workloads as WL
    w = WL.get("c3")
    dims, r = w.dims, w.rank
    keys = WL.sparse_keys(w, 1003)
    coords = np.stack(np.unravel_index(keys.astype(np.int64), dims, order="F"), 1)
    vals = np.ones(len(coords))
elif CFG == "c5":  # the whole C5 problem (generated on the device, shared by the ranks)
    import torch
    from paper_1906_01687_b200 import workloads as WL
    import dataclasses
    # a fifth of C5's nonzeros: two ranks' copies of the whole tensor fit beside the generator's
    w = dataclasses.replace(WL.get("c5"), nnz=int(os.environ.get("PROBE_NNZ", "340000000")))
    dims, r = w.dims, w.rank
    c5_keys, c5_vals = WL.c5_device_data(w)
    coords = vals = None
else:  # C5's table size with a token tensor: the exchange kernel
    dims, r = (4_800_000, 1_700_000, 1_800_000), 16
    rs = np.random.default_rng(1)
    nnz = 200_000
    coords = np.unique(np.stack([rs.integers(0, n, nnz) for n in dims], 1), axis=0)
    vals = np.ones(len(coords))


class Hub:
    def __init__(self, n):
        self.barrier = threading.Barrier(n)
        self.slots = [None] * n

    def allgather(self, rank, v):
        self.slots[rank] = v
        self.barrier.wait()
        out = list(self.slots)
        self.barrier.wait()
        return out

    def allreduce(self, rank, arr):
        self.slots[rank] = arr.copy()
        self.barrier.wait()
        total = np.sum(self.slots, axis=0)
        self.barrier.wait()
        arr[:] = total


hub = Hub(R)
engines, handles = [None] * R, [None] * R


def make(rank):
    e = G.Engine(dims, r, "f32")
    if CFG == "c5":
        e.set_sparse_device(c5_keys.data_ptr(), c5_vals.data_ptr(), c5_keys.numel(), "f32")
        e.set_factors([np.full((n, r), 0.05) for n in dims])
    else:
        e.set_sparse(coords, vals)
    if CFG == "c3":
        e.set_factors([np.full((n, r), 0.3) for n in dims])
    e.comm_init_host(rank, R, lambda v: hub.allgather(rank, v), lambda a: hub.allreduce(rank, a))
    engines[rank] = e
    handles[rank] = e.peer_handle()


def run(rank):
    e = engines[rank]
    e.peer_open(handles)
    if CFG == "c3":
        sk, lf = G.SamplerKind.stratified(w.p * R, w.q * R, w.rho), G.LossFunction.bernoulli_odds()
    elif CFG == "c5":
        sk, lf = G.SamplerKind.semi_stratified(w.p * R, w.q * R), G.LossFunction.gaussian()
    else:
        sk, lf = G.SamplerKind.semi_stratified(100_000 * R, 100_000 * R), G.LossFunction.gaussian()
    for it in range(4):
        e.step(sk, lf, 9, it, 1e-3)
    e.synchronize()


for k in range(R):  # one after the other: the tensor normalisation's working memory
    make(k)
if CFG == "c5":
    del c5_keys, c5_vals
    torch.cuda.empty_cache()
ts = [threading.Thread(target=run, args=(k,)) for k in range(R)]
[t.start() for t in ts]
[t.join() for t in ts]
print("peer probe done:", R, "ranks")
