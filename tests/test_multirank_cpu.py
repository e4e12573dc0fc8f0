"""World-size-2 gloo tests of the multi-GPU decomposition, on CPU.

Each rank computes the gradient of its shard of the sample ordinals (the
product's gcpb_shard_range) with the pinned oracle, the shards are summed with
a gloo all-reduce (standing in for the NCCL all-reduce of gcpb_allreduce_grad),
and the result must equal the single-rank gradient.  The stratified merge
(gcpb_stratified_keep) must keep exactly the first q accepted zero candidates
in global candidate order.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "oracle"))
    import oracle as O
    import paper_1906_01687_b200.gcp as G
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = O.oracle()
    rs = np.random.default_rng(5)
    dims, r = (9, 8, 7), 4
    lin = np.nonzero(rs.random(int(np.prod(dims))) < 0.1)[0]
    coords = np.stack(np.unravel_index(lin, dims, order="F"), 1)
    vals = 1.0 + rs.poisson(2.0, len(lin))
    F = [rs.uniform(0.1, 1.0, (n, r)) for n in dims]
    t = O.Tensor(dims, coords, vals)
    p, q, seed, it = 101, 131, 17, 4
    # oracle gradient of the full (single-rank) semi-stratified sample set
    rc, full = orc.draw_gradient_samples(t, r, F, 1, 0.0, 2, 0, p, q, 1.1,
                                         orc.source(1, seed=seed, it=it))
    assert rc == 0
    want = orc.mttkrp(dims, r, F, full["idx"], full["y"])
    # this rank's shard: ordinals [b, e) of the picks and of the q draws
    pb, pe = G.shard_range(p, rank, world)
    qb, qe = G.shard_range(q, rank, world)
    sel = np.r_[pb:pe, p + qb:p + qe]
    part = orc.mttkrp(dims, r, F, full["idx"][sel], full["y"][sel])
    ten = torch.from_numpy(part.copy())
    dist.all_reduce(ten)
    # stratified merge: every rank tests its slice of candidates in order
    cand = rs.integers(0, 2, 50)  # 1 = accepted (non-hit), shared seed -> same on all ranks
    cb, ce = G.shard_range(len(cand), rank, world)
    mine = int(cand[cb:ce].sum())
    counts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(counts, torch.tensor([mine]))
    counts = [int(c) for c in counts]
    need = 11
    off, keep = G.stratified_keep(counts, rank, need)
    acc_idx = [cb + i for i, v in enumerate(cand[cb:ce]) if v][:keep]
    gathered = [None] * world
    dist.all_gather_object(gathered, acc_idx)
    if rank == 0:
        merged = [i for g in gathered for i in g]
        first = [i for i, v in enumerate(cand) if v][:need]
        out["grad_err"] = O.rel_error(ten.numpy(), want)
        out["merge_ok"] = merged == first
    dist.destroy_process_group()


def test_sharded_gradient_and_stratified_merge_gloo():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert out["grad_err"] <= 1e-14
    assert out["merge_ok"]
