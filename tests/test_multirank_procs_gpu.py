"""Two processes on one GPU, one engine each, as bench.py --gpus 2 runs them
but with a gloo process group as the host communicator (NCCL refuses two
ranks on one device): nonzero-sharded ranks, the device-planned multi-rank
zero sampler, peer tables mapped across the processes with CUDA IPC, and the
fused reduce-scatter + sharded Adam + all-gather kernel writing into the
other process's table.  No kernel waits on another rank's kernel: the rank
barriers are host-level (gloo all-gather).  The replicas must equal a
single-rank run of the same iterations."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    rs = np.random.default_rng(77)
    dims, r = (50, 40, 30), 8
    lin = np.unique(rs.integers(0, int(np.prod(dims)), 2500))
    coords = np.stack(np.unravel_index(lin, dims, order="F"), 1)
    vals = 1.0 + rs.poisson(2.0, len(lin))
    F = [rs.uniform(0.1, 1.0, (n, r)) for n in dims]
    return dims, r, coords, vals, F


def _samplers(G):
    return [G.SamplerKind.semi_stratified(1500, 2000), G.SamplerKind.stratified(1000, 1500, 1.1)]


def _worker(rank, world, port, il, q):
    sys.path.insert(0, str(ROOT))
    os.environ["GCPB_IL"] = il
    import torch
    import torch.distributed as dist
    import paper_1906_01687_b200.gcp as G
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dims, r, coords, vals, F = _problem()
        e = G.Engine(dims, r, "f64", device=0)
        e.set_sparse(coords, vals)
        e.set_factors(F)

        def allgather(v):
            out = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(out, torch.tensor([v], dtype=torch.int64))
            return [int(t) for t in out]

        def allreduce(a):
            t = torch.from_numpy(a.copy())
            dist.all_reduce(t)
            a[:] = t.numpy()

        e.comm_init_host(rank, world, allgather, allreduce)
        handles = [None] * world
        dist.all_gather_object(handles, e.peer_handle())
        e.peer_open(handles)
        lf = G.LossFunction.poisson()
        it = 0
        for sk in _samplers(G):
            for _ in range(2):
                e.step(sk, lf, 21, it, 1e-2, lower_bound=0.0)
                it += 1
            e.run_steps(sk, lf, 21, it, 2, 1e-2, lower_bound=0.0)  # eager (host communicator)
            it += 2
        q.put((rank, [f.copy() for f in e.factors()]))
        dist.barrier()
        e.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("il", ["1", "0"])
def test_two_processes_peer_step_equals_single_rank(il):
    import torch.multiprocessing as mp
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as O
    os.environ["GCPB_IL"] = il
    import paper_1906_01687_b200.gcp as G
    dims, r, coords, vals, F = _problem()
    single = G.Engine(dims, r, "f64", device=0)
    single.set_sparse(coords, vals)
    single.set_factors(F)
    lf = G.LossFunction.poisson()
    it = 0
    for sk in _samplers(G):
        for _ in range(4):
            single.step(sk, lf, 21, it, 1e-2, lower_bound=0.0)
            it += 1
    want = single.factors()
    single.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, 2, port, il, q)) for k in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(2):
        rank, fac = q.get(timeout=300)
        got[rank] = fac
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank in (0, 1):
        for x, y in zip(got[rank], want):
            assert O.rel_error(x, y) <= 1e-12
