"""Multi-rank decomposition on one GPU, through the engine's host-callback
communicator (NCCL refuses two ranks on one device).  R contexts, one per
"rank", run in R host threads; the callbacks exchange accept counts and
gradients through a barrier-synchronised hub.  No kernel ever waits on
another rank's kernel — every exchange is a host-level synchronisation.

Checks, for every sampler: the multi-rank gradient (sharded samples + summed
gradient) equals the single-rank gradient, and for the stratified sampler the
global RejectionStats and the kept zero set equal the single-rank run's
(first q non-hits in candidate order).
"""
import threading

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


class Hub:
    def __init__(self, n):
        self.n = n
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


def _problem(seed):
    rs = np.random.default_rng(seed)
    dims, r = (40, 30, 20, 10), 6
    lin = np.nonzero(rs.random(int(np.prod(dims))) < 0.03)[0]
    coords = np.stack(np.unravel_index(lin, dims, order="F"), 1)
    vals = np.ones(len(lin))
    F = [rs.uniform(0.1, 1.0, (n, r)) for n in dims]
    return dims, r, coords, vals, F


def _run_ranks(nranks, fn):
    out = [None] * nranks
    err = []

    def worker(rank):
        try:
            out[rank] = fn(rank)
        except Exception as ex:  # pragma: no cover - surfaced below
            err.append(ex)

    ts = [threading.Thread(target=worker, args=(k,)) for k in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if err:
        raise err[0]
    return out


@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("strategy", [0, 1, 2])
def test_multirank_gradient_equals_single_rank(nranks, strategy):
    import paper_1906_01687_b200.gcp as G
    dims, r, coords, vals, F = _problem(11 + strategy)
    sk = {0: G.SamplerKind.uniform(5000), 1: G.SamplerKind.stratified(1500, 2500, 1.05),
          2: G.SamplerKind.semi_stratified(1500, 2500)}[strategy]
    lf = G.LossFunction.bernoulli_odds()
    single = G.Engine(dims, r, "f64")
    single.set_sparse(coords, vals)
    single.set_factors(F)
    st1 = single.stoch_grad(sk, lf, 5, 2)
    want = single.grad_flat()
    hub = Hub(nranks)

    def rank_fn(rank):
        e = G.Engine(dims, r, "f64")
        e.set_sparse(coords, vals)
        e.set_factors(F)
        e.comm_init_host(rank, nranks, lambda v: hub.allgather(rank, v),
                         lambda a: hub.allreduce(rank, a))
        st = e.stoch_grad(sk, lf, 5, 2)
        e.allreduce_grad()
        return st, e.grad_flat()

    res = _run_ranks(nranks, rank_fn)
    for st, g in res:
        assert O.rel_error(g, want) <= 1e-12
        if strategy == 1:
            assert (st.tested, st.accepted, st.rejected) == (st1.tested, st1.accepted, st1.rejected)


def test_multirank_steps_match_single_rank():
    """gcpb_step with the host communicator: sharded samples, summed gradient,
    replicated Adam keep the factor replicas identical to a single-rank run."""
    import paper_1906_01687_b200.gcp as G
    dims, r, coords, vals, F = _problem(29)
    sk, lf = G.SamplerKind.stratified(800, 1200, 1.1), G.LossFunction.bernoulli_odds()
    single = G.Engine(dims, r, "f64")
    single.set_sparse(coords, vals)
    single.set_factors(F)
    for it in range(4):
        single.step(sk, lf, 9, it, 1e-2, lower_bound=0.0)
    want = single.factors()
    hub = Hub(2)

    def rank_fn(rank):
        e = G.Engine(dims, r, "f64")
        e.set_sparse(coords, vals)
        e.set_factors(F)
        e.comm_init_host(rank, 2, lambda v: hub.allgather(rank, v),
                         lambda a: hub.allreduce(rank, a))
        for it in range(4):
            e.step(sk, lf, 9, it, 1e-2, lower_bound=0.0)
        return e.factors()

    for got in _run_ranks(2, rank_fn):
        for x, y in zip(got, want):
            assert O.rel_error(x, y) <= 1e-12


def _skewed_problem(seed, dims=(60, 40, 30), nnz=1500, r=8):
    rs = np.random.default_rng(seed)
    cols = [np.minimum((rs.pareto(1.2, nnz * 2) * 2).astype(np.int64), n - 1) for n in dims]
    lin = np.unique(sum(c * int(np.prod(dims[:k])) for k, c in enumerate(cols)))[:nnz]
    coords = np.stack(np.unravel_index(lin, dims, order="F"), 1)
    vals = 1.0 + rs.poisson(2.0, len(lin))
    F = [rs.uniform(0.1, 1.0, (n, r)) for n in dims]
    return dims, r, coords, vals, F


@pytest.mark.parametrize("il", ["0", "1"])
@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("strategy", [0, 1, 2])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_peer_adam_steps_match_single_rank(monkeypatch, il, nranks, strategy, dtype):
    """The peer-memory step: nonzero-sharded ranks (records of a contiguous
    range, the global pick stream compacted per rank), the device-planned
    multi-rank zero sampler, and the fused reduce-scatter + sharded Adam +
    all-gather kernel on peer-mapped tables (one GPU: the ranks' tables are
    peers in one process, rank barriers through the host communicator), on
    the interleaved and the plain layout.  Factor replicas must equal a
    single-rank run, with identical RejectionStats for stratified draws."""
    import paper_1906_01687_b200.gcp as G
    monkeypatch.setenv("GCPB_IL", il)
    monkeypatch.setenv("GCPB_HOT_T", "4")  # hot rows on: folded into the table before the exchange
    dims, r, coords, vals, F = _skewed_problem(40 + strategy)
    if dtype == "f32":
        F = [np.asarray(f, np.float32).astype(np.float64) for f in F]
    sk = {0: G.SamplerKind.uniform(4000), 1: G.SamplerKind.stratified(1500, 2500, 1.05),
          2: G.SamplerKind.semi_stratified(1500, 2500)}[strategy]
    lf = G.LossFunction.poisson()
    single = G.Engine(dims, r, dtype)
    single.set_sparse(coords, vals)
    single.set_factors(F)
    for it in range(3):
        single.step(sk, lf, 9, it, 1e-2, lower_bound=0.0)
    want = single.factors()
    hub = Hub(nranks)
    engines = [None] * nranks

    def make(rank):
        e = G.Engine(dims, r, dtype)
        e.set_sparse(coords, vals)
        e.set_factors(F)
        e.comm_init_host(rank, nranks, lambda v: hub.allgather(rank, v),
                         lambda a: hub.allreduce(rank, a))
        engines[rank] = e
        return e.peer_handle()

    handles = _run_ranks(nranks, make)

    def run(rank):
        e = engines[rank]
        e.peer_open(handles)
        for it in range(3):
            e.step(sk, lf, 9, it, 1e-2, lower_bound=0.0)
        return e.factors()

    tol = 1e-12 if dtype == "f64" else 2e-5
    for got in _run_ranks(nranks, run):
        for x, y in zip(got, want):
            assert O.rel_error(x, y) <= tol


def test_multirank_run_steps_with_host_communicator():
    """run_steps on ranks with the host communicator (not capturable in a
    graph): the iterations run eagerly and equal single-rank stepping."""
    import paper_1906_01687_b200.gcp as G
    dims, r, coords, vals, F = _problem(31)
    sk, lf = G.SamplerKind.stratified(800, 1200, 1.1), G.LossFunction.bernoulli_odds()
    single = G.Engine(dims, r, "f64")
    single.set_sparse(coords, vals)
    single.set_factors(F)
    for it in range(5):
        single.step(sk, lf, 3, it, 1e-2, lower_bound=0.0)
    want = single.factors()
    hub = Hub(2)

    def rank_fn(rank):
        e = G.Engine(dims, r, "f64")
        e.set_sparse(coords, vals)
        e.set_factors(F)
        e.comm_init_host(rank, 2, lambda v: hub.allgather(rank, v),
                         lambda a: hub.allreduce(rank, a))
        e.run_steps(sk, lf, 3, 0, 5, 1e-2, lower_bound=0.0)
        return e.factors()

    for got in _run_ranks(2, rank_fn):
        for x, y in zip(got, want):
            assert O.rel_error(x, y) <= 1e-12


def test_peer_close_returns_to_the_allreduce_path():
    """gcpb_peer_close before any peer step: the ranks all-reduce the gradient
    and run the replicated adam_step (the fallback bench.py takes when a rank
    cannot map a peer), equal to single-rank stepping; after peer steps the
    Adam moments are sharded over the ranks, so leaving the peer path is a
    usage error until adam_reset."""
    import paper_1906_01687_b200.gcp as G
    dims, r, coords, vals, F = _skewed_problem(45)
    sk, lf = G.SamplerKind.semi_stratified(1500, 2500), G.LossFunction.poisson()
    single = G.Engine(dims, r, "f64")
    single.set_sparse(coords, vals)
    single.set_factors(F)
    for it in range(3):
        single.step(sk, lf, 9, it, 1e-2, lower_bound=0.0)
    want = single.factors()
    nranks = 2
    hub = Hub(nranks)
    engines = [None] * nranks

    def make(rank):
        e = G.Engine(dims, r, "f64")
        e.set_sparse(coords, vals)
        e.set_factors(F)
        e.comm_init_host(rank, nranks, lambda v: hub.allgather(rank, v),
                         lambda a: hub.allreduce(rank, a))
        engines[rank] = e
        return e.peer_handle()

    handles = _run_ranks(nranks, make)

    def run(rank):
        e = engines[rank]
        e.peer_open(handles)
        e.peer_close()
        for it in range(3):
            e.step(sk, lf, 9, it, 1e-2, lower_bound=0.0)
        got = e.factors()
        e.peer_open(handles)
        e.step(sk, lf, 9, 3, 1e-2, lower_bound=0.0)
        with pytest.raises(G.LogicError):
            e.peer_close()
        return got

    for got in _run_ranks(nranks, run):
        for x, y in zip(got, want):
            assert O.rel_error(x, y) <= 1e-12


@pytest.mark.parametrize("il", ["0", "1"])
def test_peer_step_host_matches_single_rank(monkeypatch, il):
    """gcpb_step_host on ranks in the peer path (what bench.py's e2e leg runs
    at N > 1): every rank uploads the same host model, the sharded step runs
    with the peer-memory exchange, every rank downloads the same updated
    model -- equal to the single-rank host-model step."""
    import paper_1906_01687_b200.gcp as G
    monkeypatch.setenv("GCPB_IL", il)
    dims, r, coords, vals, F = _skewed_problem(47)
    sk, lf = G.SamplerKind.semi_stratified(1500, 2500), G.LossFunction.poisson()
    flat0 = np.concatenate([f.ravel() for f in F])

    def host_steps(e, n):
        m_in, m_out = flat0.copy(), np.empty_like(flat0)
        for it in range(n):
            e.step_host(sk, lf, 9, it, 1e-2, m_in, m_out, lower_bound=0.0)
            m_in, m_out = m_out, m_in
        return m_in

    single = G.Engine(dims, r, "f64")
    single.set_sparse(coords, vals)
    single.set_factors(F)
    want = host_steps(single, 3)
    nranks = 2
    hub = Hub(nranks)
    engines = [None] * nranks

    def make(rank):
        e = G.Engine(dims, r, "f64")
        e.set_sparse(coords, vals)
        e.set_factors(F)
        e.comm_init_host(rank, nranks, lambda v: hub.allgather(rank, v),
                         lambda a: hub.allreduce(rank, a))
        engines[rank] = e
        return e.peer_handle()

    handles = _run_ranks(nranks, make)

    def run(rank):
        e = engines[rank]
        e.peer_open(handles)
        return host_steps(e, 3)

    for got in _run_ranks(nranks, run):
        assert O.rel_error(got, want) <= 1e-12


@pytest.mark.parametrize("ahead", ["0", "1"])  # the next step's picks compacted under the exchange
@pytest.mark.parametrize("nranks,rank", [(2, 1), (8, 3)])
def test_lone_rank_step_graph_matches_eager_steps(monkeypatch, nranks, rank, ahead):
    """The multi-rank step as gcpb_run_steps captures it (NCCL communicator on
    real ranks): with GCPB_DEBUG_LONE_RANK a sharded rank alone on the GPU skips
    the rank barriers and maps every peer to its own table, so the step graph —
    compaction of the global pick stream on the side stream, ordered list launch
    first, pick launch, hot fold, peer exchange kernel — is captured and
    replayed here, and must leave what the same steps leave when issued one by
    one (the model itself is not a valid multi-rank result)."""
    import paper_1906_01687_b200.gcp as G
    monkeypatch.setenv("GCPB_DEBUG_LONE_RANK", "1")
    monkeypatch.setenv("GCPB_PICK_AHEAD", ahead)
    monkeypatch.setenv("GCPB_IL", "1")
    monkeypatch.setenv("GCPB_HOT_T", "4")
    dims, r, coords, vals, F = _skewed_problem(77)
    F = [np.asarray(f, np.float32).astype(np.float64) for f in F]
    sk, lf = G.SamplerKind.semi_stratified(1500 * nranks, 2500 * nranks), G.LossFunction.poisson()

    launches = []

    def run(graph):
        e = G.Engine(dims, r, "f32")
        e.set_sparse(coords, vals)
        e.set_factors(F)
        e.set_shard(rank, nranks)
        e.peer_open([e.peer_handle()] * nranks)
        if graph:
            e.run_steps(sk, lf, 9, 0, 4, 1e-2, lower_bound=0.0)
            e.synchronize()
            assert e.steps_path == "graph" and e.run_steps_launches() > 0
            launches.append(e.run_steps_launches())
        else:
            for it in range(4):
                e.step(sk, lf, 9, it, 1e-2, lower_bound=0.0)
        out = e.factors()
        e.adam_reset()
        e.peer_close()
        e.close()
        return out

    got, want = run(True), run(False)
    # 8 kernels per step; compacting ahead adds the iteration snapshot to all but the last
    assert launches[0] == (4 * 8 + 3 if ahead == "1" else 4 * 8)
    assert any(np.abs(x - f).max() > 1e-4 for x, f in zip(got, F))  # the steps moved the model
    for x, y in zip(got, want):
        assert O.rel_error(x, y) <= 2e-5
