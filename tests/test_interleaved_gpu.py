"""GPU parity of the interleaved factor/gradient table: for
factor tables beyond L2 the fused step gathers factor rows from, and scatters
gradient rows into, one table of [A row | G row] lines, and Adam updates the
factors in that table only (the contiguous factors are refreshed from it when
anything else reads them).  Only the addresses change (and the replica count:
one), so iterations must give the same model as the plain layout, through
every path that reads or writes the factors in between: the estimator,
get_factors, set_factors, snapshots, a standalone stoch_grad + adam_step,
graph replay and the host-buffer step.

GCPB_IL=1 forces the layout on problems the oracle finishes in seconds.
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def G():
    import paper_1906_01687_b200.gcp as g
    return g


def _zipf_coords(rs, dims, nnz, a=1.2):
    keys, out = set(), []
    perms = [rs.permutation(n) for n in dims]
    probs = []
    for n in dims:
        p = 1.0 / np.arange(1, n + 1) ** a
        probs.append(p / p.sum())
    while len(out) < nnz:
        c = tuple(int(perms[k][rs.choice(len(perms[k]), p=probs[k])]) for k in range(len(dims)))
        if c not in keys:
            keys.add(c)
            out.append(c)
    return np.array(out, dtype=np.int64), 1.0 + rs.poisson(2.0, nnz)


def _flat(e):
    return np.concatenate([f.ravel() for f in e.factors()])


def _engine(g, monkeypatch, il, dims, r, dtype, coords, vals, F):
    monkeypatch.setenv("GCPB_IL", "1" if il else "0")
    e = g.Engine(dims, r, dtype=dtype)
    e.set_sparse(coords, vals)
    e.set_factors(F)
    assert e.interleaved[0] == il
    return e


@pytest.mark.parametrize("dims,r,dtype,strategy,hot", [
    ((50, 30, 40, 20), 16, "f32", 2, "4"),    # semi-stratified, hot rows on
    ((50, 30, 40, 20), 20, "f32", 1, "0"),    # stratified, 96-byte rows
    ((80, 12, 70), 5, "f64", 2, "4"),         # d = 3, fp64
    ((60, 40, 50), 16, "f32", 2, "0"),
])
def test_interleaved_steps_match_plain(monkeypatch, dims, r, dtype, strategy, hot):
    monkeypatch.setenv("GCPB_HOT_T", hot)
    g = G()
    rs = np.random.default_rng(sum(dims) + r)
    coords, vals = _zipf_coords(rs, dims, 2500)
    F = [rs.uniform(0.1, 1.0, (n, r)) for n in dims]
    F2 = [rs.uniform(0.1, 1.0, (n, r)) for n in dims]
    sk = (g.SamplerKind.stratified(8000, 8000) if strategy == 1
          else g.SamplerKind.semi_stratified(8000, 8000))
    lf = g.LossFunction.poisson()
    tol = 1e-10 if dtype == "f64" else 2e-5

    def run(il):
        e = _engine(g, monkeypatch, il, dims, r, dtype, coords, vals, F)
        for it in range(3):
            e.step(sk, lf, 7, it, 1e-2, lower_bound=0.0)
        assert e.interleaved[1] == il
        e.estimator_draw(1, 4000, 13)            # reads the factors after interleaved updates
        est = e.estimate(lf)
        snaps = [_flat(e)]
        e.snapshot_save()
        e.run_steps(sk, lf, 7, 3, 4, 1e-2, lower_bound=0.0)        # graph replay
        snaps.append(_flat(e))
        e.snapshot_restore()                                        # A rewritten
        e.step(sk, lf, 7, 7, 1e-2, lower_bound=0.0)
        snaps.append(_flat(e))
        e.set_factors(F2)                                           # A rewritten
        e.step(sk, lf, 7, 8, 1e-2, lower_bound=0.0)
        snaps.append(_flat(e))
        e.stoch_grad(sk, lf, 7, 9)                                  # plain gradient
        e.adam_step(1e-2, lower_bound=0.0)                          # A rewritten
        e.run_steps(sk, lf, 7, 10, 2, 1e-2, lower_bound=0.0)
        snaps.append(_flat(e))
        e.run_steps(sk, lf, 7, 12, 2, 1e-2, lower_bound=0.0)    # replay of the cached graph
        snaps.append(_flat(e))
        e.close()
        return snaps, est

    (plain, est0), (inter, est1) = run(False), run(True)
    assert abs(est1 - est0) <= tol * 10 * abs(est0)
    for k, (x, y) in enumerate(zip(inter, plain)):
        assert O.rel_error(x, y) <= tol, (k, O.rel_error(x, y))


def test_interleaved_step_matches_oracle_adam(orc, monkeypatch):
    """One interleaved step = the oracle gradient on the same draws followed
    by the oracle Adam update (optimizer.cpp:47-66)."""
    g = G()
    rs = np.random.default_rng(11)
    dims, r = (40, 30, 20, 10), 8
    coords, vals = _zipf_coords(rs, dims, 1500)
    F = [rs.uniform(0.1, 1.0, (n, r)) for n in dims]
    e = _engine(g, monkeypatch, True, dims, r, "f64", coords, vals, F)
    sk, lf = g.SamplerKind.semi_stratified(3000, 3000), g.LossFunction.poisson()
    ref = g.Engine(dims, r, dtype="f64")  # plain layout, gradient materialised
    ref.set_sparse(coords, vals)
    ref.set_factors(F)
    ref.stoch_grad(sk, lf, 5, 0)
    t = O.Tensor(dims, coords, vals)
    rc, want = orc.draw_gradient_samples(t, r, F, 1, 0.0, 2, sk.num_samples, sk.nonzero_samples,
                                         sk.zero_samples, sk.oversample,
                                         orc.source(1, seed=5, it=0))
    assert rc == 0
    grad = orc.mttkrp(dims, r, F, want["idx"], want["y"])
    assert O.rel_error(ref.grad_flat(), grad) <= 1e-10
    e.step(sk, lf, 5, 0, 1e-3, lower_bound=0.0)
    assert e.interleaved[1]
    ref.adam_step(1e-3, lower_bound=0.0)
    assert O.rel_error(_flat(e), _flat(ref)) <= 1e-12


def test_interleaved_step_host(monkeypatch):
    """The host-buffer step (model in/out per call) on the interleaved table."""
    g = G()
    rs = np.random.default_rng(3)
    dims, r = (60, 40, 50), 16
    coords, vals = _zipf_coords(rs, dims, 2000)
    F = [rs.uniform(0.1, 1.0, (n, r)) for n in dims]
    sk, lf = g.SamplerKind.semi_stratified(6000, 6000), g.LossFunction.poisson()
    outs = []
    for il in (False, True):
        e = _engine(g, monkeypatch, il, dims, r, "f32", coords, vals, F)
        flat = np.concatenate([f.ravel() for f in F])
        out = np.zeros_like(flat)
        for it in range(3):
            e.step_host(sk, lf, 2, it, 1e-2, flat, out, lower_bound=0.0)
            flat = out.copy()
        assert e.interleaved[1] == il
        outs.append(out)
        e.close()
    assert O.rel_error(outs[1], outs[0]) <= 2e-5


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_small_step_host_zero_copy_matches_stepping(dtype):
    """Small problems: gcpb_step_host on page-locked buffers runs one cluster
    launch that reads and writes the host model directly; it must equal the
    device-resident stepping path (same draws, summation order aside)."""
    import torch
    g = G()
    rs = np.random.default_rng(17)
    dims, r = (30, 25, 20), 5
    dense = rs.normal(size=int(np.prod(dims)))
    F = [rs.normal(size=(n, r)) for n in dims]
    sk, lf = g.SamplerKind.uniform(300), g.LossFunction.gaussian()
    a, b = (g.Engine(dims, r, dtype=dtype) for _ in range(2))
    for e in (a, b):
        e.set_dense(dense, "f64")
        e.set_factors(F)
    n = sum(dims) * r
    pin_in = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    pin_out = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    pin_in[:] = np.concatenate([f.ravel() for f in F])
    for it in range(6):
        a.step_host(sk, lf, 4, 100 + it, 1e-2, pin_in, pin_out)
        pin_in[:] = pin_out
        b.step(sk, lf, 4, 100 + it, 1e-2)
    assert a.steps_path == "small"
    want = np.concatenate([f.ravel() for f in b.factors()])
    tol = 1e-10 if dtype == "f64" else 1e-5
    assert O.rel_error(pin_out, want) <= tol
    # the device copy of the model follows too (a later device-side call sees it)
    assert O.rel_error(np.concatenate([f.ravel() for f in a.factors()]), want) <= tol
    assert a.iterations == b.iterations == 6


def test_interleaved_sharded_steps_match_single_rank(monkeypatch):
    """Sharded steps on the interleaved table (host-callback communicator, two
    contexts on one GPU): the scatter goes to AG, is packed into the
    contiguous gradient for the all-reduce, and Adam updates AG's factor rows;
    the replicas must equal a single-rank run on the plain layout."""
    import threading
    monkeypatch.setenv("GCPB_HOT_T", "4")
    g = G()
    rs = np.random.default_rng(29)
    dims, r = (40, 30, 20, 10), 8
    coords, vals = _zipf_coords(rs, dims, 2000)
    F = [rs.uniform(0.1, 1.0, (n, r)) for n in dims]
    sk, lf = g.SamplerKind.semi_stratified(6000, 6000), g.LossFunction.poisson()
    single = _engine(g, monkeypatch, False, dims, r, "f64", coords, vals, F)
    for it in range(4):
        single.step(sk, lf, 9, it, 1e-2, lower_bound=0.0)
    want = _flat(single)
    monkeypatch.setenv("GCPB_IL", "1")
    n = 2
    barrier, slots = threading.Barrier(n), [None] * n

    def allgather(rank, v):
        slots[rank] = v
        barrier.wait()
        out = list(slots)
        barrier.wait()
        return out

    def allreduce(rank, arr):
        slots[rank] = arr.copy()
        barrier.wait()
        total = np.sum(slots, axis=0)
        barrier.wait()
        arr[:] = total

    out, err = [None] * n, []

    def worker(rank):
        try:
            e = g.Engine(dims, r, "f64")
            e.set_sparse(coords, vals)
            e.set_factors(F)
            e.comm_init_host(rank, n, lambda v: allgather(rank, v), lambda a: allreduce(rank, a))
            for it in range(4):
                e.step(sk, lf, 9, it, 1e-2, lower_bound=0.0)
            out[rank] = (_flat(e), e.interleaved, e.hot_rows[1])
        except Exception as ex:  # pragma: no cover - surfaced below
            err.append(ex)

    ts = [threading.Thread(target=worker, args=(k,)) for k in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if err:
        raise err[0]
    for flat, il, copies in out:
        assert il == (True, True)
        assert copies >= 2
        assert O.rel_error(flat, want) <= 1e-12


@pytest.mark.parametrize("qshift", ["6", "2"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_ordered_segments_match_ordinal_order(monkeypatch, qshift, dtype):
    """Tables beyond L2 walk the semi-stratified unrestricted draws in mode-0
    row order (GCPB_SORTQ, default on with the interleaved table): the same
    draws and weights in another order, so gradient and iterations equal the
    ordinal-order walk up to summation order."""
    monkeypatch.setenv("GCPB_HOT_T", "4")
    g = G()
    rs = np.random.default_rng(5)
    dims, r = (300, 40, 50), 8
    coords, vals = _zipf_coords(rs, dims, 3000)
    F = [rs.uniform(0.1, 1.0, (n, r)) for n in dims]
    sk, lf = g.SamplerKind.semi_stratified(7000, 9000), g.LossFunction.poisson()
    tol = 1e-10 if dtype == "f64" else 2e-5

    def run(sq):
        monkeypatch.setenv("GCPB_SORTQ", sq)
        monkeypatch.setenv("GCPB_QSHIFT", qshift)
        e = _engine(g, monkeypatch, True, dims, r, dtype, coords, vals, F)
        e.stoch_grad(sk, lf, 3, 0)
        grad = e.grad_flat().copy()
        e.adam_step(1e-2, lower_bound=0.0)
        for it in range(1, 4):
            e.step(sk, lf, 3, it, 1e-2, lower_bound=0.0)
        e.run_steps(sk, lf, 3, 4, 3, 1e-2, lower_bound=0.0)
        out = _flat(e)
        e.close()
        return grad, out

    g0, m0 = run("0")
    g1, m1 = run("1")
    assert O.rel_error(g1, g0) <= tol
    assert O.rel_error(m1, m0) <= tol


@pytest.mark.parametrize("strategy", [2, 1])
def test_side_stream_sampling_matches_main_stream(monkeypatch, strategy):
    """The ordering of the unrestricted draws (semi-stratified, interleaved
    table) and the device-planned zero sampler (stratified) run on a side
    stream under the pick segment's launch, and the fused launch is split at
    the join.  Same draws, same lists: iterations and the
    replayed step graph equal the main-stream run, and the split really
    happened (one more fused launch per step in the captured graph)."""
    monkeypatch.setenv("GCPB_HOT_T", "4")
    g = G()
    rs = np.random.default_rng(9)
    dims, r = (300, 40, 50), 8
    coords, vals = _zipf_coords(rs, dims, 3000)
    F = [rs.uniform(0.1, 1.0, (n, r)) for n in dims]
    if strategy == 2:
        sk, lf = g.SamplerKind.semi_stratified(7000, 9000), g.LossFunction.poisson()
    else:
        sk, lf = g.SamplerKind.stratified(7000, 9000), g.LossFunction.poisson()

    def run(side):
        monkeypatch.setenv("GCPB_ORD_SIDE", side)
        e = _engine(g, monkeypatch, True, dims, r, "f64", coords, vals, F)
        for it in range(3):
            e.step(sk, lf, 3, it, 1e-2, lower_bound=0.0)
        e.run_steps(sk, lf, 3, 3, 4, 1e-2, lower_bound=0.0)
        launches = e.run_steps_launches()
        out = _flat(e)
        e.close()
        return out, launches

    m0, l0 = run("0")
    m1, l1 = run("1")
    assert O.rel_error(m1, m0) <= 1e-10
    assert l1 == l0 + 4  # 4 replayed steps, each with the fused launch split in two
