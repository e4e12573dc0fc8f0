"""GPU parity of the hot-row path: reductions into the most
frequent rows of each mode go to privatized L2-resident copies, folded back
after the fused kernel.  Only the summation order changes, so the gradient
must still match the oracle on the same draws (rel_error <= 1e-4 fp32,
<= 1e-10 fp64), through every consumer of the gradient: stoch_grad (copies
folded into the gradient or into replica 0 ahead of Adam's replica fold),
graph-replayed steps, and sharded ranks.

GCPB_HOT_T (target reductions per address) is lowered so that problems the
oracle finishes in seconds already take the hot path; each test asserts that
the last scatter used hot copies.
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-10, "f32": 1e-4}


def G():
    import paper_1906_01687_b200.gcp as g
    return g


def _zipf(rs, n, a, size):
    p = 1.0 / np.arange(1, n + 1) ** a
    return rs.choice(n, size=size, p=p / p.sum())


def _skewed(rs, dims, nnz, a=1.2):
    """Unique coordinates with Zipf(a) per mode (hot rows at random positions)."""
    perms = [rs.permutation(n) for n in dims]
    keys, coords = set(), []
    while len(coords) < nnz:
        c = tuple(int(p[_zipf(rs, len(p), a, 1)[0]]) for p in perms)
        if c not in keys:
            keys.add(c)
            coords.append(c)
    return np.array(coords, dtype=np.int64), 1.0 + rs.poisson(2.0, nnz)


def _as(F, dtype):
    return [np.asarray(f, np.float32).astype(np.float64) if dtype == "f32" else f for f in F]


def _sampler(g, strategy, p, q):
    return g.SamplerKind.stratified(p, q) if strategy == 1 else g.SamplerKind.semi_stratified(p, q)


@pytest.mark.parametrize("dims,r,dtype,strategy", [
    ((60, 40, 50, 30), 16, "f32", 2),
    ((60, 40, 50, 30), 20, "f32", 1),
    ((80, 12, 70), 5, "f64", 2),
    ((80, 12, 70), 16, "f32", 2),
    ((60, 40, 50, 30), 8, "f64", 1),
])
def test_hot_rows_gradient_matches_oracle(orc, monkeypatch, dims, r, dtype, strategy):
    monkeypatch.setenv("GCPB_HOT_T", "4")
    g = G()
    rs = np.random.default_rng(sum(dims) * r + strategy)
    coords, vals = _skewed(rs, dims, 4000)
    F = _as([rs.uniform(0.05, 1.0, (n, r)) for n in dims], dtype)
    e = g.Engine(dims, r, dtype=dtype)
    e.set_sparse(coords, vals)
    e.set_factors(F)
    sk = _sampler(g, strategy, 30000, 30000)
    st = e.stoch_grad(sk, g.LossFunction.poisson(), 41, 2)
    rows, copies = e.hot_rows
    assert rows > 0 and copies >= 2, (rows, copies)
    t = O.Tensor(dims, coords, vals)
    rc, want = orc.draw_gradient_samples(t, r, F, 1, 0.0, strategy, sk.num_samples,
                                         sk.nonzero_samples, sk.zero_samples, sk.oversample,
                                         orc.source(1, seed=41, it=2))
    assert rc == 0
    if strategy == 1:
        assert (st.tested, st.accepted, st.rejected) == want["stats"]
    grad = orc.mttkrp(dims, r, F, want["idx"], want["y"])
    assert O.rel_error(e.grad_flat(), grad) <= TOL[dtype]
    # copies are re-zeroed by the fold: a second call gives the same gradient
    e.stoch_grad(sk, g.LossFunction.poisson(), 41, 2)
    assert O.rel_error(e.grad_flat(), grad) <= TOL[dtype]


@pytest.mark.parametrize("dtype,reps", [("f64", None), ("f32", None), ("f64", "1")])
def test_hot_rows_steps_match_plain_steps(monkeypatch, dtype, reps):
    """Iterations with hot rows (copies folded into replica 0 ahead of Adam's
    replica fold, or straight into the gradient without replicas; and graph
    replay) give the same model as without."""
    if reps:
        monkeypatch.setenv("GCPB_REPLICAS", reps)
    g = G()
    rs = np.random.default_rng(5)
    dims, r = (50, 30, 40, 20), 12
    coords, vals = _skewed(rs, dims, 3000)
    F = _as([rs.uniform(0.1, 1.0, (n, r)) for n in dims], dtype)
    sk, lf = g.SamplerKind.semi_stratified(20000, 20000), g.LossFunction.poisson()

    def run(hot_t, graph):
        monkeypatch.setenv("GCPB_HOT_T", hot_t)
        e = g.Engine(dims, r, dtype=dtype)
        e.set_sparse(coords, vals)
        e.set_factors(F)
        if graph:
            e.run_steps(sk, lf, 9, 0, 4, 1e-2, lower_bound=0.0)
        else:
            for it in range(4):
                e.step(sk, lf, 9, it, 1e-2, lower_bound=0.0)
        used = e.hot_rows[1]
        out = np.concatenate([f.ravel() for f in e.factors()])
        e.close()
        return out, used

    plain, used0 = run("0", False)
    assert used0 == 0
    tol = 1e-10 if dtype == "f64" else 1e-4
    for graph in (False, True):
        hot, used = run("4", graph)
        assert used >= 2
        assert O.rel_error(hot, plain) <= tol


def test_hot_rows_sharded_sum(monkeypatch):
    """Per-rank gradients with hot rows sum to the single-rank gradient."""
    monkeypatch.setenv("GCPB_HOT_T", "4")
    g = G()
    rs = np.random.default_rng(23)
    dims, r = (40, 30, 20), 8
    coords, vals = _skewed(rs, dims, 1500)
    F = [rs.uniform(0.1, 1, (n, r)) for n in dims]
    sk, lf = g.SamplerKind.semi_stratified(20000, 20000), g.LossFunction.poisson()
    full = g.Engine(dims, r, dtype="f64")
    full.set_sparse(coords, vals)
    full.set_factors(F)
    full.stoch_grad(sk, lf, 3, 1)
    assert full.hot_rows[1] >= 2
    want = full.grad_flat()
    total = np.zeros_like(want)
    for rank in range(3):
        e = g.Engine(dims, r, dtype="f64")
        e.set_sparse(coords, vals)
        e.set_factors(F)
        e.set_shard(rank, 3)
        e.stoch_grad(sk, lf, 3, 1)
        total += e.grad_flat()
    assert O.rel_error(total, want) <= 1e-12


def test_hot_rows_follow_tensor_changes(monkeypatch):
    """The selection is rebuilt when the tensor changes: after set_sparse the
    engine's gradient equals a fresh engine's on the new tensor (no stale hot
    slots); GCPB_HOT_T is read once, when the engine is created (0 disables)."""
    g = G()
    rs = np.random.default_rng(3)
    dims, r = (60, 40, 50), 8
    coords, vals = _skewed(rs, dims, 3000)
    F = [rs.uniform(0.1, 1, (n, r)) for n in dims]
    sk, lf = g.SamplerKind.semi_stratified(20000, 20000), g.LossFunction.poisson()
    monkeypatch.setenv("GCPB_HOT_T", "0")
    off = g.Engine(dims, r, dtype="f64")
    monkeypatch.setenv("GCPB_HOT_T", "4")
    e = g.Engine(dims, r, dtype="f64")
    for x in (off, e):
        x.set_sparse(coords, vals)
        x.set_factors(F)
        x.stoch_grad(sk, lf, 1, 1)
    rows0, copies0 = e.hot_rows
    assert rows0 > 0 and copies0 >= 2
    assert off.hot_rows[1] == 0
    assert O.rel_error(e.grad_flat(), off.grad_flat()) <= 1e-12
    # a different tensor (rows hot in the old one are cold now, and back)
    lin = rs.choice(int(np.prod(dims)), 3000, replace=False)
    c2 = np.stack(np.unravel_index(lin[::-1], dims, order="F"), 1)
    c2[:1000, 0] = 7  # a new hot row in mode 0
    c2 = np.unique(c2, axis=0)
    for x in (off, e):
        x.set_sparse(c2, np.ones(len(c2)))
        x.stoch_grad(sk, lf, 1, 2)
    assert e.hot_rows[1] >= 2
    fresh = g.Engine(dims, r, dtype="f64")
    fresh.set_sparse(c2, np.ones(len(c2)))
    fresh.set_factors(F)
    fresh.stoch_grad(sk, lf, 1, 2)
    assert O.rel_error(e.grad_flat(), fresh.grad_flat()) <= 1e-12
    assert O.rel_error(off.grad_flat(), fresh.grad_flat()) <= 1e-12
    for x in (off, e, fresh):
        x.close()