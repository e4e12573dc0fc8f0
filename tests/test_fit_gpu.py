"""GPU tests of the device-resident iteration and the native fit driver:
gcpb_step == stoch_grad + adam_step, gcpb_run_steps (CUDA graph) == n x
gcpb_step, fit_gcp_adam's init == the reference's init, its epoch logic
(accept / rollback / decay / stop) and its result against the reference's
own fit_gcp_adam on the same problem."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def G():
    import paper_1906_01687_b200.gcp as g
    return g


def _sparse(rs, dims, density, counts=False):
    lin = np.nonzero(rs.random(int(np.prod(dims))) < density)[0]
    coords = np.stack(np.unravel_index(lin, dims, order="F"), 1)
    vals = 1.0 + rs.poisson(2.0, len(lin)) if counts else np.ones(len(lin))
    return coords, vals


def test_step_equals_stoch_grad_plus_adam():
    g = G()
    rs = np.random.default_rng(1)
    dims, r = (30, 20, 10), 6
    coords, vals = _sparse(rs, dims, 0.05, counts=True)
    F = [rs.uniform(0.1, 1, (n, r)) for n in dims]
    a, b = g.Engine(dims, r, "f64"), g.Engine(dims, r, "f64")
    for e in (a, b):
        e.set_sparse(coords, vals)
        e.set_factors(F)
    sk, lf = g.SamplerKind.semi_stratified(400, 600), g.LossFunction.poisson()
    for it in range(3):
        a.step(sk, lf, 9, it, 1e-2, lower_bound=0.0)
        b.stoch_grad(sk, lf, 9, it)
        b.adam_step(1e-2, lower_bound=0.0)
    for x, y in zip(a.factors(), b.factors()):
        assert O.rel_error(x, y) <= 1e-12
    assert a.iterations == b.iterations == 3


@pytest.mark.parametrize("kind", ["uniform_dense", "semi", "stratified", "uniform_sparse"])
def test_run_steps_graph_equals_stepping(kind):
    g = G()
    rs = np.random.default_rng(2)
    dims, r = (40, 30, 20), 8
    F = [rs.uniform(0.1, 1, (n, r)) for n in dims]
    engines = [g.Engine(dims, r, "f64") for _ in range(2)]
    if kind == "uniform_dense":
        dense = rs.uniform(0, 2, int(np.prod(dims)))
        for e in engines:
            e.set_dense(dense, "f64")
        sk, lf, lb = g.SamplerKind.uniform(3000), g.LossFunction.gaussian(), None
    else:
        coords, vals = _sparse(rs, dims, 0.02)
        for e in engines:
            e.set_sparse(coords, vals)
        lf, lb = g.LossFunction.bernoulli_odds(), 0.0
        sk = {"semi": g.SamplerKind.semi_stratified(800, 1200),
              "stratified": g.SamplerKind.stratified(800, 6000),
              "uniform_sparse": g.SamplerKind.uniform(3000)}[kind]
    for e in engines:
        e.set_factors(F)
    a, b = engines
    a.run_steps(sk, lf, 5, 10, 7, 1e-2, lower_bound=lb)
    a.synchronize()
    for it in range(10, 17):
        b.step(sk, lf, 5, it, 1e-2, lower_bound=lb)
    for x, y in zip(a.factors(), b.factors()):
        assert O.rel_error(x, y) <= 1e-10
    assert a.iterations == b.iterations == 7
    # a second replay of the cached graph continues the stream
    a.run_steps(sk, lf, 5, 17, 7, 1e-2, lower_bound=lb)
    for it in range(17, 24):
        b.step(sk, lf, 5, it, 1e-2, lower_bound=lb)
    for x, y in zip(a.factors(), b.factors()):
        assert O.rel_error(x, y) <= 1e-10


def test_run_steps_graph_recaptured_after_scratch_regrows():
    """A plain step with a larger zero budget regrows the zero-sampler scratch
    (the old buffer is freed); replaying the cached step graph afterwards must
    not touch the freed buffer: the graph key carries the scratch generation,
    so the graph is re-captured and the run equals plain stepping."""
    g = G()
    rs = np.random.default_rng(3)
    dims, r = (40, 30, 20), 8
    coords, vals = _sparse(rs, dims, 0.02)
    F = [rs.uniform(0.1, 1, (n, r)) for n in dims]
    a, b = g.Engine(dims, r, "f64"), g.Engine(dims, r, "f64")
    for e in (a, b):
        e.set_sparse(coords, vals)
        e.set_factors(F)
    lf = g.LossFunction.bernoulli_odds()
    small, big = g.SamplerKind.stratified(500, 2000), g.SamplerKind.stratified(500, 20000)
    a.run_steps(small, lf, 6, 0, 3, 1e-2, lower_bound=0.0)
    a.step(big, lf, 6, 3, 1e-2, lower_bound=0.0)
    a.run_steps(small, lf, 6, 4, 3, 1e-2, lower_bound=0.0)
    for it in range(7):
        b.step(big if it == 3 else small, lf, 6, it, 1e-2, lower_bound=0.0)
    for x, y in zip(a.factors(), b.factors()):
        assert O.rel_error(x, y) <= 1e-10
    assert a.iterations == b.iterations == 7


def _expected_init(orc, seed, dims, r, data_norm):
    """Reference init (kruskal.cpp:33-45, 85-93) via the restated RngStream."""
    import ctypes as C
    root = orc.rng_stream(seed)
    init = orc.split(root, "init")
    F = []
    for n in dims:
        F.append(np.array([orc.lib.or_rng_next_double(C.byref(init)) for _ in range(n * r)])
                 .reshape(n, r))
    gram = np.ones((r, r))
    for f in F:
        gram = gram * (f.T @ f)
    ratio = (data_norm / np.sqrt(gram.sum())) ** (1.0 / len(dims))
    return [f * ratio for f in F]


def test_fit_init_is_reference_init(orc):
    from paper_1906_01687_b200.fit import FitConfig, fit_gcp_adam
    g = G()
    rs = np.random.default_rng(3)
    dims, r = (12, 10, 8), 3
    dense = rs.uniform(0, 1, int(np.prod(dims)))
    e = g.Engine(dims, r, "f64")
    e.set_dense(dense, "f64")
    res = fit_gcp_adam(e, g.LossFunction.gaussian(),
                       FitConfig(rank=r, sampler=g.SamplerKind.uniform(30), max_epochs=0,
                                 estimator_samples=200, seed=11))
    want = _expected_init(orc, 11, dims, r, np.linalg.norm(dense))
    for x, y in zip(res.model, want):
        assert O.rel_error(x, y) <= 1e-13
    assert len(res.trace) == 1 and res.trace[0].epoch == 0 and res.trace[0].accepted


def test_fit_rollback_decay_and_stop():
    """An absurd learning rate makes epochs fail: each failure restores the
    snapshot, multiplies alpha by decay, and the fit stops after
    max_bad_epochs + 1 failures (optimizer.cpp:128-146)."""
    from paper_1906_01687_b200.fit import FitConfig, fit_gcp_adam
    g = G()
    rs = np.random.default_rng(4)
    dims, r = (15, 12, 10), 3
    dense = rs.uniform(0, 1, int(np.prod(dims)))
    e = g.Engine(dims, r, "f64")
    e.set_dense(dense, "f64")
    cfg = FitConfig(rank=r, sampler=g.SamplerKind.uniform(100), learning_rate=50.0,
                    epoch_iters=20, max_bad_epochs=2, decay=0.1, estimator_samples=2000,
                    max_epochs=20, seed=5)
    res = fit_gcp_adam(e, g.LossFunction.gaussian(), cfg)
    fails = [t for t in res.trace if not t.accepted]
    assert len(fails) >= 1
    lrs = [t.learning_rate for t in res.trace[1:]]
    for prev, cur, rec in zip(lrs, lrs[1:], res.trace[1:]):
        assert cur == pytest.approx(prev * (0.1 if not rec.accepted else 1.0))
    if len(fails) == 3:
        assert not res.trace[-1].accepted  # stopped right after the third failure
    accepted = [t.loss_estimate for t in res.trace if t.accepted]
    assert all(b <= a for a, b in zip(accepted, accepted[1:]))  # monotone best
    assert res.final_loss_estimate == min(accepted)


def test_fit_matches_reference_fit(ref):
    """C1-like problem (dense, gaussian, rank-5 CP + noise): our device fit and
    the reference's own fit_gcp_adam (same seed, same init; different draw
    streams) reach the same exact objective within 5%."""
    from paper_1906_01687_b200.fit import FitConfig, fit_gcp_adam
    g = G()
    rs = np.random.default_rng(1001)
    dims, R = (20, 20, 20), 3
    A = [rs.standard_normal((n, R)) for n in dims]
    A = [a / np.linalg.norm(a, axis=0) for a in A]
    M = np.einsum("ir,jr,kr->ijk", *A)
    E = rs.standard_normal(M.shape)
    X = M + 0.1 * (np.linalg.norm(M) / np.linalg.norm(E)) * E
    xflat = X.reshape(-1, order="F")
    common = dict(rank=R, learning_rate=1e-2, epoch_iters=200, estimator_samples=3000,
                  max_epochs=15, seed=7)
    e = g.Engine(dims, R, "f64")
    e.set_dense(xflat, "f64")
    res = fit_gcp_adam(e, g.LossFunction.gaussian(),
                       FitConfig(sampler=g.SamplerKind.uniform(60), **common))
    rt = ref.dense(dims, xflat)
    import ctypes as C
    trace = np.zeros((64, 5))
    nt = C.c_int64()
    Fout = np.zeros(sum(dims) * R)
    fin = C.c_double()
    ref._ck(ref.lib.ref_fit_gcp_adam(
        rt.h, 0, 0.0, R, 0, 60, 0, 0, 1.1, 1e-2, 0.9, 0.999, 1e-8, 200, 1, 0.1, 0, 0.0, 3000, -1,
        15, 7, 1, 64, O._f64(trace), C.byref(nt), O._f64(Fout), C.byref(fin)))
    at = 0
    Fref = []
    for n in dims:
        Fref.append(Fout[at:at + n * R].reshape(n, R))
        at += n * R

    def objective(F):
        Mh = np.einsum("ir,jr,kr->ijk", *F)
        return float(((X - Mh) ** 2).sum())

    ours, theirs = objective(res.model), objective(Fref)
    init = objective(_expected_init(O.oracle(), 7, dims, R, np.linalg.norm(X)))
    assert ours < 0.5 * init and theirs < 0.5 * init
    assert abs(ours - theirs) / theirs <= 0.05


@pytest.mark.parametrize("dims,r,dtype,storage,s", [
    ((100, 100, 100), 5, "f64", "f64", 300),      # C1
    ((20, 15, 10, 8), 6, "f32", "bit", 600),
    ((20, 15, 10, 8), 6, "f32", "bit", 5000),     # over the scatter budget: graph path
    ((50, 40), 3, "f64", "u8", 700),
    ((12, 10, 9, 8, 7), 4, "f32", "f32", 64),     # d = 5
])
def test_small_persistent_kernel_equals_stepping(dims, r, dtype, storage, s):
    """run_steps on a small problem (model in shared memory, s*d*r <= 16384)
    takes the one-launch cluster kernel (gcpb_small.cuh); it must reproduce
    the per-step path (same draws; gradient sums differ only in order)."""
    g = G()
    rs = np.random.default_rng(len(dims) + r)
    F = [rs.uniform(0.1, 1, (n, r)) for n in dims]
    if storage in ("bit", "u8"):
        dense = (rs.random(int(np.prod(dims))) < 0.3).astype(np.float64)
        lf, lb = g.LossFunction.bernoulli_odds(), 0.0
    else:
        dense = rs.normal(size=int(np.prod(dims)))
        lf, lb = g.LossFunction.gaussian(), None
    engines = [g.Engine(dims, r, dtype) for _ in range(2)]
    for e in engines:
        e.set_dense(dense, storage)
        e.set_factors(F)
    a, b = engines
    sk = g.SamplerKind.uniform(s)
    a.run_steps(sk, lf, 9, 0, 40, 1e-3, lower_bound=lb)
    for it in range(40):
        b.step(sk, lf, 9, it, 1e-3, lower_bound=lb)
    tol = 1e-10 if dtype == "f64" else 2e-4
    for x, y in zip(a.factors(), b.factors()):
        assert O.rel_error(x, y) <= tol
    assert a.iterations == b.iterations == 40
    # continues the stream on the next call
    a.run_steps(sk, lf, 9, 40, 10, 1e-3, lower_bound=lb)
    for it in range(40, 50):
        b.step(sk, lf, 9, it, 1e-3, lower_bound=lb)
    for x, y in zip(a.factors(), b.factors()):
        assert O.rel_error(x, y) <= tol


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_step_host_equals_set_step_get(dtype):
    """gcpb_step_host (model in, one iteration, model out) is exactly
    set_factors + step + factors."""
    g = G()
    rs = np.random.default_rng(3)
    dims, r = (30, 20, 10), 4
    coords, vals = _sparse(rs, dims, 0.05)
    F = [rs.uniform(0.1, 1, (n, r)) for n in dims]
    a, b = g.Engine(dims, r, dtype), g.Engine(dims, r, dtype)
    for e in (a, b):
        e.set_sparse(coords, vals)
    sk, lf = g.SamplerKind.semi_stratified(300, 300), g.LossFunction.bernoulli_odds()
    flat = np.concatenate([f.ravel() for f in F])
    out = np.zeros_like(flat)
    for it in range(3):
        a.step_host(sk, lf, 4, it, 1e-2, flat, out, lower_bound=0.0)
        b.set_factors(F if it == 0 else b.factors())
        b.step(sk, lf, 4, it, 1e-2, lower_bound=0.0)
        want = np.concatenate([f.ravel() for f in b.factors()])
        assert O.rel_error(out, want) <= (1e-12 if dtype == "f64" else 1e-6)
        flat = out.copy()
