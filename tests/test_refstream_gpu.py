"""RefStream (parity mode): the device samplers reproduce the reference's own
RngStream draws, and the device fit reproduces the reference's own
fit_gcp_adam trajectory (same init, same estimator set, same gradient draws,
same accept/rollback decisions) — SURVEY.md §8c(6) / §8f(1).

Tolerances (fp64 contexts): indices and counts bit-exact; per-sample values
and gradients <= 1e-12 relative; per-epoch loss estimates <= 1e-9 relative
over the whole trajectory (differences come only from fp summation order:
L2 atomics, parallel norms)."""
import ctypes as C

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def G():
    import paper_1906_01687_b200.gcp as g
    return g


def _root_key(orc, seed):
    return orc.rng_stream(seed).key


def _sparse(rs, dims, density, counts=False):
    lin = np.nonzero(rs.random(int(np.prod(dims))) < density)[0]
    coords = np.stack(np.unravel_index(lin, dims, order="F"), 1)
    vals = 1.0 + rs.poisson(2.0, len(lin)) if counts else np.ones(len(lin))
    return coords, vals


@pytest.mark.parametrize("strategy,loss", [(0, 0), (0, 1), (1, 2), (1, 1), (2, 2), (2, 1)])
def test_refstream_samples_equal_reference_draws(orc, ref, strategy, loss):
    g = G()
    rs = np.random.default_rng(40 + strategy * 3 + loss)
    dims, r = (9, 7, 5, 4), 3
    coords, vals = _sparse(rs, dims, 0.08, counts=(loss != 2))
    F = [rs.uniform(0.1, 1, (n, r)) for n in dims]
    s, p, q = (150, 0, 0) if strategy == 0 else (0, 60, 90)
    seed = 1234 + strategy
    rt = ref.sparse(dims, coords, vals)
    want_idx, want_y = rt.draw_seeded(r, F, loss, 0.0, strategy, s, p, q, 1.1, seed)
    e = g.Engine(dims, r, "f64")
    e.set_sparse(coords, vals)
    e.set_factors(F)
    e.set_draw_stream("reference", 0)
    sk = {0: lambda: g.SamplerKind.uniform(s), 1: lambda: g.SamplerKind.stratified(p, q),
          2: lambda: g.SamplerKind.semi_stratified(p, q)}[strategy]()
    out = e.draw_samples(sk, g.LossFunction(loss), _root_key(orc, seed), 0)
    assert np.array_equal(out["idx"], want_idx)
    assert O.rel_error(out["y"], want_y) <= 1e-12
    consumed = s * 4 if strategy == 0 else (p + (out["stats"].tested if strategy == 1 else q) * 4)
    assert e.draw_counter == consumed
    # the gradient of the same draws
    e.set_draw_stream("reference", 0)
    e.stoch_grad(sk, g.LossFunction(loss), _root_key(orc, seed), 0)
    assert O.rel_error(e.grad_flat(), ref.mttkrp(dims, r, F, want_idx, want_y)) <= 1e-12


def _ref_fit(ref, rt, loss, R, strategy, s, p, q, lr, iters, est, epochs, seed, est_kind=-1,
             has_lb=0):
    trace = np.zeros((epochs + 2, 5))
    nt = C.c_int64()
    dims = rt.dims
    Fout = np.zeros(int(np.sum(dims)) * R)
    fin = C.c_double()
    ref._ck(ref.lib.ref_fit_gcp_adam(rt.h, loss, 0.0, R, strategy, s, p, q, 1.1, lr, 0.9, 0.999,
                                     1e-8, iters, 1, 0.1, has_lb, 0.0, est, est_kind, epochs, seed,
                                     1, epochs + 2, O._f64(trace), C.byref(nt), O._f64(Fout),
                                     C.byref(fin)))
    return trace[:nt.value], Fout, fin.value


def test_refstream_fit_reproduces_reference_trajectory_dense(ref):
    from paper_1906_01687_b200.fit import FitConfig, fit_gcp_adam
    g = G()
    rs = np.random.default_rng(1001)
    dims, R = (15, 12, 10), 3
    A = [rs.standard_normal((n, R)) for n in dims]
    X = np.einsum("ir,jr,kr->ijk", *A) + 0.1 * rs.standard_normal(dims)
    xflat = X.reshape(-1, order="F")
    rt = ref.dense(dims, xflat)
    want_trace, want_F, want_fin = _ref_fit(ref, rt, 0, R, 0, 37, 0, 0, 2e-2, 150, 800, 12, 5)
    e = g.Engine(dims, R, "f64")
    e.set_dense(xflat, "f64")
    res = fit_gcp_adam(e, g.LossFunction.gaussian(),
                       FitConfig(rank=R, sampler=g.SamplerKind.uniform(37), learning_rate=2e-2,
                                 epoch_iters=150, estimator_samples=800, max_epochs=12, seed=5,
                                 draw_stream="reference"))
    assert len(res.trace) == len(want_trace)
    for rec, w in zip(res.trace, want_trace):
        assert rec.epoch == int(w[0])
        assert rec.loss_estimate == pytest.approx(w[1], rel=1e-9)
        assert rec.learning_rate == pytest.approx(w[2], rel=1e-15)
        assert rec.accepted == bool(w[4])
    assert res.final_loss_estimate == pytest.approx(want_fin, rel=1e-9)
    assert O.rel_error(np.concatenate([f.reshape(-1) for f in res.model]), want_F) <= 1e-8


@pytest.mark.parametrize("strategy", [1, 2])
def test_refstream_fit_reproduces_reference_trajectory_sparse(ref, strategy):
    from paper_1906_01687_b200.fit import FitConfig, fit_gcp_adam
    g = G()
    rs = np.random.default_rng(77 + strategy)
    dims, R = (14, 12, 10, 8), 3
    coords, vals = _sparse(rs, dims, 0.05)
    rt = ref.sparse(dims, coords, vals)
    p, q = 40, 60
    want_trace, want_F, want_fin = _ref_fit(ref, rt, 2, R, strategy, 0, p, q, 5e-2, 60, 600, 6, 9)
    e = g.Engine(dims, R, "f64")
    e.set_sparse(coords, vals)
    sk = g.SamplerKind.stratified(p, q) if strategy == 1 else g.SamplerKind.semi_stratified(p, q)
    res = fit_gcp_adam(e, g.LossFunction.bernoulli_odds(),
                       FitConfig(rank=R, sampler=sk, learning_rate=5e-2, epoch_iters=60,
                                 estimator_samples=600, max_epochs=6, seed=9,
                                 draw_stream="reference"))
    assert len(res.trace) == len(want_trace)
    for rec, w in zip(res.trace, want_trace):
        assert rec.loss_estimate == pytest.approx(w[1], rel=1e-9)
        assert rec.accepted == bool(w[4])
    assert O.rel_error(np.concatenate([f.reshape(-1) for f in res.model]), want_F) <= 1e-8
