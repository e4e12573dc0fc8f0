"""Exact gradients and the sampler bias/variance diagnostic on the device
 against the reference's own
gradient_full (kernels.cpp:170-198), gradient_poisson_implicit
(kernels.cpp:200-235) and empirical_bias_variance (samplers.cpp:134-168).

Tolerances: fp64 gradients <= 1e-10 relative (summation order differs: L2
atomics vs the reference's serial walk); fp32 <= 1e-4.  bias/variance in
RefStream mode (the reference's own trial draws) <= 1e-9 relative."""
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


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("dims,r,loss", [((9, 7, 5), 4, 0), ((6, 5, 4, 3), 3, 2),
                                         ((11, 13), 5, 1), ((40, 30, 20), 16, 5)])
def test_gradient_full_sparse_matches_reference(ref, dtype, dims, r, loss):
    g = G()
    rs = np.random.default_rng(sum(dims) + r)
    coords, vals = _sparse(rs, dims, 0.1, counts=(loss == 1))
    F = [rs.uniform(0.1, 1, (n, r)) for n in dims]
    if dtype == "f32":
        F = [f.astype(np.float32).astype(np.float64) for f in F]
    delta = 0.7 if loss == 5 else 0.0
    want = ref.sparse(dims, coords, vals).gradient_full(r, F, loss, delta)
    e = g.Engine(dims, r, dtype)
    e.set_sparse(coords, vals)
    e.set_factors(F)
    e.gradient_full(g.LossFunction(loss, delta))
    assert O.rel_error(e.grad_flat(), want) <= (1e-10 if dtype == "f64" else 1e-4)


@pytest.mark.parametrize("storage", ["f64", "u8", "bit"])
def test_gradient_full_dense_matches_reference(ref, storage):
    g = G()
    rs = np.random.default_rng(7)
    dims, r = (8, 9, 10), 5
    x = (rs.random(int(np.prod(dims))) < 0.3).astype(np.float64)
    F = [rs.uniform(0.1, 1, (n, r)) for n in dims]
    want = ref.dense(dims, x).gradient_full(r, F, 2, 0.0)
    e = g.Engine(dims, r, "f64")
    e.set_dense(x, storage)
    e.set_factors(F)
    e.gradient_full(g.LossFunction(2))
    assert O.rel_error(e.grad_flat(), want) <= 1e-10


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("dims,r", [((9, 7, 5), 4), ((6, 5, 4, 3), 3), ((50, 40), 8),
                                    ((30, 20, 25), 32)])
def test_poisson_implicit_matches_reference(ref, dtype, dims, r):
    g = G()
    rs = np.random.default_rng(r * 3 + len(dims))
    coords, vals = _sparse(rs, dims, 0.05, counts=True)
    F = [rs.uniform(0.1, 1, (n, r)) for n in dims]
    if dtype == "f32":
        F = [f.astype(np.float32).astype(np.float64) for f in F]
    rt = ref.sparse(dims, coords, vals)
    want = rt.gradient_poisson_implicit(r, F)
    # the implicit form equals the full-entry walk (kernels.cpp:200 docs)
    assert O.rel_error(want, rt.gradient_full(r, F, 1, 0.0)) <= 1e-10
    e = g.Engine(dims, r, dtype)
    e.set_sparse(coords, vals)
    e.set_factors(F)
    e.gradient_poisson_implicit(g.LossFunction(1))
    assert O.rel_error(e.grad_flat(), want) <= (1e-10 if dtype == "f64" else 1e-4)


def test_exact_gradient_errors_follow_reference():
    g = G()
    e = g.Engine((4, 5, 6), 2, "f64")
    e.set_sparse(np.array([[0, 1, 2]]), np.array([3.0]))
    with pytest.raises(g.InvalidArgument, match="implicit gradient requires the poisson loss"):
        e.gradient_poisson_implicit(g.LossFunction(0))
    big = g.Engine((1000, 1000, 1000), 2, "f64")
    big.set_sparse(np.array([[0, 1, 2]]), np.array([1.0]))
    with pytest.raises(g.InvalidArgument, match="too large for the full-entry walk"):
        big.gradient_full(g.LossFunction(0))
    d = g.Engine((4, 5), 2, "f64")
    d.set_dense(np.ones(20))
    with pytest.raises(g.InvalidArgument, match="sparse"):
        d.gradient_poisson_implicit(g.LossFunction(1))
    with pytest.raises(g.InvalidArgument, match="trials"):
        e.bias_variance(g.SamplerKind.uniform(10), g.LossFunction(0), 1, 3)


@pytest.mark.parametrize("strategy,loss", [(0, 0), (1, 2), (2, 1)])
def test_bias_variance_refstream_equals_reference(orc, ref, strategy, loss):
    g = G()
    rs = np.random.default_rng(90 + strategy)
    dims, r = (9, 7, 5, 4), 3
    coords, vals = _sparse(rs, dims, 0.08, counts=(loss == 1))
    F = [rs.uniform(0.1, 1, (n, r)) for n in dims]
    s, p, q = (120, 0, 0) if strategy == 0 else (0, 50, 70)
    seed, trials = 77 + strategy, 24
    want_b, want_v = ref.sparse(dims, coords, vals).bias_variance(r, F, loss, 0.0, strategy, s, p,
                                                                  q, 1.1, trials, seed)
    e = g.Engine(dims, r, "f64")
    e.set_sparse(coords, vals)
    e.set_factors(F)
    e.set_draw_stream("reference", 0)
    sk = {0: lambda: g.SamplerKind.uniform(s), 1: lambda: g.SamplerKind.stratified(p, q),
          2: lambda: g.SamplerKind.semi_stratified(p, q)}[strategy]()
    b, v = e.bias_variance(sk, g.LossFunction(loss), trials, orc.rng_stream(seed).key)
    assert abs(b - want_b) <= 1e-9 * max(1.0, abs(want_b))
    assert abs(v - want_v) <= 1e-9 * max(1.0, abs(want_v))


def test_bias_variance_philox_is_unbiased_and_shrinks(ref):
    """Philox trials: the stratified estimator is unbiased (squared bias at
    the variance/trials noise floor) and its variance scales ~1/p."""
    g = G()
    rs = np.random.default_rng(5)
    dims, r = (12, 10, 8), 4
    coords, vals = _sparse(rs, dims, 0.1)
    F = [rs.uniform(0.1, 1, (n, r)) for n in dims]
    exact = ref.sparse(dims, coords, vals).gradient_full(r, F, 2, 0.0)
    e = g.Engine(dims, r, "f64")
    e.set_sparse(coords, vals)
    e.set_factors(F)
    b1, v1 = e.bias_variance(g.SamplerKind.stratified(50, 50), g.LossFunction(2), 2000, 11, exact)
    b2, v2 = e.bias_variance(g.SamplerKind.stratified(200, 200), g.LossFunction(2), 2000, 11, exact)
    b0, _ = e.bias_variance(g.SamplerKind.stratified(200, 200), g.LossFunction(2), 2000, 11)
    assert abs(b0 - b2) <= 1e-8 * max(1.0, b2)  # exact=None -> device gradient_full
    assert v2 < v1 * 0.4
    # unbiased: E||mean - exact||^2 = variance / trials
    assert b1 ** 2 < 2.0 * v1 / 2000
    assert b2 ** 2 < 2.0 * v2 / 2000
