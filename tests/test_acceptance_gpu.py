"""The reference's acceptance gate (tests/acceptance.cpp), hot-path criteria,
run on the device engine.  Criterion 5 is in test_reference_relations_gpu.py;
criteria 1-3 are covered by the exact-gradient parity tests
(test_exact_gpu.py, test_reference_relations_gpu.py).

4  all three samplers unbiased on the seeded 6x5x4 instance: 2000 trials,
   every coordinate within 3 standard errors, 5 % overall (:166-213) — with
   the reference's own trial draws (RefStream, rng.split(token).split(t));
6  recovery on scaled dense gamma problems: >= 8/10 seeds reach similarity
   0.9 (:252-269) — problem generated on the device, fit on the device;
7  recovery on sparse binary problems: stratified >= 6/10 and >= uniform
   (:271-308) — ditto;
10 the fixed-sample loss estimators are unbiased: 500 draws within 2 % of F
   (:432-461).
The instances are the reference's own (its fixtures, its RngStream seeds);
similarity is the reference's cosine_similarity_score (scoring.cpp), used
as the checker."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def G():
    import paper_1906_01687_b200.gcp as g
    return g


def _fnv1a(label: str) -> int:
    h = 0xcbf29ce484222325
    for c in label.encode():
        h = ((h ^ c) * 0x100000001b3) & ((1 << 64) - 1)
    return h


def _split(flat, dims, r):
    return [m.reshape(n, r) for m, n in zip(np.split(flat, np.cumsum([n * r for n in dims])[:-1]),
                                            dims)]


def test_criterion4_samplers_unbiased(ref):
    g = G()
    rt, model = ref.acceptance_instance(4)
    dims, r = (6, 5, 4), 2
    coords, vals = rt.export()
    e = g.Engine(dims, r, "f64")
    e.set_sparse(coords, vals)
    e.set_factors(_split(model, dims, r))
    loss = g.LossFunction.gaussian()
    e.gradient_full(loss)
    exact = e.grad_flat()
    e.set_draw_stream("reference", 0)
    trials = 2000
    for token in ("uniform", "stratified", "semi-stratified"):
        key = g.RngStream(1004).split(_fnv1a(token)).key
        mean, var = e.gradient_moments(g.SamplerKind.from_token(token, 60), loss, trials, key)
        se = np.sqrt(np.maximum(var, 0.0) / trials)
        assert np.all(np.abs(mean - exact) <= 3.0 * se + 1e-12), token
        assert np.linalg.norm(mean - exact) / np.linalg.norm(exact) <= 0.05, token


def test_criterion6_gamma_recovery(ref):
    g = G()
    from paper_1906_01687_b200.fit import FitConfig, fit_gcp_adam
    dims, r = (20, 15, 10, 5), 2
    recovered = 0
    for seed in range(10):
        e = g.Engine(dims, r, "f64")
        truth = e.gen_gamma_problem(g.RngStream(4000 + seed), "f64")
        cfg = FitConfig(rank=r, sampler=g.SamplerKind.uniform(50), seed=9000 + seed)
        fit = fit_gcp_adam(e, g.LossFunction.gamma(), cfg)
        if ref.similarity(dims, fit.model, r, truth, r) >= 0.9:
            recovered += 1
        e.close()
    assert recovered >= 8, recovered


def test_criterion7_binary_recovery(ref):
    g = G()
    from paper_1906_01687_b200.fit import FitConfig, fit_gcp_adam
    dims, r = (40, 30, 20, 10), 2
    counts = {"stratified": 0, "uniform": 0}
    for seed in range(10):
        e = g.Engine(dims, r, "f64")
        truth = e.gen_binary_problem(g.BinaryProblemSpec(0.15, 0.9, 0.0025),
                                     g.RngStream(5000 + seed))
        for token in ("stratified", "uniform"):
            cfg = FitConfig(rank=r, sampler=g.SamplerKind.from_token(token, 100),
                            max_bad_epochs=3, estimator_samples=200000, seed=7000 + seed)
            fit = fit_gcp_adam(e, g.LossFunction.bernoulli_odds(), cfg)
            if ref.similarity(dims, fit.model, r, truth, r) >= 0.9:
                counts[token] += 1
        e.close()
    assert counts["stratified"] >= 6 and counts["stratified"] >= counts["uniform"], counts


def test_criterion10_estimators_unbiased(ref):
    g = G()
    rt, model = ref.acceptance_instance(10)
    dims, r = (10, 8, 6), 2
    coords, vals = rt.export()
    e = g.Engine(dims, r, "f64")
    e.set_sparse(coords, vals)
    e.set_factors(_split(model, dims, r))
    loss = g.LossFunction.gaussian()
    idx = np.stack(np.unravel_index(np.arange(int(np.prod(dims))), dims, order="F"), 1)
    e.estimator_set(idx, e.value_at(idx), np.ones(len(idx)))  # exhaustive: exact F
    exact = e.estimate(loss)
    for kind in (0, 1):  # EstimatorSamples::Kind uniform, stratified
        total = 0.0
        for rep in range(500):
            e.estimator_draw(kind, 300, 11_000 + 1000 * kind + rep)
            total += e.estimate(loss)
        assert abs(total / 500 - exact) / abs(exact) <= 0.02, kind
