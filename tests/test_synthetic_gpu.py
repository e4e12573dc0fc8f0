"""Synthetic problem generators on the device against
the reference's own gen_gamma_problem / gen_binary_problem
(src/synthetic.cpp:26-146) on the same RngStream seed.

Parity bar: truth factors bit-exact (same draws, same glibc pow/log/sin/cos
on the host); the binary tensor's nonzero set bit-exact (candidate
Bernoullis and noise placements drawn at the same counters, entries
evaluated without FMA contraction); gamma data within 2 ulp (device log1p vs
glibc log1p); the stream's next draw after generation equal (same number of
draws consumed)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

M64 = (1 << 64) - 1
PHI = 0x9e3779b97f4a7c15


def mix64(z):
    z &= M64
    z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & M64
    z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & M64
    return z ^ (z >> 31)


def next_draw(rng):
    return mix64(rng.key + PHI * (rng.counter + 1))


def G():
    import paper_1906_01687_b200.gcp as g
    return g


def _all_indices(dims):
    return np.stack(np.unravel_index(np.arange(int(np.prod(dims))), dims, order="F"), 1)


@pytest.mark.parametrize("dims,r,seed", [((6, 5, 4), 3, 7), ((9, 8, 7, 6), 4, 11),
                                         ((300, 200), 5, 3)])
def test_gamma_problem_matches_reference(ref, dims, r, seed):
    g = G()
    rt, truth, nxt = ref.gen_gamma(dims, r, seed)
    want = rt.dense_values()
    rng = g.RngStream(seed)
    e = g.Engine(dims, r, "f64")
    got_truth = e.gen_gamma_problem(rng, "f64")
    assert np.array_equal(np.concatenate([t.ravel() for t in got_truth]), truth)
    got = e.value_at(_all_indices(dims))
    ulp = np.abs(got - want) / np.spacing(np.abs(want))
    assert ulp.max() <= 2.0
    assert next_draw(rng) == nxt
    # factors landed in the context
    assert np.array_equal(np.concatenate([f.ravel() for f in e.factors()]), truth)


def test_gamma_problem_fp32_storage(ref):
    g = G()
    dims, r = (10, 9, 8), 4
    rt, truth, _ = ref.gen_gamma(dims, r, 5)
    e = g.Engine(dims, r, "f32")
    e.gen_gamma_problem(g.RngStream(5), "f32")
    got = e.value_at(_all_indices(dims))
    assert O.rel_error(got, rt.dense_values().astype(np.float32).astype(np.float64)) <= 1e-7


@pytest.mark.parametrize("dims,r,delta,p_high,p_low,seed", [
    ((12, 10, 8), 3, 0.15, 0.9, 0.0025, 1),
    ((30, 25, 20), 4, 0.2, 0.9, 0.01, 2),
    ((200, 150, 100), 6, 0.1, 0.8, 0.0025, 3),   # ~7.5e3 noise placements
    ((40, 30, 20, 10), 5, 0.3, 0.95, 0.02, 4),   # heavy overlap between columns
    ((7, 9), 2, 0.45, 0.6, 0.3, 5),              # dense-ish: placement collisions
])
def test_binary_problem_matches_reference(ref, dims, r, delta, p_high, p_low, seed):
    g = G()
    rt, truth, nxt = ref.gen_binary(dims, r, delta, p_high, p_low, seed)
    want_c, want_v = rt.export()
    rng = g.RngStream(seed)
    e = g.Engine(dims, r, "f64")
    got_truth = e.gen_binary_problem(g.BinaryProblemSpec(delta, p_high, p_low), rng)
    assert np.array_equal(np.concatenate([t.ravel() for t in got_truth]), truth)
    got_c, got_v = e.get_sparse()
    assert np.array_equal(got_c, want_c)
    assert np.array_equal(got_v, want_v)
    assert next_draw(rng) == nxt


def test_binary_problem_validation_follows_reference():
    g = G()
    e = g.Engine((5, 5), 1, "f64")
    with pytest.raises(g.InvalidArgument, match="rank must be >= 2"):
        e.gen_binary_problem(g.BinaryProblemSpec(), g.RngStream(1))
    e = g.Engine((5, 5), 3, "f64")
    with pytest.raises(g.InvalidArgument, match="delta must be in"):
        e.gen_binary_problem(g.BinaryProblemSpec(delta=0.5), g.RngStream(1))
    with pytest.raises(g.InvalidArgument, match="0 < p_low < p_high < 1"):
        e.gen_binary_problem(g.BinaryProblemSpec(p_low=0.95), g.RngStream(1))


def test_generated_problem_fits_on_device():
    """The generated problem feeds the hot path directly (no host round trip)."""
    g = G()
    e = g.Engine((60, 50, 40), 4, "f32")
    e.gen_binary_problem(g.BinaryProblemSpec(0.15, 0.9, 0.005), g.RngStream(9))
    assert e.nnz > 0
    st = e.stoch_grad(g.SamplerKind.stratified(500, 500), g.LossFunction(2), 3, 0)
    assert st.tested == st.accepted + st.rejected and st.accepted >= 500
    assert np.isfinite(e.grad_flat()).all()
