"""Sparse tensors with N >= 2^64 entries: 128-bit linear keys
(include/gcp/shape.hpp:12-14, src/shape.cpp:87-96, include/gcp/tensor.hpp:
44-47) through the device path -- host normalisation with 128-bit keys,
records decoded from them, the 128-bit membership hash + Bloom prefilter
(uniform lookups, stratified rejection), nonzero sharding -- against the
reference itself (oracle/_ref, whose SparseTensor keys are Index128) fed the
device's own Philox draws through its ScriptedRng."""
import threading

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
DIMS = (20000, 10000, 10000, 5000, 5000)  # N = 5e19 > 2^64


def _problem(seed, nnz=3000, r=4):
    rs = np.random.default_rng(seed)
    # a few hot coordinates so picks repeat rows; duplicates summed by normalisation
    coords = np.stack([np.where(rs.random(nnz) < 0.2, rs.integers(0, 7, nnz),
                                rs.integers(0, n, nnz)) for n in DIMS], 1).astype(np.int64)
    coords[-50:] = coords[:50]  # explicit duplicates
    vals = 1.0 + rs.poisson(2.0, nnz)
    F = [rs.uniform(0.1, 1.0, (n, r)) for n in DIMS]
    return coords, vals, F, r


def test_wide_tensor_normalises_like_the_reference(ref):
    import paper_1906_01687_b200.gcp as G
    coords, vals, F, r = _problem(1)
    assert int(np.prod(np.array(DIMS, dtype=object))) > 2**64
    e = G.Engine(DIMS, r, "f64")
    e.set_sparse(coords, vals)
    rt = ref.sparse(DIMS, coords, vals)
    assert e.nnz == rt.nnz
    got_c, got_v = e.get_sparse()
    want_c, want_v = rt.export()
    assert np.array_equal(got_c, want_c)  # ascending 128-bit key order (tensor.cpp:24-40)
    assert np.array_equal(got_v, want_v)
    # value lookups through the 128-bit hash: every stored entry, and misses
    assert np.array_equal(e.value_at(want_c), want_v)
    miss = want_c.copy()
    miss[:, 0] = (miss[:, 0] + 1) % DIMS[0]
    want_miss = np.array([rt.value_at(m) for m in miss])
    assert np.array_equal(e.value_at(miss), want_miss)


@pytest.mark.parametrize("strategy", [0, 1, 2])
@pytest.mark.parametrize("loss", [1, 0])
def test_wide_gradient_matches_reference(orc, ref, strategy, loss):
    import paper_1906_01687_b200.gcp as G
    coords, vals, F, r = _problem(10 + strategy)
    e = G.Engine(DIMS, r, "f64")
    e.set_sparse(coords, vals)
    e.set_factors(F)
    rt = ref.sparse(DIMS, coords, vals)
    s, p, q = (3000, 0, 0) if strategy == 0 else (0, 1200, 1800)
    sk = {0: lambda: G.SamplerKind.uniform(s), 1: lambda: G.SamplerKind.stratified(p, q, 1.1),
          2: lambda: G.SamplerKind.semi_stratified(p, q)}[strategy]()
    seed, it = 41 + strategy, 3
    st = e.stoch_grad(sk, G.LossFunction(loss), seed, it)
    script = O.philox_script(orc, strategy, DIMS, seed, it, s=s, p=p, eta=rt.nnz,
                             n_cand=st.tested, q=q)
    res = rt.draw_scripted(r, F, loss, 0.0, strategy, s, p, q, 1.1, script)
    assert res["consumed"] == len(script)
    want = ref.mttkrp(DIMS, r, F, res["idx"], res["y"])
    assert O.rel_error(e.grad_flat(), want) <= 1e-10
    if strategy == 1:
        assert (st.tested, st.accepted, st.rejected) == res["stats"]
    drawn = e.draw_samples(sk, G.LossFunction(loss), seed, it)
    assert np.array_equal(drawn["idx"], res["idx"])


def test_wide_nonzero_sharded_ranks_sum_to_single_rank():
    import paper_1906_01687_b200.gcp as G
    coords, vals, F, r = _problem(5)
    sk, lf = G.SamplerKind.semi_stratified(1500, 1500), G.LossFunction.poisson()
    single = G.Engine(DIMS, r, "f64")
    single.set_sparse(coords, vals)
    single.set_factors(F)
    single.stoch_grad(sk, lf, 7, 1)
    want = single.grad_flat()
    total = np.zeros_like(want)
    for rank in range(3):
        e = G.Engine(DIMS, r, "f64")
        e.set_sparse(coords, vals)
        e.set_factors(F)
        e.set_shard(rank, 3)  # this rank's records: a contiguous range of the 128-bit order
        e.stoch_grad(sk, lf, 7, 1)
        total += e.grad_flat()
    assert O.rel_error(total, want) <= 1e-12
