"""SparseTensor normalisation on the device (tensor.cpp:10-41: sum
duplicates, drop zeros, sort by first-mode-fastest linear key) against the
pinned oracle (or_sparse_normalize) and the reference; and the .tns ->
device path end to end."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def G():
    import paper_1906_01687_b200.gcp as g
    return g


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("dims,n,distinct", [((50, 40, 30), 200_000, 5_000),
                                             ((7,), 1000, 7),
                                             ((300, 200, 100, 50), 300_000, 250_000)])
def test_device_normalisation_matches_oracle(dtype, dims, n, distinct):
    g = G()
    rs = np.random.default_rng(n + len(dims))
    pool = np.stack([rs.integers(0, k, distinct) for k in dims], 1)
    coords = pool[rs.integers(0, distinct, n)]
    vals = rs.integers(-3, 4, n).astype(np.float64)  # integer sums: order-free; many cancel to 0
    t = O.Tensor(dims, coords, vals)
    e = g.Engine(dims, 4, dtype)
    e.set_sparse(coords, vals)
    assert e.nnz == t.nnz
    got_c, got_v = e.get_sparse()
    assert np.array_equal(got_c, t.coords)
    assert np.array_equal(got_v, t.values)


def test_device_normalisation_float_duplicates_match_reference(ref):
    g = G()
    rs = np.random.default_rng(4)
    dims = (20, 30, 40)
    lin = rs.choice(int(np.prod(dims)), 12_000, replace=False)   # distinct keys
    base = np.stack(np.unravel_index(lin, dims, order="F"), 1)
    coords = np.concatenate([base, base[:6_000]])  # exact pairs: a 2-term sum is order-free
    coords = coords[rs.permutation(len(coords))]
    vals = rs.normal(size=len(coords))
    want_c, want_v = ref.sparse(dims, coords, vals).export()
    e = g.Engine(dims, 3, "f64")
    e.set_sparse(coords, vals)
    got_c, got_v = e.get_sparse()
    assert np.array_equal(got_c, want_c) and np.array_equal(got_v, want_v)


def test_first_bad_index_in_input_order_is_reported(ref):
    g = G()
    dims = (10, 10, 10)
    coords = np.zeros((100_000, 3), dtype=np.int64)
    coords[70_000] = (3, 10, 1)   # first offending entry
    coords[90_000] = (11, 0, 0)
    coords[5] = (1, 2, 3)
    with pytest.raises(g.OutOfRange) as ours:
        g.Engine(dims, 2, "f64").set_sparse(coords, np.ones(len(coords)))
    with pytest.raises(O.RefError) as theirs:
        ref.sparse(dims, coords, np.ones(len(coords)))
    assert str(ours.value) == str(theirs.value).split("] ", 1)[1]


def test_tns_file_to_device(ref, tmp_path):
    from paper_1906_01687_b200 import io
    g = G()
    rs = np.random.default_rng(8)
    dims = (40, 30, 20, 10)
    coords = np.stack([rs.integers(0, k, 20_000) for k in dims], 1)
    vals = rs.poisson(2.0, 20_000).astype(np.float64)  # zeros dropped on ingest
    rt = ref.sparse(dims, coords, vals)
    p = tmp_path / "t.tns"
    io.write_tns(io.CooTensor(dims, coords, vals), p)
    e = io.engine_from_file(p, rank=5, dtype="f32")
    want_c, want_v = rt.export()
    got_c, got_v = e.get_sparse()
    assert np.array_equal(got_c, want_c) and np.array_equal(got_v, want_v)
    q = tmp_path / "t.coo"
    io.write_coo(io.CooTensor(dims, coords, vals), q)
    got2 = io.engine_from_file(q, rank=5, dtype="f64").get_sparse()
    assert np.array_equal(got2[0], want_c) and np.array_equal(got2[1], want_v)
