"""Factor tables beyond 2^31 padded elements (64-bit row offsets, the fused
kernel's OFF64 instantiations) and a 2^29 extent; the explicit limits.

dims (2^29 + 3, 3, 5), r = 1 fp32: rows pad to 8 elements, so mode 0 holds
2^32 + 24 elements and every row of modes 1 and 2 sits beyond 2^32 elements
-- a 32-bit offset would wrap.  Mode-0 factors are ones, so the gradient of
modes 1 and 2 is a small closed form of the recorded samples:
G_1[i1] += y * A_2[i2], G_2[i2] += y * A_1[i1] (kernels.cpp:21-37)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def _free_gb():
    import torch
    free, _ = torch.cuda.mem_get_info()
    return free / 2**30


def test_tables_beyond_2_32_elements(monkeypatch):
    import paper_1906_01687_b200.gcp as G
    if _free_gb() < 90:
        pytest.skip("needs ~75 GB of device memory")
    monkeypatch.setenv("GCPB_IL", "0")  # plain layout: offsets are element offsets of A / G
    n0 = 2**29 + 3
    dims, r = (n0, 3, 5), 1
    rs = np.random.default_rng(3)
    e = G.Engine(dims, r, "f32")
    top = n0 - 1 - rs.integers(0, 1000, 400)  # nonzeros in the top rows of mode 0
    coords = np.stack([top, rs.integers(0, 3, 400), rs.integers(0, 5, 400)], 1)
    coords = np.unique(coords, axis=0)
    vals = rs.uniform(0.5, 2.0, len(coords))
    e.set_sparse(coords, vals)
    A1 = rs.uniform(0.5, 1.5, (3, 1))
    A2 = rs.uniform(0.5, 1.5, (5, 1))
    e.set_factor(0, np.ones((n0, 1)))
    e.set_factor(1, A1)
    e.set_factor(2, A2)
    sk = G.SamplerKind.semi_stratified(3000, 3000)
    lf = G.LossFunction.gaussian()
    out = e.draw_samples(sk, lf, 5, 1)
    idx, y = out["idx"], out["y"]
    assert np.all(idx[:3000, 0] >= n0 - 1000)  # the picks: top rows
    assert np.all(out["x"][:3000] == e.value_at(idx[:3000]))
    e.stoch_grad(sk, lf, 5, 1)  # same draws
    A1f, A2f = A1.astype(np.float32).astype(np.float64), A2.astype(np.float32).astype(np.float64)
    g1 = np.zeros(3)
    g2 = np.zeros(5)
    np.add.at(g1, idx[:, 1], y * A2f[idx[:, 2], 0])
    np.add.at(g2, idx[:, 2], y * A1f[idx[:, 1], 0])
    assert O.rel_error(e.grad_mode(1).ravel(), g1) <= 1e-5
    assert O.rel_error(e.grad_mode(2).ravel(), g2) <= 1e-5
    # an iteration (Adam over 2^32+ elements) moves modes 1 and 2 by the step
    e.adam_step(1e-2)
    assert np.all(np.abs(e.factor(1) - A1f) > 0)
    e.close()


def test_extent_limit_is_explicit():
    """Extents >= 2^31 are refused with invalid_argument (per-mode 32-bit
    indices; such a factor matrix alone needs >= 64 GB per buffer)."""
    import paper_1906_01687_b200.gcp as G
    with pytest.raises(G.InvalidArgument, match="extents < 2\\^31"):
        G.Engine((2**31, 3, 5), 1, "f32")


def test_off64_shape_limit_is_explicit():
    """Beyond 2^31 padded elements only d = 3, 4 run (OFF64 instantiations):
    other mode counts are refused up front, not mis-addressed."""
    import paper_1906_01687_b200.gcp as G
    if _free_gb() < 90:
        pytest.skip("needs ~75 GB of device memory")
    e = G.Engine((2**28 + 1, 2), 1, "f32")  # 2^31 + 8 elements, d = 2
    coords = np.array([[0, 0]])
    e.set_sparse(coords, np.ones(1))
    with pytest.raises(G.InvalidArgument, match="2\\^31 padded elements"):
        e.stoch_grad(G.SamplerKind.semi_stratified(10, 10), G.LossFunction.gaussian(), 1, 0)
    e.close()
