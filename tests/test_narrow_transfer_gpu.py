"""GPU test of the narrowed model transfer (include/gcpb.h,
gcpb_last_transfer_bytes): an fp32 engine moves a large page-locked fp64 model
as fp32 — host threads round chunk after chunk under the DMA and widen the
result; a share of the upload's rows crosses as fp64 without a host pass — and the host-buffer step (gcpb_step_host, the reference's loop body
optimizer.cpp:116-119 on a host KruskalModel) must return bit-identical
factors to the fp64 transfer (up to the summation order of the step's fp32
atomics), with half the bytes on the bus."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def G():
    import paper_1906_01687_b200.gcp as g
    return g


def _problem(rs, dims, nnz):
    coords = np.stack([rs.integers(0, n, nnz) for n in dims], 1).astype(np.int64)
    coords = np.unique(coords, axis=0)
    return coords, 1.0 + rs.poisson(2.0, len(coords)).astype(np.float64)


@pytest.mark.parametrize("rank", [16, 18])  # unpadded rows land in the table; 18 -> padded to 20
@pytest.mark.parametrize("threads,tail", [("3", None), (None, "0"), (None, "40")])
def test_narrowed_step_host_is_bit_identical(monkeypatch, rank, threads, tail):
    import torch
    g = G()
    rs = np.random.default_rng(23)
    # 280k rows x rank >= 2^22 elements: narrowed, 9-10 chunks; the padded case has an
    # element count that is not a multiple of 8 (the conversions' scalar tails run)
    dims = (150_000 + (rank == 18), 90_000, 40_000)
    coords, vals = _problem(rs, dims, 5000)
    n = sum(dims) * rank
    assert n >= 1 << 22
    model = rs.uniform(0.05, 1.0, n)  # not fp32-representable: the rounding is exercised
    sk, lf = g.SamplerKind.semi_stratified(4000, 4000), g.LossFunction.poisson()
    want32 = model.astype(np.float32).astype(np.float64)
    outs, moved = [], []
    for narrow in ("0", "1"):
        monkeypatch.setenv("GCPB_NARROW", narrow)
        if threads:
            monkeypatch.setenv("GCPB_HOST_THREADS", threads)
        if tail:
            monkeypatch.setenv("GCPB_NARROW_TAIL", tail)
        e = g.Engine(dims, rank, dtype="f32")
        e.set_sparse(coords, vals)
        pin_in = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
        pin_out = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
        pin_in[:] = model
        # a step of learning rate 0 returns the model as the device holds it:
        # the host's rounding must be the device's, bit for bit, in every chunk
        pin_out[:] = -1.0
        e.step_host(sk, lf, 5, 0, 0.0, pin_in, pin_out, lower_bound=0.0)
        assert np.array_equal(pin_out, want32)
        moved.append(e.last_transfer_bytes())
        e.adam_reset()
        for it in range(2):
            pin_out[:] = -1.0
            e.step_host(sk, lf, 5, it, 1e-2, pin_in, pin_out, lower_bound=0.0)
            pin_in[:] = pin_out
        outs.append(pin_out.copy())
        # the device copy agrees with what was returned
        dev = np.concatenate([f.ravel() for f in e.factors()])
        assert np.array_equal(dev, pin_out)
        e.close()
    # the last rows of the upload (15 % by default) cross as fp64 without a host pass
    rows = sum(dims)
    rows_tail = rows * int(tail if tail else 15) // 100
    mixed = ((rows - rows_tail) * 4 + rows_tail * 8) * rank
    assert moved[0] == (n * 8, n * 8)
    assert moved[1] == (mixed, n * 4)
    # same steps through both transfers (the fp32 atomics' summation order is
    # the only freedom between two runs)
    assert np.max(np.abs(outs[0] - outs[1])) <= 1e-5 * np.max(np.abs(outs[0]))
    assert np.all(outs[1] >= 0.0) and np.array_equal(outs[1], outs[1].astype(np.float32))


def test_small_and_pageable_models_keep_the_fp64_copy(monkeypatch):
    """Below 2^22 elements, or from pageable memory, the model crosses as fp64."""
    import torch
    g = G()
    rs = np.random.default_rng(5)
    dims, rank = (3000, 2000, 1000), 16
    coords, vals = _problem(rs, dims, 2000)
    n = sum(dims) * rank
    sk, lf = g.SamplerKind.semi_stratified(1000, 1000), g.LossFunction.poisson()
    e = g.Engine(dims, rank, dtype="f32")
    e.set_sparse(coords, vals)
    pin_in = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    pin_out = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    pin_in[:] = rs.uniform(0.05, 1.0, n)
    e.step_host(sk, lf, 5, 0, 1e-2, pin_in, pin_out, lower_bound=0.0)
    assert e.last_transfer_bytes() == (n * 8, n * 8)
    e.close()
    big = (150_000, 90_000, 40_000)
    nb = sum(big) * rank
    coords, vals = _problem(rs, big, 2000)
    e = g.Engine(big, rank, dtype="f32")
    e.set_sparse(coords, vals)
    a, b = rs.uniform(0.05, 1.0, nb), np.zeros(nb)  # pageable
    e.step_host(sk, lf, 5, 0, 1e-2, a, b, lower_bound=0.0)
    assert e.last_transfer_bytes() == (nb * 8, nb * 8)
    assert np.array_equal(b, b.astype(np.float32))
    e.close()
