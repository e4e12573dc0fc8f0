"""GPU parity: the sm_100a engine, called through the C-ABI, against the
reference (golden fixtures produced by the reference itself) and the pinned
C oracle, on identical inputs.

Tolerances (BASELINE.json north_star):
  * indices, sampler counts, weights, script consumption: bit-exact;
  * gradient / loss estimate: rel_error <= 1e-10 in fp64, <= 1e-4 in fp32
    (fp32 compared against the fp64 reference evaluated on the same fp32
    factor values upcast exactly).
"""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-10, "f32": 1e-4}
GOLD = json.loads((Path(__file__).parent / "golden" / "reference_vectors.json").read_text())


def G():
    import paper_1906_01687_b200.gcp as g
    return g


def _as_dtype(F, dtype):
    if dtype == "f32":
        return [np.asarray(f, np.float32).astype(np.float64) for f in F]
    return [np.asarray(f, np.float64) for f in F]


def _sampler(c):
    g = G()
    if c["strategy"] == 0:
        return g.SamplerKind.uniform(c["s"])
    if c["strategy"] == 1:
        return g.SamplerKind.stratified(c["p"], c["q"], c["rho"])
    return g.SamplerKind.semi_stratified(c["p"], c["q"])


def _engine_for(c, dtype):
    g = G()
    e = g.Engine(c["dims"], c["r"], dtype=dtype)
    if c.get("tensor_kind", "sparse") == "dense":
        e.set_dense(np.array(c["dense"]), "f64" if dtype == "f64" else "f32")
    else:
        e.set_sparse(np.array(c["coords"], dtype=np.int64).reshape(-1, len(c["dims"])),
                     np.array(c["values"]))
    return e


# --------------------------------------------------------------------------
# Golden: the reference's own outputs
# --------------------------------------------------------------------------
@pytest.mark.parametrize("case", GOLD["samplers"], ids=lambda c: c["name"])
def test_sampler_and_gradient_match_reference_fp64(case):
    g = G()
    e = _engine_for(case, "f64")
    F = [np.array(f) for f in case["factors"]]
    e.set_factors(F)
    loss = g.LossFunction(case["loss"], case["delta"])
    out = e.draw_samples(_sampler(case), loss, case["seed"], case["iter"])
    want_idx = np.array(case["idx"]).reshape(out["idx"].shape)
    assert np.array_equal(out["idx"], want_idx)  # bit-exact indices
    assert O.rel_error(out["y"], case["y"]) <= TOL["f64"]
    if case["strategy"] == 1:
        assert (out["stats"].tested, out["stats"].accepted, out["stats"].rejected) == tuple(case["stats"])
    st = e.stoch_grad(_sampler(case), loss, case["seed"], case["iter"])
    assert O.rel_error(e.grad_flat(), case["grad"]) <= TOL["f64"]
    if case["strategy"] == 1:
        assert (st.tested, st.accepted, st.rejected) == tuple(case["stats"])


@pytest.mark.parametrize("case", GOLD["samplers"], ids=lambda c: c["name"])
def test_sampler_and_gradient_fp32(orc, case):
    g = G()
    e = _engine_for(case, "f32")
    F = _as_dtype(case["factors"], "f32")
    e.set_factors(F)
    loss = g.LossFunction(case["loss"], case["delta"])
    out = e.draw_samples(_sampler(case), loss, case["seed"], case["iter"])
    assert np.array_equal(out["idx"], np.array(case["idx"]).reshape(out["idx"].shape))
    # expected on the upcast fp32 factors, by the pinned oracle (same script)
    t = O.Tensor(case["dims"], dense=np.array(case["dense"], np.float32)) \
        if case.get("tensor_kind") == "dense" else \
        O.Tensor(case["dims"], np.array(case["coords"]).reshape(-1, len(case["dims"])),
                 np.array(case["values"], np.float32))
    rc, want = orc.draw_gradient_samples(t, case["r"], F, case["loss"], case["delta"],
                                         case["strategy"], case["s"], case["p"], case["q"],
                                         case["rho"], orc.source(0, script=case["script"]))
    assert rc == 0
    assert np.array_equal(want["idx"], out["idx"])
    e.stoch_grad(_sampler(case), loss, case["seed"], case["iter"])
    grad = orc.mttkrp(case["dims"], case["r"], F, want["idx"], want["y"])
    assert O.rel_error(e.grad_flat(), grad) <= TOL["f32"]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_mttkrp_matches_reference(orc, dtype):
    g = G()
    for c in GOLD["mttkrp"]:
        e = g.Engine(c["dims"], c["r"], dtype=dtype)
        F = _as_dtype(c["factors"], dtype)
        e.set_factors(F)
        e.mttkrp_samples(np.array(c["idx"]), np.array(c["y"]))
        want = c["grad"] if dtype == "f64" else orc.mttkrp(c["dims"], c["r"], F, np.array(c["idx"]),
                                                            np.array(c["y"]))
        assert O.rel_error(e.grad_flat(), want) <= TOL[dtype]


def test_adam_matches_reference():
    g = G()
    for c in GOLD["adam"]:
        e = g.Engine(c["dims"], c["r"], dtype="f64")
        e.set_factors([np.array(f) for f in c["factors"]])
        for st in c["steps"]:
            gr = np.array(st["grad"])
            at, mats = 0, []
            for nk in c["dims"]:
                mats.append(gr[at:at + nk * c["r"]].reshape(nk, c["r"]))
                at += nk * c["r"]
            e.set_grad(mats)
            e.adam_step(c["lr"], lower_bound=c["lb"])
            A = np.concatenate([f.reshape(-1) for f in e.factors()])
            B = np.concatenate([f.reshape(-1) for f in e.moment(0)])
            Cm = np.concatenate([f.reshape(-1) for f in e.moment(1)])
            assert O.rel_error(A, st["A"]) <= 1e-12
            assert O.rel_error(B, st["B"]) <= 1e-12
            assert O.rel_error(Cm, st["C"]) <= 1e-12
            assert e.iterations == st["iterations"]
            assert np.abs(e.grad_flat()).max() == 0.0  # gradient zeroed by the fused step


def test_estimator_matches_reference():
    g = G()
    for c in GOLD["estimator"]:
        e = g.Engine(c["dims"], c["r"], dtype="f64")
        e.set_sparse(np.array(c["coords"]), np.array(c["values"]))
        e.set_factors([np.array(f) for f in c["factors"]])
        loss = g.LossFunction(c["loss"])
        # device draw from the Philox stream == the reference's draw on that script
        e.estimator_draw(c["kind"], c["count"], c["seed"])
        idx, x, w = e.estimator_get()
        assert np.array_equal(idx, np.array(c["idx"]).reshape(idx.shape))
        assert np.array_equal(x, np.array(c["x"]))
        assert np.array_equal(w, np.array(c["w"]))
        assert e.estimate(loss) == pytest.approx(c["estimate"], rel=1e-12)
        e.estimator_set(np.array(c["idx"]), np.array(c["x"]), np.array(c["w"]))
        assert e.estimate(loss) == pytest.approx(c["estimate"], rel=1e-12)


def test_sparse_normalisation_matches_reference():
    g = G()
    c = GOLD["normalize"]
    e = g.Engine(c["dims"], 2, dtype="f64")
    e.set_sparse(np.array(c["coords"]), np.array(c["values"]))
    coords, vals = e.get_sparse()
    assert np.array_equal(coords, np.array(c["out_coords"]))
    assert np.array_equal(vals, np.array(c["out_values"]))


# --------------------------------------------------------------------------
# Loss derivative on the device, every loss
# --------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("kind,delta", [(0, 0.0), (1, 0.0), (2, 0.0), (3, 0.0), (4, 0.0), (5, 0.6)])
def test_eval_deriv_all_losses(orc, dtype, kind, delta):
    g = G()
    rs = np.random.default_rng(kind * 3 + (dtype == "f32"))
    dims, r = (7, 6, 5), 4
    F = _as_dtype([rs.uniform(0.05, 1.0, (n, r)) for n in dims], dtype)
    e = g.Engine(dims, r, dtype=dtype)
    e.set_factors(F)
    n = 500
    idx = np.stack([rs.integers(0, k, n) for k in dims], 1)
    x = rs.integers(0, 2, n).astype(float) if kind == 2 else rs.uniform(0, 3, n)
    if dtype == "f32":
        x = x.astype(np.float32).astype(np.float64)
    w = rs.uniform(0.5, 3.0, n)
    flags = rs.integers(0, 2, n).astype(np.int32)
    m, y = e.eval_deriv(idx, x, w, g.LossFunction(kind, delta), flags)
    m_want = orc.entries(dims, r, F, idx)
    y_want = np.array([w[i] * (orc.lib.or_loss_deriv(kind, delta, x[i], m_want[i]) -
                               (orc.lib.or_loss_deriv(kind, delta, 0.0, m_want[i]) if flags[i] else 0.0))
                       for i in range(n)])
    assert O.rel_error(m, m_want) <= (1e-14 if dtype == "f64" else 1e-6)
    assert O.rel_error(y, y_want) <= TOL[dtype]


# --------------------------------------------------------------------------
# Random parity at moderate sizes (oracle finishes in seconds)
# --------------------------------------------------------------------------
def _zipf(rs, n, a, size):
    p = 1.0 / np.arange(1, n + 1) ** a
    return rs.choice(n, size=size, p=p / p.sum())


def _sparse_problem(rs, dims, nnz, a=1.1, values="binary"):
    keys = set()
    coords = []
    while len(coords) < nnz:
        c = tuple(int(_zipf(rs, n, a, 1)[0]) if n > 50 else int(rs.integers(0, n)) for n in dims)
        if c not in keys:
            keys.add(c)
            coords.append(c)
    coords = np.array(coords, dtype=np.int64)
    if values == "binary":
        vals = np.ones(nnz)
    else:
        vals = 1.0 + rs.poisson(2.0, nnz)
    return coords, vals


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("strategy,loss,r", [(1, 2, 32), (2, 1, 20), (0, 0, 16), (2, 2, 8),
                                             (1, 1, 24), (0, 2, 18)])
def test_random_sparse_parity(orc, dtype, strategy, loss, r):
    g = G()
    rs = np.random.default_rng(strategy * 10 + loss + r)
    dims = (60, 40, 50, 30)
    coords, vals = _sparse_problem(rs, dims, 3000, values="binary" if loss == 2 else "count")
    F = _as_dtype([rs.uniform(0.05, 1.0, (n, r)) for n in dims], dtype)
    e = g.Engine(dims, r, dtype=dtype)
    e.set_sparse(coords, vals)
    e.set_factors(F)
    sk = {0: g.SamplerKind.uniform(4000), 1: g.SamplerKind.stratified(2000, 2500),
          2: g.SamplerKind.semi_stratified(2000, 2500)}[strategy]
    lf = g.LossFunction(loss)
    st = e.stoch_grad(sk, lf, 77, 12)
    t = O.Tensor(dims, coords, vals)
    src = orc.source(1, seed=77, it=12)
    rc, want = orc.draw_gradient_samples(t, r, F, loss, 0.0, strategy, sk.num_samples,
                                         sk.nonzero_samples, sk.zero_samples, sk.oversample, src)
    assert rc == 0
    if strategy == 1:
        assert (st.tested, st.accepted, st.rejected) == want["stats"]
    grad = orc.mttkrp(dims, r, F, want["idx"], want["y"])
    assert O.rel_error(e.grad_flat(), grad) <= TOL[dtype]
    drawn = e.draw_samples(sk, lf, 77, 12)
    assert np.array_equal(drawn["idx"], want["idx"])
    assert np.array_equal(drawn["w"], want["w"])
    assert np.array_equal(drawn["flag"], want["flag"])


@pytest.mark.parametrize("dims,r,dtype", [((7,), 3, "f64"), ((9, 8), 5, "f32"),
                                          ((5, 4, 3, 4, 3), 6, "f32"), ((3,) * 9, 4, "f64"),
                                          ((11, 9, 7), 130, "f32"), ((11, 9, 7), 40, "f64")])
def test_shapes_and_ranks(orc, dims, r, dtype):
    """d = 1..9 (all mode-count instantiations), r from 3 to 130 (all lane
    geometries incl. multi-chunk lanes).  Extents of 2^29 and tables beyond
    2^32 elements: tests/test_large_tables_gpu.py."""
    g = G()
    rs = np.random.default_rng(len(dims) * 100 + r)
    F = _as_dtype([rs.uniform(-1, 1, (n, r)) for n in dims], dtype)
    total = int(np.prod(dims))
    dense = rs.uniform(-1, 1, total)
    e = g.Engine(dims, r, dtype=dtype)
    e.set_dense(dense, dtype)
    e.set_factors(F)
    sk = g.SamplerKind.uniform(1500)
    e.stoch_grad(sk, g.LossFunction.gaussian(), 5, 1)
    t = O.Tensor(dims, dense=dense.astype(np.float32) if dtype == "f32" else dense)
    rc, want = orc.draw_gradient_samples(t, r, F, 0, 0.0, 0, 1500, 0, 0, 1.1,
                                         orc.source(1, seed=5, it=1))
    assert rc == 0
    grad = orc.mttkrp(dims, r, F, want["idx"], want["y"])
    assert O.rel_error(e.grad_flat(), grad) <= TOL[dtype]


# --------------------------------------------------------------------------
# Edge cases the reference tests
# --------------------------------------------------------------------------
def test_empty_nonzero_stratum_forfeits_budget(orc):
    """test_samplers.cpp:236-261: eta = 0 -> all p + q samples are zeros."""
    g = G()
    dims, r = (2, 3), 2
    rs = np.random.default_rng(59)
    F = [rs.uniform(0.1, 1.0, (n, r)) for n in dims]
    for sk in (g.SamplerKind.stratified(2, 3), g.SamplerKind.semi_stratified(2, 3)):
        e = g.Engine(dims, r, dtype="f64")
        e.set_sparse(np.zeros((0, 2), np.int64), np.zeros(0))
        e.set_factors(F)
        out = e.draw_samples(sk, g.LossFunction.gaussian(), 3, 0)
        assert len(out["y"]) == 5
        m = orc.entries(dims, r, F, out["idx"])
        np.testing.assert_allclose(out["y"], (6.0 / 5.0) * 2.0 * m, rtol=1e-12)


def test_duplicate_samples_accumulate():
    """test_kernels.cpp:102-123."""
    g = G()
    dims, r = (3, 4, 5), 2
    rs = np.random.default_rng(23)
    F = [rs.uniform(0.5, 1.5, (n, r)) for n in dims]
    e = g.Engine(dims, r, dtype="f64")
    e.set_factors(F)
    idx = np.array([[1, 2, 4]])
    e.mttkrp_samples(idx, np.array([3.0]))
    g1 = e.grad()
    np.testing.assert_allclose(g1[0][1], 3.0 * F[1][2] * F[2][4], rtol=1e-14)
    assert np.abs(g1[0][0]).max() == 0 and np.abs(g1[0][2]).max() == 0
    e.mttkrp_samples(np.repeat(idx, 2, 0), np.array([3.0, 3.0]))
    np.testing.assert_allclose(e.grad_flat(), 2.0 * np.concatenate([m.reshape(-1) for m in g1]),
                               rtol=1e-14)
    e.mttkrp_samples(np.zeros((0, 3), np.int64), np.zeros(0))
    assert np.abs(e.grad_flat()).max() == 0.0  # empty sample set -> zero gradient


def test_perfect_gaussian_fit_gives_zero_gradient():
    """test_kernels.cpp:192-199 with a uniform pass over every entry."""
    g = G()
    dims, r = (4, 3, 2), 2
    rs = np.random.default_rng(41)
    F = [rs.uniform(0.1, 1.0, (n, r)) for n in dims]
    full = np.einsum("ir,jr,kr->ijk", *F).reshape(-1, order="F")
    e = g.Engine(dims, r, dtype="f64")
    e.set_dense(full, "f64")
    e.set_factors(F)
    e.stoch_grad(g.SamplerKind.uniform(500), g.LossFunction.gaussian(), 1, 0)
    assert np.abs(e.grad_flat()).max() <= 1e-12


def test_errors_follow_reference_exceptions():
    g = G()
    e = g.Engine((2, 2), 1, dtype="f64")
    e.set_dense(np.zeros(4), "f64")
    e.set_factors([np.ones((2, 1)), np.ones((2, 1))])
    with pytest.raises(g.InvalidArgument):  # samplers.hpp:232-240
        e.stoch_grad(g.SamplerKind.stratified(1, 1), g.LossFunction.gaussian(), 1, 0)
    with pytest.raises(g.InvalidArgument):
        e.stoch_grad(g.SamplerKind.semi_stratified(1, 1), g.LossFunction.gaussian(), 1, 0)
    s = g.Engine((2, 2), 1, dtype="f64")
    s.set_sparse(np.array([[0, 0], [1, 0], [0, 1]]), np.ones(3))
    s.set_factors([np.ones((2, 1)), np.ones((2, 1))])
    with pytest.raises(g.InvalidArgument):  # zeta < q (samplers.hpp:108-111)
        s.stoch_grad(g.SamplerKind.stratified(0, 2), g.LossFunction.gaussian(), 1, 0)
    out = s.draw_samples(g.SamplerKind.stratified(0, 1, 1.5), g.LossFunction.gaussian(), 29, 0)
    assert out["idx"].tolist() == [[1, 1]]  # a lone zero is always found
    with pytest.raises(g.OutOfRange):  # check_index (shape.cpp:73-85)
        s.set_sparse(np.array([[0, 2]]), np.ones(1))
    c = g.Engine((2, 2), 1, dtype="f32")
    c.set_sparse(np.array([[0, 0]]), np.array([3.0]))
    with pytest.raises(g.DomainError):  # loss.cpp:55-60
        c.stoch_grad(g.SamplerKind.semi_stratified(1, 1), g.LossFunction.bernoulli_odds(), 1, 0)
    with pytest.raises(g.DomainError):
        c.eval_deriv(np.array([[0, 0]]), np.array([-1.0]), np.array([1.0]), g.LossFunction.poisson())


def test_snapshot_rollback_is_exact():
    g = G()
    rs = np.random.default_rng(3)
    dims, r = (20, 15, 10), 4
    e = g.Engine(dims, r, dtype="f32")
    e.set_dense(rs.uniform(0, 1, int(np.prod(dims))), "f32")
    e.set_factors([rs.uniform(0, 1, (n, r)) for n in dims])
    e.snapshot_save()
    A0 = e.factors()
    t0 = e.iterations
    for it in range(3):
        e.stoch_grad(g.SamplerKind.uniform(300), g.LossFunction.gaussian(), 9, it)
        e.adam_step(1e-2)
    assert e.iterations == t0 + 3
    e.snapshot_restore()
    assert e.iterations == t0
    for a, b in zip(A0, e.factors()):
        assert np.array_equal(a, b)


def test_stratified_small_q_needs_several_batches(orc):
    """Tiny q on a dense-ish tensor: the device batch planner and the host
    continuation must reproduce the reference's batch sequence exactly."""
    g = G()
    rs = np.random.default_rng(8)
    dims, r = (5, 4, 3), 3
    lin = np.nonzero(rs.random(60) < 0.7)[0]
    coords = np.stack(np.unravel_index(lin, dims, order="F"), 1)
    F = [rs.uniform(0.1, 1.0, (n, r)) for n in dims]
    t = O.Tensor(dims, coords, np.ones(len(lin)))
    for seed in range(20):
        e = g.Engine(dims, r, dtype="f64")
        e.set_sparse(coords, np.ones(len(lin)))
        e.set_factors(F)
        sk = g.SamplerKind.stratified(3, 4, 1.05)
        out = e.draw_samples(sk, g.LossFunction.bernoulli_odds(), seed, 2)
        rc, want = orc.draw_gradient_samples(t, r, F, 2, 0.0, 1, 0, 3, 4, 1.05,
                                             orc.source(1, seed=seed, it=2))
        assert rc == 0
        assert np.array_equal(out["idx"], want["idx"])
        st = out["stats"]
        assert (st.tested, st.accepted, st.rejected) == want["stats"]


def test_stratified_graph_batches_match_stepping():
    """Graph-replayed steps plan rejection batches 2 and 3 on the device (the
    previous batch's last scatter block) on a reduced grid: on a dense-ish
    tensor where the first batch often falls short they must give the same
    iterations as host-checked stepping; a problem three batches cannot
    satisfy is reported at the next synchronisation."""
    g = G()
    rs = np.random.default_rng(8)
    dims, r = (5, 4, 3), 3
    lin = np.nonzero(rs.random(60) < 0.7)[0]
    coords = np.stack(np.unravel_index(lin, dims, order="F"), 1)
    F = [rs.uniform(0.1, 1.0, (n, r)) for n in dims]
    sk, lf = g.SamplerKind.stratified(3, 4, 1.05), g.LossFunction.bernoulli_odds()
    ok = 0
    for seed in range(12):
        a, b = (g.Engine(dims, r, dtype="f64") for _ in range(2))
        for e in (a, b):
            e.set_sparse(coords, np.ones(len(lin)))
            e.set_factors(F)
        try:
            a.run_steps(sk, lf, seed, 0, 3, 1e-2, lower_bound=0.0)
            a.synchronize()
        except RuntimeError as ex:  # more than three batches needed by some step
            assert "fewer than q zeros" in str(ex)
            continue
        for it in range(3):
            b.step(sk, lf, seed, it, 1e-2, lower_bound=0.0)
        for x, y in zip(a.factors(), b.factors()):
            assert O.rel_error(x, y) <= 1e-12
        ok += 1
    assert ok >= 6


def test_seed_and_iteration_determinism():
    g = G()
    rs = np.random.default_rng(99)
    dims, r = (30, 20, 10), 8
    e = g.Engine(dims, r, dtype="f64")
    e.set_dense(rs.uniform(0, 1, int(np.prod(dims))), "f64")
    e.set_factors([rs.uniform(0, 1, (n, r)) for n in dims])
    sk, lf = g.SamplerKind.uniform(2000), g.LossFunction.gaussian()
    a = e.draw_samples(sk, lf, 5, 3)["idx"]
    b = e.draw_samples(sk, lf, 5, 3)["idx"]
    c = e.draw_samples(sk, lf, 5, 4)["idx"]
    d = e.draw_samples(sk, lf, 6, 3)["idx"]
    assert np.array_equal(a, b)
    assert not np.array_equal(a, c) and not np.array_equal(a, d)


def test_sharded_samples_sum_to_single_rank_gradient():
    """Samples sharded by ordinal range over ranks sum (allreduce) to the
    single-rank gradient — the multi-GPU decomposition, emulated on one GPU
    by running each rank's shard on its own context."""
    g = G()
    rs = np.random.default_rng(17)
    dims, r = (40, 30, 20), 8
    coords, vals = _sparse_problem(rs, dims, 800, values="count")
    F = [rs.uniform(0.1, 1, (n, r)) for n in dims]
    sk, lf = g.SamplerKind.semi_stratified(700, 900), g.LossFunction.poisson()
    full = g.Engine(dims, r, dtype="f64")
    full.set_sparse(coords, vals)
    full.set_factors(F)
    full.stoch_grad(sk, lf, 3, 1)
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


def test_bit_and_byte_storage_agree(orc):
    """BIT-packed and U8 storage of the same generated binary tensor give the
    same values and the same gradient; set_dense('bit') matches the oracle."""
    g = G()
    rs = np.random.default_rng(12)
    dims, R, r = (33, 17, 9, 5), 3, 6
    T = [rs.uniform(0, 1, (n, R)) for n in dims]
    F = [rs.uniform(0.05, 1.0, (n, r)) for n in dims]
    eb = g.Engine(dims, r, dtype="f64")
    eu = g.Engine(dims, r, dtype="f64")
    eb.generate_dense_bernoulli(T, seed=5, storage="bit")
    eu.generate_dense_bernoulli(T, seed=5, storage="u8")
    idx = np.stack([rs.integers(0, n, 4000) for n in dims], 1)
    xb, xu = eb.value_at(idx), eu.value_at(idx)
    assert np.array_equal(xb, xu) and set(np.unique(xb)) <= {0.0, 1.0} and xb.sum() > 0
    assert eb.tensor_norm() == pytest.approx(eu.tensor_norm(), rel=1e-15)
    for e in (eb, eu):
        e.set_factors(F)
        e.stoch_grad(g.SamplerKind.uniform(5000), g.LossFunction.bernoulli_odds(), 3, 1)
    assert O.rel_error(eb.grad_flat(), eu.grad_flat()) <= 1e-12
    # host-packed bits against the oracle
    dense = (rs.random(int(np.prod(dims))) < 0.2).astype(float)
    e = g.Engine(dims, r, dtype="f32")
    e.set_dense(dense, "bit")
    F32 = _as_dtype(F, "f32")
    e.set_factors(F32)
    e.stoch_grad(g.SamplerKind.uniform(3000), g.LossFunction.bernoulli_odds(), 8, 2)
    rc, want = orc.draw_gradient_samples(O.Tensor(dims, dense=dense), r, F32, 2, 0.0, 0, 3000, 0,
                                         0, 1.1, orc.source(1, seed=8, it=2))
    assert rc == 0
    grad = orc.mttkrp(dims, r, F32, want["idx"], want["y"])
    assert O.rel_error(e.grad_flat(), grad) <= TOL["f32"]
