"""Pins the C restatement oracle (oracle/gcp_oracle.c) before it is trusted:
  * against tests/golden/reference_vectors.json — outputs of the reference
    itself (oracle/_ref), so this runs anywhere, including the GPU box;
  * against the live compiled reference on fresh random cases, when
    oracle/_ref is present (this container).
The bar: bit-exact for integer work (RNG, indices, counts), <= 1e-12 relative
for fp64 arithmetic (the reference's own pins, tests/test_kernels.cpp)."""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle as O

GOLD = json.loads((Path(__file__).parent / "golden" / "reference_vectors.json").read_text())


def _tensor(c):
    if c.get("tensor_kind", "sparse") == "dense":
        return O.Tensor(c["dims"], dense=np.array(c["dense"]))
    return O.Tensor(c["dims"], np.array(c["coords"], dtype=np.int64).reshape(-1, len(c["dims"])),
                    np.array(c["values"]))


# ---------------------------------------------------------------- golden pins
def test_rngstream_known_answers(orc):
    import ctypes as C
    for c in GOLD["rng"]:
        seed = int(c["seed"])
        r = orc.rng_stream(seed)
        got = [str(orc.lib.or_rng_next_u64(C.byref(r))) for _ in range(4)]
        assert got == c["next_u64"]
        assert [orc.lib.or_rng_next_double(C.byref(r)) for _ in range(2)] == c["next_double"]
        assert [orc.lib.or_rng_next_below(C.byref(r), 1000) for _ in range(4)] == c["next_below_1000"]
        assert [orc.lib.or_rng_next_below(C.byref(r), 3) for _ in range(4)] == c["next_below_3"]
        root = orc.rng_stream(seed)
        gs = orc.split(root, "gradients")
        assert [str(orc.lib.or_rng_next_u64(C.byref(gs))) for _ in range(2)] == c["split_gradients_u64"]
        s7 = orc.split(root, 7)
        assert [str(orc.lib.or_rng_next_u64(C.byref(s7)))] == c["split_7_u64"]


def test_loss_known_answers(orc):
    for c in GOLD["loss"]:
        v = orc.lib.or_loss_value(c["kind"], c["delta"], c["x"], c["m"])
        g = orc.lib.or_loss_deriv(c["kind"], c["delta"], c["x"], c["m"])
        assert v == c["value"] or (np.isnan(v) and np.isnan(c["value"])), c
        assert g == c["deriv"], c


def test_mttkrp_known_answers(orc):
    for c in GOLD["mttkrp"]:
        got = orc.mttkrp(c["dims"], c["r"], [np.array(f) for f in c["factors"]],
                         np.array(c["idx"]), np.array(c["y"]))
        assert O.rel_error(got, c["grad"]) <= 1e-14


@pytest.mark.parametrize("case", GOLD["samplers"], ids=lambda c: c["name"])
def test_sampler_known_answers(orc, case):
    """Scripted replay (ScriptedRng semantics) and the Philox source both
    reproduce the reference sampler's samples, counts and script length."""
    t = _tensor(case)
    F = [np.array(f) for f in case["factors"]]
    for src in (orc.source(0, script=case["script"]),
                orc.source(1, seed=case["seed"], it=case["iter"])):
        rc, out = orc.draw_gradient_samples(t, case["r"], F, case["loss"], case["delta"],
                                            case["strategy"], case["s"], case["p"], case["q"],
                                            case["rho"], src)
        assert rc == 0
        assert np.array_equal(out["idx"], np.array(case["idx"]).reshape(out["idx"].shape))
        assert O.rel_error(out["y"], case["y"]) <= 1e-14
        assert out["consumed"] == case["consumed"]
        if case["strategy"] == 1:
            assert list(out["stats"]) == case["stats"]
    g = orc.mttkrp(case["dims"], case["r"], F, np.array(case["idx"]), np.array(case["y"]))
    assert O.rel_error(g, case["grad"]) <= 1e-14


def test_adam_known_answers(orc):
    for c in GOLD["adam"]:
        A = [np.array(f) for f in c["factors"]]
        n = sum(len(f) for f in c["factors"]) * c["r"]
        B, Cm, it = np.zeros(n), np.zeros(n), 0
        for st in c["steps"]:
            mats, at = [], 0
            flat = O.Oracle.flat(A)
            for nk in c["dims"]:
                mats.append(flat[at:at + nk * c["r"]].reshape(nk, c["r"]))
                at += nk * c["r"]
            Af, B, Cm, it = orc.adam(c["dims"], c["r"], mats, B, Cm, it, c["lr"],
                                     np.array(st["grad"]), lb=c["lb"])
            assert np.array_equal(Af, np.array(st["A"]))
            assert np.array_equal(B, np.array(st["B"]))
            assert np.array_equal(Cm, np.array(st["C"]))
            assert it == st["iterations"]
            A = [Af]
            A = [Af[sum(c["dims"][:k]) * c["r"]:sum(c["dims"][:k + 1]) * c["r"]].reshape(nk, c["r"])
                 for k, nk in enumerate(c["dims"])]


def test_estimator_known_answers(orc):
    for c in GOLD["estimator"]:
        t = O.Tensor(c["dims"], np.array(c["coords"]), np.array(c["values"]))
        F = [np.array(f) for f in c["factors"]]
        for src in (orc.source(0, script=c["script"]),
                    orc.source(1, seed=c["seed"], it=0, estimator=True)):
            rc, idx, x, w = orc.estimator_draw(t, c["kind"], c["count"], 1.1, src)
            assert rc == 0
            assert np.array_equal(idx, np.array(c["idx"]).reshape(idx.shape))
            assert np.array_equal(x, np.array(c["x"]))
            assert np.array_equal(w, np.array(c["w"]))
        v = orc.estimate(c["dims"], c["r"], F, c["loss"], 0.0, np.array(c["idx"]), np.array(c["x"]),
                         np.array(c["w"]))
        assert v == pytest.approx(c["estimate"], rel=1e-14)


def test_sparse_normalize_known_answer():
    c = GOLD["normalize"]
    t = O.Tensor(c["dims"], np.array(c["coords"]), np.array(c["values"]))
    assert np.array_equal(t.coords, np.array(c["out_coords"]))
    assert np.array_equal(t.values, np.array(c["out_values"]))


def test_philox_known_answers(orc):
    for c in GOLD["philox"]:
        assert orc.draw_bounded(int(c["seed"]), c["tag"], c["iter"], c["t"], c["k"], c["n"]) == c["value"]


# ---------------------------------------------------------- live reference pins
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_live_rng_matches_reference(orc, ref, seed):
    import ctypes as C
    rs = np.random.default_rng(seed)
    for _ in range(5):
        s = int(rs.integers(0, 2**63))
        a = ref.rng(s)
        b = orc.rng_stream(s)
        for n in [1, 2, 7, 1000, 2**33 + 5, 2**63 + 11]:
            assert a.next_below(n) == orc.lib.or_rng_next_below(C.byref(b), n)
        assert a.next_u64() == orc.lib.or_rng_next_u64(C.byref(b))


@pytest.mark.parametrize("kind,delta", [(0, 0), (1, 0), (2, 0), (3, 0), (4, 0), (5, 0.3)])
def test_live_loss_matches_reference(orc, ref, kind, delta):
    rs = np.random.default_rng(kind)
    for _ in range(200):
        x = float(rs.integers(0, 2)) if kind == 2 else float(rs.uniform(0, 5))
        m = float(rs.uniform(0, 4)) if kind not in (0, 5) else float(rs.uniform(-3, 3))
        assert orc.lib.or_loss_value(kind, delta, x, m) == ref.loss_value(kind, delta, x, m)
        assert orc.lib.or_loss_deriv(kind, delta, x, m) == ref.loss_deriv(kind, delta, x, m)


@pytest.mark.parametrize("dims,r", [((5, 4, 3, 2), 3), ((30, 20, 10), 8), ((9, 8), 5)])
def test_live_mttkrp_matches_reference(orc, ref, dims, r):
    rs = np.random.default_rng(sum(dims))
    F = [rs.uniform(-1, 1, (n, r)) for n in dims]
    n = 5000
    idx = np.stack([rs.integers(0, k, n) for k in dims], 1)
    y = rs.uniform(-1, 1, n)
    want = ref.mttkrp(dims, r, F, idx, y)
    assert O.rel_error(orc.mttkrp(dims, r, F, idx, y), want) <= 1e-14
    # threaded reference (kernels.cpp:148-166) agrees to the reference's own 1e-12 pin
    assert O.rel_error(ref.mttkrp(dims, r, F, idx, y, threads=4), want) <= 1e-12


@pytest.mark.parametrize("strategy,loss", [(0, 0), (0, 1), (1, 2), (1, 1), (2, 2), (2, 1), (2, 4)])
def test_live_samplers_match_reference(orc, ref, strategy, loss):
    rs = np.random.default_rng(100 + strategy * 7 + loss)
    dims = (9, 7, 5, 4)
    total = int(np.prod(dims))
    lin = np.nonzero(rs.random(total) < 0.05)[0]
    coords = np.stack(np.unravel_index(lin, dims, order="F"), 1)
    vals = np.ones(len(lin)) if loss == 2 else 1.0 + rs.poisson(2.0, len(lin))
    rt = ref.sparse(dims, coords, vals)
    ot = O.Tensor(dims, coords, vals)
    r = 4
    F = [rs.uniform(0.1, 1, (n, r)) for n in dims]
    s, p, q = (200, 0, 0) if strategy == 0 else (0, 150, 170)
    src = orc.source(1, seed=5 + loss, it=3)
    rc, out = orc.draw_gradient_samples(ot, r, F, loss, 0.0, strategy, s, p, q, 1.1, src)
    assert rc == 0
    if strategy == 0:
        script = O.philox_script(orc, 0, dims, 5 + loss, 3, s=s)
    else:
        script = O.philox_script(orc, strategy, dims, 5 + loss, 3, p=p, eta=rt.nnz,
                                 n_cand=(src.at - p) // len(dims), q=q)
    res = rt.draw_scripted(r, F, loss, 0.0, strategy, s, p, q, 1.1, script)
    assert res["consumed"] == len(script) == src.at
    assert np.array_equal(res["idx"], out["idx"])
    assert O.rel_error(out["y"], res["y"]) <= 1e-14
    if strategy == 1:
        assert tuple(res["stats"]) == out["stats"]


def test_live_zero_batch_formula(orc, ref):
    import paper_1906_01687_b200.gcp as G  # host helper of the product (no GPU needed)
    for total, zeta, rho, sf in [(1e12, 1e12 - 1e7, 1.1, 1_000_000), (24.0, 23.0, 1.1, 3),
                                 (4.0, 3.0, 1.1, 3), (1e6, 5e5, 1.5, 17), (10.0, 1.0, 1.01, 1)]:
        want = orc.lib.or_zero_batch_size(total, zeta, rho, sf)
        assert G.zero_batch_size(total, zeta, rho, sf) == want
    assert orc.lib.or_zero_batch_size(4.0, 3.0, 1.1, 3) == 5  # test_samplers.cpp:163-165


def test_oracle_error_codes(orc):
    t = O.Tensor((2, 2), np.array([[0, 0], [1, 0], [0, 1]]), np.ones(3))
    F = [np.ones((2, 1)), np.ones((2, 1))]
    # asking for more zeros than exist (samplers.hpp:108-111) -> usage
    rc, _ = orc.draw_gradient_samples(t, 1, F, 0, 0.0, 1, 0, 0, 2, 1.1, orc.source(1, seed=1))
    assert rc == 2
    rc, _ = orc.draw_gradient_samples(t, 1, F, 0, 0.0, 1, 0, 1, 1, 1.0, orc.source(1, seed=1))
    assert rc == 2
    # bernoulli loss on a count value -> domain
    t2 = O.Tensor((2, 2), np.array([[0, 0]]), np.array([3.0]))
    rc, _ = orc.draw_gradient_samples(t2, 1, F, 2, 0.0, 1, 0, 1, 0, 1.1, orc.source(1, seed=1))
    assert rc == 3
