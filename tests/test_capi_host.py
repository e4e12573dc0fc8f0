"""C-ABI checks that need no GPU: the engine library loads, exports every
entry point include/gcpb.h declares, and its host-side logic (Philox replica,
rejection batch formula, shard ranges, stratified merge, loss functions,
argument validation) matches the oracle / the reference semantics."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import oracle as O

ROOT = Path(__file__).resolve().parent.parent


def test_library_exports_every_declared_symbol():
    from paper_1906_01687_b200 import _capi
    header = (ROOT / "include" / "gcpb.h").read_text()
    declared = set(re.findall(r"\b(gcpb_[a-z0-9_]+)\s*\(", header))
    declared.discard("gcpb_ctx")
    assert len(declared) >= 40
    for name in sorted(declared):
        assert hasattr(_capi.lib, name), name
    assert declared == set(_capi.EXPORTED), declared ^ set(_capi.EXPORTED)
    assert _capi.lib.gcpb_version().startswith(b"gcpb")


def test_engine_library_is_sm100a():
    import subprocess
    lib = ROOT / "paper_1906_01687_b200" / "libgcpb.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(lib)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


@pytest.mark.parametrize("trial", range(4))
def test_host_philox_matches_oracle_replica(orc, trial):
    import paper_1906_01687_b200.gcp as G
    rs = np.random.default_rng(trial)
    for _ in range(3000):
        seed = int(rs.integers(0, 2**63)) * 2 + int(rs.integers(0, 2))
        tag = int(rs.integers(1, 8))
        it = int(rs.integers(0, 2**47))
        t = int(rs.integers(0, 2**47))
        k = int(rs.integers(0, 16))
        n = int(rs.choice([1, 2, 3, 200, 1000, 4_800_000, 2**31 - 1, 2**32, 2**32 + 1,
                           2**45 + 3, 2**63 - 25]))
        assert G.philox_bounded(seed, tag, it, t, k, n) == orc.draw_bounded(seed, tag, it, t, k, n)


def test_philox_draws_are_uniform(orc):
    """Lemire bounded draws: chi-square over 7 buckets, and range checks."""
    vals = np.array([orc.draw_bounded(3, 1, 0, t, 1, 7) for t in range(14000)])
    assert vals.min() >= 0 and vals.max() <= 6
    counts = np.bincount(vals, minlength=7)
    chi2 = ((counts - 2000.0) ** 2 / 2000.0).sum()
    assert chi2 < 22.46  # p = 0.001 at 6 dof


def test_zero_batch_size_matches_reference_formula(orc):
    import paper_1906_01687_b200.gcp as G
    rs = np.random.default_rng(5)
    for _ in range(500):
        total = float(rs.integers(2, 10**12))
        zeta = float(rs.integers(1, int(total)))
        rho = float(rs.uniform(1.0001, 3.0))
        sf = int(rs.integers(1, 10**7))
        assert G.zero_batch_size(total, zeta, rho, sf) == orc.lib.or_zero_batch_size(total, zeta, rho, sf)
    assert G.zero_batch_size(1e300, 1.0, 1.1, 10**9) == 9 * 10**15  # clamp (samplers.hpp:121)


@pytest.mark.parametrize("n,nranks", [(0, 3), (1, 2), (10, 3), (1_000_003, 8), (7, 8)])
def test_shard_ranges_partition(n, nranks):
    import paper_1906_01687_b200.gcp as G
    spans = [G.shard_range(n, r, nranks) for r in range(nranks)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    for (b0, e0), (b1, e1) in zip(spans, spans[1:]):
        assert e0 == b1 and b0 <= e0
    sizes = [e - b for b, e in spans]
    assert max(sizes) - min(sizes) <= 1


def test_stratified_keep_takes_first_accepts_in_rank_order():
    import paper_1906_01687_b200.gcp as G
    acc = [5, 0, 7, 3]
    need = 10
    kept = []
    for r in range(4):
        off, keep = G.stratified_keep(acc, r, need)
        assert off == sum(acc[:r])
        kept.append(keep)
    assert kept == [5, 0, 5, 0]
    assert sum(kept) == need


@pytest.mark.parametrize("kind,delta", [(0, 0.0), (1, 0.0), (2, 0.0), (3, 0.0), (4, 0.0), (5, 0.7)])
def test_host_loss_matches_oracle(orc, kind, delta):
    import paper_1906_01687_b200.gcp as G
    L = G.LossFunction(kind, delta)
    rs = np.random.default_rng(kind + 10)
    for _ in range(100):
        x = float(rs.integers(0, 2)) if kind == 2 else float(rs.uniform(0, 4))
        m = float(rs.uniform(0, 3))
        assert L.deriv(x, m) == orc.lib.or_loss_deriv(kind, delta, x, m)
        assert L.value(x, m) == orc.lib.or_loss_value(kind, delta, x, m)


def test_loss_parse_and_domain():
    import paper_1906_01687_b200.gcp as G
    assert G.LossFunction.parse("bernoulli-odds").kind == G.BERNOULLI_ODDS
    assert G.LossFunction.parse("huber:0.25").delta == 0.25
    assert G.LossFunction.parse("poisson").default_lower_bound() == 0.0
    assert G.LossFunction.parse("gaussian").default_lower_bound() is None
    with pytest.raises(G.InvalidArgument):
        G.LossFunction.parse("cauchy")
    with pytest.raises(G.InvalidArgument):
        G.LossFunction.parse("huber:x")
    with pytest.raises(G.InvalidArgument):
        G.LossFunction.huber(0.0)
    with pytest.raises(G.DomainError):
        G.LossFunction.bernoulli_odds().deriv(2.0, 1.0)
    with pytest.raises(G.DomainError):
        G.LossFunction.poisson().value(-1.0, 1.0)


def test_sampler_kind_tokens_and_validation():
    """test_samplers.cpp:38-61."""
    import paper_1906_01687_b200.gcp as G
    u = G.SamplerKind.from_token("uniform", 10)
    assert u.strategy == G.UNIFORM and u.num_samples == 10 and u.token() == "uniform"
    st = G.SamplerKind.from_token("stratified", 11)
    assert (st.nonzero_samples, st.zero_samples) == (5, 6)
    se = G.SamplerKind.from_token("semi-stratified", 1)
    assert (se.nonzero_samples, se.zero_samples) == (0, 1)
    for bad in [lambda: G.SamplerKind.from_token("hybrid", 10),
                lambda: G.SamplerKind.from_token("uniform", 0), lambda: G.SamplerKind.uniform(0),
                lambda: G.SamplerKind.stratified(0, 0), lambda: G.SamplerKind.stratified(-1, 2),
                lambda: G.SamplerKind.stratified(1, 1, 1.0)]:
        with pytest.raises(G.InvalidArgument):
            bad()
    G.SamplerKind.semi_stratified(0, 1).validate()


def test_create_validates_arguments_before_touching_the_device():
    import paper_1906_01687_b200.gcp as G
    with pytest.raises(G.InvalidArgument):
        G.Engine([3, 0, 2], 2)  # Shape: every extent must be positive
    with pytest.raises(G.InvalidArgument):
        G.Engine([], 2)
    with pytest.raises(G.InvalidArgument):
        G.Engine([2] * 17, 2)
    with pytest.raises(G.InvalidArgument):
        G.Engine([3, 4], 0)
    with pytest.raises(G.InvalidArgument):
        G.Engine([3, 4], 2, dtype="f16")
