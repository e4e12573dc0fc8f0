"""fp32 device gradients against the fp64 reference at BASELINE.json sizes.

north_star: on identical sampled index sets and factor matrices the GPU
gradient must match the reference within 1e-4 relative (fp32).  Here every
config C2-C5 is built at its full size exactly as bench.py builds it, >= 1e6
draws are recorded from the device sampler (index, stored value, weight,
flag), and the reference's own code in oracle/_ref computes the gradient of
those draws in fp64 from the same (fp32-representable) factors:

    y_e  = w_e * deriv(x_e, entry(i_e))                 samplers.hpp:87-93
           w_e * (deriv(x_e, m) - deriv(0, m))  (semi)  samplers.hpp:199-207
    G    = mttkrp_sampled_all(samples, model, threads)  kernels.cpp:137-168

and the fused kernel's gradient of the same call (same seed/iteration, hence
the same draws) must agree to rel_error <= 1e-4 (tests/oracles.hpp:174-182).
This covers the Zipf-hot rows (~1e5 fp32 reductions per address, SURVEY.md
§7 hard part 4) that the small parity cases cannot.

C1 at full config size (100^3 dense fp64, r=5, s=300, 3000 estimator samples,
tau=1000) runs the device fit in RefStream mode against the reference's own
fit_gcp_adam(seed) epoch by epoch.
"""
import ctypes as C
import gc
import os
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

LOSS = {"gaussian": 0, "poisson": 1, "bernoulli-odds": 2}


def _engine(name):
    import bench
    from paper_1906_01687_b200 import workloads as WL
    w = WL.get(name)
    return w, bench.setup_engine(w, 0, lambda m: None)


def _free_gb():
    import torch
    free, _ = torch.cuda.mem_get_info()
    return free / 2**30


def _reference_gradient(ref, w, F, out):
    """The reference's fp64 gradient of the recorded draws."""
    lk = LOSS[w.loss]
    idx, x, wt, flag = out["idx"], out["x"], out["w"], out["flag"]
    y = np.empty(len(x))
    semi = flag == 1
    for sel, sub in ((semi, True), (~semi, False)):
        if sel.any():
            y[sel] = ref.weighted_derivs(w.dims, w.rank, F, lk, 0.0, idx[sel], x[sel], wt[sel],
                                         subtract_zero=sub)
    return ref.mttkrp(w.dims, w.rank, F, idx, y, threads=os.cpu_count() or 1)


def _check(ref, name, sampler, seed, it, n_min=1_000_000):
    g = pytest.importorskip("paper_1906_01687_b200.gcp")
    w, e = _engine(name)
    F = e.factors()  # fp32 factors, upcast exactly
    loss = g.LossFunction.parse(w.loss)
    sk = sampler(g, w)
    out = e.draw_samples(sk, loss, seed, it)
    assert len(out["idx"]) >= n_min
    e.stoch_grad(sk, loss, seed, it)  # the fused kernel: same seed/iteration = same draws
    fused = e.grad_flat()
    e.close()
    del e
    gc.collect()
    want = _reference_gradient(ref, w, F, out)
    err = O.rel_error(fused, want)
    assert err <= 1e-4, (name, err)
    return out, err


def test_c2_fullsize_fp32_gradient_matches_fp64_reference(ref):
    out, _ = _check(ref, "c2", lambda g, w: g.SamplerKind.uniform(2_000_000), 3002, 21)
    assert np.all(out["flag"] == 0)


def test_c3_fullsize_fp32_gradient_matches_fp64_reference(ref):
    out, _ = _check(ref, "c3", lambda g, w: g.SamplerKind.stratified(w.p, w.q, w.rho), 3003, 22,
                    n_min=2_000_000)
    assert np.all(out["x"][:1_000_000] == 1.0) and np.all(out["x"][1_000_000:] == 0.0)


def test_c4_fullsize_fp32_gradient_matches_fp64_reference(ref):
    # the config's own p = q = 1e5 step, and a 1e6-draw call
    _check(ref, "c4", lambda g, w: g.SamplerKind.semi_stratified(w.p, w.q), 3004, 23,
           n_min=200_000)
    _check(ref, "c4", lambda g, w: g.SamplerKind.semi_stratified(500_000, 500_000), 3004, 24)


def test_c5_fullsize_fp32_gradient_matches_fp64_reference(ref):
    if _free_gb() < 100:
        pytest.skip("C5 needs ~60 GB of device memory")
    out, _ = _check(ref, "c5", lambda g, w: g.SamplerKind.semi_stratified(1_000_000, 1_000_000),
                    3005, 25, n_min=2_000_000)
    assert np.all(out["flag"][:1_000_000] == 1) and np.all(out["flag"][1_000_000:] == 0)


def test_c5_fullsize_step_gradient_matches_fp64_reference(ref):
    """The C5 step itself (p = q = 1.6e7: interleaved table, unrestricted
    draws walked in mode-0 order, hot-row copies) against the reference on
    the same 3.2e7 draws."""
    if _free_gb() < 100:
        pytest.skip("C5 needs ~60 GB of device memory")
    g = pytest.importorskip("paper_1906_01687_b200.gcp")
    w, e = _engine("c5")
    F = e.factors()
    loss = g.LossFunction.parse(w.loss)
    sk = g.SamplerKind.semi_stratified(w.p, w.q)
    out = e.draw_samples(sk, loss, 3005, 26)
    # one iteration through the step path with a zero learning rate leaves
    # the factors unchanged; its gradient is the fused scatter on the
    # interleaved table (read back through the moments: B = (1-b1) G)
    e.step(sk, loss, 3005, 26, 0.0, lower_bound=w.lower_bound)
    assert e.interleaved[1]
    first = np.concatenate([m.ravel() for m in e.moment(0)])
    e.close()
    del e
    gc.collect()
    want = _reference_gradient(ref, w, F, out)
    assert O.rel_error(first / 0.1, want) <= 1e-4


def test_c1_fullsize_refstream_fit_matches_reference(ref):
    """C1 as configured: the device fit_gcp_adam in RefStream mode against the
    reference's fit_gcp_adam(seed), per-epoch loss estimates <= 1e-9."""
    import bench
    from paper_1906_01687_b200.fit import FitConfig, fit_gcp_adam
    g = pytest.importorskip("paper_1906_01687_b200.gcp")
    dims, R, epochs, seed = (100, 100, 100), 5, 4, 2001
    X = bench.c1_tensor()
    rt = ref.dense(dims, X)
    trace = np.zeros((epochs + 2, 5))
    nt = C.c_int64()
    Fout = np.zeros(int(np.sum(dims)) * R)
    fin = C.c_double()
    ref._ck(ref.lib.ref_fit_gcp_adam(rt.h, 0, 0.0, R, 0, 300, 0, 0, 1.1, 1e-3, 0.9, 0.999, 1e-8,
                                     1000, 1, 0.1, 0, 0.0, 3000, -1, epochs, seed, 1, epochs + 2,
                                     O._f64(trace), C.byref(nt), O._f64(Fout), C.byref(fin)))
    want = trace[:nt.value]
    e = g.Engine(dims, R, "f64")
    e.set_dense(X, "f64")
    res = fit_gcp_adam(e, g.LossFunction.gaussian(),
                       FitConfig(rank=R, sampler=g.SamplerKind.uniform(300), learning_rate=1e-3,
                                 epoch_iters=1000, estimator_samples=3000, max_epochs=epochs,
                                 seed=seed, draw_stream="reference"))
    assert len(res.trace) == len(want)
    for rec, wrow in zip(res.trace, want):
        assert rec.epoch == int(wrow[0])
        assert rec.loss_estimate == pytest.approx(wrow[1], rel=1e-9)
        assert rec.accepted == bool(wrow[4])
    assert O.rel_error(np.concatenate([f.reshape(-1) for f in res.model]), Fout) <= 1e-8
    e.close()
