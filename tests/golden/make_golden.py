"""Generates tests/golden/reference_vectors.json from the REFERENCE ITSELF.

Run here (where /root/reference exists and oracle/_ref/libgcpref.so was built
from the unmodified reference sources by oracle/Makefile):

    python tests/golden/make_golden.py

Every output value below is produced by the reference's own code
(RngStream, LossFunction, draw_gradient_samples with ScriptedRng,
mttkrp_sampled_all, adam_step, EstimatorSamples) — the fixtures pin the oracle
restatement and the GPU engine on the GPU box, where /root/reference is absent.
The draw scripts are the product's Philox stream (oracle replica), so the same
(seed, iter) on the GPU must reproduce the indices bit-exactly.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT / "oracle"))
import oracle as O  # noqa: E402

OUT = Path(__file__).resolve().parent / "reference_vectors.json"
U64 = (1 << 64) - 1


def rand_factors(rng, dims, r, lo=0.1, hi=1.0):
    return [rng.uniform(lo, hi, size=(n, r)) for n in dims]


def random_sparse(rng, dims, density, valfn):
    total = int(np.prod(dims))
    lin = np.nonzero(rng.random(total) < density)[0]
    coords = np.stack(np.unravel_index(lin, dims, order="F"), axis=1).astype(np.int64)
    return coords, valfn(len(lin))


def main():
    ref = O.reference()
    if ref is None:
        raise SystemExit("build oracle/_ref first (make -C oracle ref)")
    orc = O.oracle()
    g = {"generator": "tests/golden/make_golden.py", "source": "oracle/_ref (reference)"}

    # 1. RngStream known answers (rng.cpp:12-61)
    rng_cases = []
    for seed in [0, 1, 42, 2**63 + 5]:
        s = ref.rng(seed)
        c = {"seed": str(seed), "next_u64": [str(s.next_u64()) for _ in range(4)],
             "next_double": [s.next_double() for _ in range(2)],
             "next_below_1000": [s.next_below(1000) for _ in range(4)],
             "next_below_3": [s.next_below(3) for _ in range(4)]}
        root = ref.rng(seed)
        gsplit = root.split("gradients")
        c["split_gradients_u64"] = [str(gsplit.next_u64()) for _ in range(2)]
        c["split_7_u64"] = [str(root.split(7).next_u64()) for _ in range(1)]
        rng_cases.append(c)
    g["rng"] = rng_cases

    # 2. Loss values / derivatives (loss.cpp:64-110)
    loss_cases = []
    for kind, delta in [(0, 0.0), (1, 0.0), (2, 0.0), (3, 0.0), (4, 0.0), (5, 0.5)]:
        xs = [0.0, 1.0] if kind == 2 else [0.0, 0.5, 3.0]
        ms = [0.0, 1e-3, 0.7, 2.5] + ([-1.2] if kind in (0, 5) else [])
        for x in xs:
            for m in ms:
                loss_cases.append({"kind": kind, "delta": delta, "x": x, "m": m,
                                   "value": ref.loss_value(kind, delta, x, m),
                                   "deriv": ref.loss_deriv(kind, delta, x, m)})
    g["loss"] = loss_cases

    rs = np.random.default_rng(20261020)

    # 3. mttkrp_sampled_all on given samples (kernels.cpp:137-168)
    mt = []
    for dims, r, n in [((3, 4, 5), 2, 40), ((5, 4, 3, 2), 3, 60), ((4, 3, 2), 5, 25),
                       ((7,), 3, 10), ((6, 5), 4, 30)]:
        F = rand_factors(rs, dims, r, -1.0, 1.0)
        idx = np.stack([rs.integers(0, nk, size=n) for nk in dims], axis=1)
        y = rs.uniform(-2.0, 2.0, size=n)
        grad = ref.mttkrp(dims, r, F, idx, y)
        mt.append({"dims": list(dims), "r": r, "factors": [f.tolist() for f in F],
                   "idx": idx.tolist(), "y": y.tolist(), "grad": grad.tolist()})
    g["mttkrp"] = mt

    # 4. Samplers on the product's Philox stream, evaluated by the reference
    #    sampler code via ScriptedRng (samplers.hpp:75-245).
    samp = []
    sparse_dims = (6, 5, 4)
    coords, vals = random_sparse(rs, sparse_dims, 0.3, lambda n: np.ones(n))
    counts, cvals = random_sparse(rs, sparse_dims, 0.25, lambda n: 1.0 + rs.poisson(2.0, n))
    real, rvals = random_sparse(rs, sparse_dims, 0.2, lambda n: rs.uniform(0.5, 2.0, n))
    dense_dims = (4, 3, 5)
    dense_vals = rs.uniform(0.0, 2.0, size=int(np.prod(dense_dims)))
    cases = [
        # (name, tensor, loss kind, delta, strategy, s, p, q, rho, seed, iter)
        ("uniform_dense_gaussian", ("dense", dense_dims, dense_vals), 0, 0.0, 0, 25, 0, 0, 1.1, 7, 0),
        ("uniform_dense_huber", ("dense", dense_dims, dense_vals), 5, 0.4, 0, 25, 0, 0, 1.1, 9, 3),
        ("uniform_sparse_poisson", ("sparse", sparse_dims, counts, cvals), 1, 0.0, 0, 30, 0, 0, 1.1, 11, 2),
        ("stratified_binary_bern", ("sparse", sparse_dims, coords, vals), 2, 0.0, 1, 0, 12, 15, 1.1, 13, 5),
        ("stratified_count_poisson", ("sparse", sparse_dims, counts, cvals), 1, 0.0, 1, 0, 10, 10, 1.3, 17, 1),
        ("stratified_real_gamma", ("sparse", sparse_dims, real, rvals), 3, 0.0, 1, 0, 8, 9, 1.1, 19, 4),
        ("semi_binary_bern", ("sparse", sparse_dims, coords, vals), 2, 0.0, 2, 0, 12, 15, 1.1, 23, 6),
        ("semi_count_poisson", ("sparse", sparse_dims, counts, cvals), 1, 0.0, 2, 0, 10, 10, 1.1, 29, 0),
        ("semi_real_betahalf", ("sparse", sparse_dims, real, rvals), 4, 0.0, 2, 0, 7, 9, 1.1, 31, 8),
        ("semi_real_gaussian", ("sparse", sparse_dims, real, rvals), 0, 0.0, 2, 0, 7, 9, 1.1, 37, 9),
    ]
    for name, tens, lk, delta, strat, s, p, q, rho, seed, it in cases:
        dims = tens[1]
        r = 3
        F = rand_factors(rs, dims, r, 0.1, 1.0)
        if tens[0] == "dense":
            rt = ref.dense(dims, tens[2])
            ot = O.Tensor(dims, dense=tens[2])
            eta = 0
        else:
            rt = ref.sparse(dims, tens[2], tens[3])
            ot = O.Tensor(dims, tens[2], tens[3])
            eta = rt.nnz
        # run the oracle's Philox source first to learn how many candidates
        # the stratified sampler tests (the script length)
        src = orc.source(1, seed=seed, it=it)
        rc, osm = orc.draw_gradient_samples(ot, r, F, lk, delta, strat, s, p, q, rho, src)
        assert rc == 0, (name, rc)
        consumed = osm["consumed"]
        if strat == 0:
            script = O.philox_script(orc, 0, dims, seed, it, s=s)
        else:
            n_cand = (consumed - p) // len(dims)
            script = O.philox_script(orc, strat, dims, seed, it, p=p, eta=eta, n_cand=n_cand, q=q)
        assert len(script) == consumed
        res = rt.draw_scripted(r, F, lk, delta, strat, s, p, q, rho, script)
        grad = ref.mttkrp(dims, r, F, res["idx"], res["y"])
        entry = {"name": name, "dims": list(dims), "r": r, "loss": lk, "delta": delta,
                 "strategy": strat, "s": s, "p": p, "q": q, "rho": rho, "seed": seed, "iter": it,
                 "factors": [f.tolist() for f in F], "tensor_kind": tens[0],
                 "script": [int(v) for v in script], "idx": res["idx"].tolist(),
                 "y": res["y"].tolist(), "stats": list(res["stats"]),
                 "consumed": res["consumed"], "grad": grad.tolist()}
        if tens[0] == "dense":
            entry["dense"] = tens[2].tolist()
        else:
            entry["coords"] = tens[2].tolist()
            entry["values"] = tens[3].tolist()
        samp.append(entry)
    g["samplers"] = samp

    # 5. adam_step (optimizer.cpp:47-66), two chained steps incl. projection
    ad = []
    for dims, r, lb in [((3, 2), 2, None), ((2, 4, 3), 3, 0.0)]:
        F = rand_factors(rs, dims, r, -0.5, 1.0)
        n = int(np.sum(dims)) * r
        B = np.zeros(n)
        Cm = np.zeros(n)
        it = 0
        grads = [rs.uniform(-3, 3, size=n) for _ in range(2)]
        steps = []
        A = O.Oracle.flat(F)
        for gr in grads:
            mats = []
            at = 0
            for nk in dims:
                mats.append(A[at:at + nk * r].reshape(nk, r))
                at += nk * r
            A, B, Cm, it = ref.adam(dims, r, mats, B, Cm, it, 0.05, gr, lb=lb)
            steps.append({"grad": gr.tolist(), "A": A.tolist(), "B": B.tolist(),
                          "C": Cm.tolist(), "iterations": it})
        ad.append({"dims": list(dims), "r": r, "lb": lb, "lr": 0.05,
                   "factors": [f.tolist() for f in F], "steps": steps})
    g["adam"] = ad

    # 6. EstimatorSamples (samplers.hpp:263-315, samplers.cpp:114-124)
    est = []
    for kind, lk, seed, count in [(0, 2, 41, 20), (1, 2, 43, 21), (1, 1, 47, 16)]:
        dims = sparse_dims
        r = 3
        F = rand_factors(rs, dims, r, 0.1, 1.0)
        cc, vv = (coords, vals) if lk == 2 else (counts, cvals)
        rt = ref.sparse(dims, cc, vv)
        ot = O.Tensor(dims, cc, vv)
        src = orc.source(1, seed=seed, it=0, estimator=True)
        rc, oi, ox, ow = orc.estimator_draw(ot, kind, count, 1.1, src)
        assert rc == 0
        consumed = src.at
        if kind == 0:
            script = O.philox_script(orc, 0, dims, seed, 0, s=count, estimator=True)
        else:
            p = count // 2
            n_cand = (consumed - p) // len(dims)
            script = O.philox_script(orc, 1, dims, seed, 0, p=p, eta=rt.nnz, n_cand=n_cand,
                                     estimator=True)
        assert len(script) == consumed
        idx, x, w, value = rt.estimator_scripted(kind, count, 1.1, script, r, F, lk, 0.0)
        est.append({"kind": kind, "loss": lk, "seed": seed, "count": count, "dims": list(dims),
                    "r": r, "factors": [f.tolist() for f in F], "coords": cc.tolist(),
                    "values": vv.tolist(), "script": [int(v) for v in script],
                    "idx": idx.tolist(), "x": x.tolist(), "w": w.tolist(), "estimate": value})
    g["estimator"] = est

    # 7. SparseTensor normalisation (tensor.cpp:10-41) with duplicates and zeros
    dims = (4, 3, 2)
    raw = np.array([[1, 2, 0], [0, 0, 0], [1, 2, 0], [3, 1, 1], [2, 2, 1], [2, 2, 1], [0, 1, 0]])
    rv = np.array([1.5, 2.0, -0.5, 0.0, 1.0, -1.0, 4.0])
    rt = ref.sparse(dims, raw, rv)
    c, v = rt.export()
    g["normalize"] = {"dims": list(dims), "coords": raw.tolist(), "values": rv.tolist(),
                      "out_coords": c.tolist(), "out_values": v.tolist()}

    # 8. Product Philox stream known answers (oracle replica; pins the design)
    ph = []
    for seed, tag, it, t, k, n in [(0, 1, 0, 0, 0, 1000), (123, 1, 5, 77, 3, 200),
                                   (2**63 + 1, 3, 2**40 + 3, 2**44 + 9, 2, 4_800_000),
                                   (99, 2, 1, 5, 0, 10_000_000), (7, 4, 9, 1, 1, 2**32),
                                   (11, 2, 3, 4, 0, 2**40 + 7), (5, 1, 0, 3, 15, 3)]:
        ph.append({"seed": str(seed), "tag": tag, "iter": it, "t": t, "k": k, "n": n,
                   "value": orc.draw_bounded(seed, tag, it, t, k, n)})
    g["philox"] = ph

    OUT.write_text(json.dumps(g, separators=(",", ":")))
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
