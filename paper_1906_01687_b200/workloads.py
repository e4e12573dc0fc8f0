"""BASELINE.json configs as synthetic workloads.

No public datasets are available offline; each config is a seeded generator
with the config's shape, size, value distribution and loss.  Seeds: data
1000 + c, init 2000 + c, Philox key = 3000 + c.

C1 dense 100^3 fp64, gaussian, r=5, uniform s=300
C2 dense 200^4 binary (bit-packed; u8 via GCPB_C2_STORAGE=u8), bernoulli-odds, r=16, uniform s in {1e5,1e6,1.6e7}
C3 sparse 1000^4, 1e7 nnz Zipf(1.1), bernoulli-odds, r=32, stratified p=q=1e6
C4 sparse 183x24x1140x1717, 3.3e6 nnz, poisson, r=20, semi-stratified p=q=1e5
C5 sparse 4.8e6x1.7e6x1.8e6, 1.7e9 nnz Zipf(1.05), gaussian, r=16, semi p=q=1.6e7
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np


@dataclass
class Workload:
    name: str
    dims: tuple
    rank: int
    dtype: str
    loss: str
    sampler: str           # uniform / stratified / semi-stratified
    s: int = 0
    p: int = 0
    q: int = 0
    rho: float = 1.1
    kind: str = "dense"    # dense / sparse
    nnz: int = 0
    description: str = ""
    lower_bound: Optional[float] = None
    extra: dict = field(default_factory=dict)

    @property
    def d(self) -> int:
        return len(self.dims)

    @property
    def samples_per_step(self) -> int:
        return self.s if self.sampler == "uniform" else self.p + self.q

    def bytes_per_sample(self) -> int:
        """Algorithmic bytes: int32 index per mode + gathered + scattered rows."""
        F = 4 if self.dtype == "f32" else 8
        return 4 * self.d + 2 * self.d * self.rank * F


def get(name: str, s: Optional[int] = None) -> Workload:
    name = name.lower()
    if name == "c1":
        return Workload("c1", (100, 100, 100), 5, "f64", "gaussian", "uniform", s=s or 300,
                        description="dense 100^3 fp64 rank-5 CP + 10% noise, gaussian, r=5, "
                                    "uniform s=300")
    if name == "c2":
        return Workload("c2", (200, 200, 200, 200), 16, "f32", "bernoulli-odds", "uniform",
                        s=s or 16_000_000, lower_bound=0.0,
                        description="dense 200^4 binary (bit-packed in HBM, 200 MB) from a rank-8 nonnegative "
                                    "odds model (mean p~0.1), bernoulli-odds, r=16, uniform")
    if name == "c3":
        return Workload("c3", (1000, 1000, 1000, 1000), 32, "f32", "bernoulli-odds", "stratified",
                        p=1_000_000, q=1_000_000, kind="sparse", nnz=10_000_000, lower_bound=0.0,
                        description="sparse 1000^4 binary, 1e7 unique Zipf(1.1) nonzeros, "
                                    "bernoulli-odds, r=32, stratified p=q=1e6 (hash rejection)")
    if name == "c4":
        return Workload("c4", (183, 24, 1140, 1717), 20, "f32", "poisson", "semi-stratified",
                        p=100_000, q=100_000, kind="sparse", nnz=3_300_000, lower_bound=0.0,
                        description="sparse 183x24x1140x1717 counts (1+Poisson(2)), 3.3e6 nnz, "
                                    "poisson, r=20, semi-stratified p=q=1e5")
    if name == "c5":
        return Workload("c5", (4_800_000, 1_700_000, 1_800_000), 16, "f32", "gaussian",
                        "semi-stratified", p=16_000_000, q=16_000_000, kind="sparse",
                        nnz=1_700_000_000,
                        description="sparse 4.8e6x1.7e6x1.8e6, 1.7e9 Zipf(1.05) nonzeros, "
                                    "log(1+Poisson(3)) values, gaussian, r=16, semi p=q=1.6e7")
    raise ValueError(f"unknown workload {name}")


# ---------------------------------------------------------------------------
# generators
# ---------------------------------------------------------------------------
def c2_true_factors(seed: int = 1002, target_p: float = 0.1):
    """Rank-8 nonnegative odds model, U(0,1) entries scaled by c so that
    mean m/(1+m) over 1e6 random entries ~= target_p (bisection)."""
    rs = np.random.default_rng(seed)
    dims, R = (200, 200, 200, 200), 8
    A = [rs.uniform(0.0, 1.0, (n, R)) for n in dims]
    idx = [rs.integers(0, n, 1_000_000) for n in dims]
    m1 = np.ones((1_000_000, R))
    for k in range(4):
        m1 *= A[k][idx[k]]
    m1 = m1.sum(1)
    lo, hi = 1e-12, 1e6  # scale s = c^4 on m
    for _ in range(200):
        mid = np.sqrt(lo * hi)
        p = np.mean(mid * m1 / (1.0 + mid * m1))
        if p < target_p:
            lo = mid
        else:
            hi = mid
    c = np.sqrt(lo * hi) ** 0.25
    return [a * c for a in A]


def model_norm(F) -> float:
    """KruskalModel::norm (kruskal.cpp:75-83): sqrt(1' (hadamard_k A_k'A_k) 1)."""
    gram = np.ones((F[0].shape[1], F[0].shape[1]))
    for f in F:
        gram = gram * (f.T @ f)
    return float(np.sqrt(max(0.0, gram.sum())))


def init_factors(dims, rank, seed, data_norm=None, lo=0.0, hi=1.0):
    """Default fit init (optimizer.cpp:80-82): U(0,1), scaled so ||M|| = ||X||."""
    rs = np.random.default_rng(seed)
    F = [rs.uniform(lo, hi, (n, rank)) for n in dims]
    if data_norm and data_norm > 0:
        ratio = (data_norm / model_norm(F)) ** (1.0 / len(dims))
        F = [f * ratio for f in F]
    return F


def zipf_indices(rs, n: int, a: float, size: int) -> np.ndarray:
    """P(i) ∝ (i+1)^-a on {0..n-1}, by inverse CDF."""
    w = 1.0 / np.arange(1, n + 1, dtype=np.float64) ** a
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    return np.searchsorted(cdf, rs.random(size), side="right").clip(0, n - 1)


def unique_first(keys: np.ndarray, target: int) -> np.ndarray:
    """First `target` distinct keys in generation order, returned sorted."""
    uniq, first = np.unique(keys, return_index=True)
    if len(uniq) < target:
        raise RuntimeError("not enough unique keys generated")
    order = np.argsort(first, kind="stable")[:target]
    return np.sort(uniq[order])


def sparse_keys(w: Workload, seed: int) -> np.ndarray:
    """Sorted unique u64 linear keys (first-mode-fastest) for C3/C4."""
    rs = np.random.default_rng(seed)
    strides = np.cumprod((1,) + w.dims[:-1]).astype(np.uint64)
    want = w.nnz
    gen = int(want * 1.6)
    while True:
        cols = []
        for k, n in enumerate(w.dims):
            if w.name == "c3":
                cols.append(zipf_indices(rs, n, 1.1, gen))
            elif w.name == "c4":
                cols.append(rs.integers(0, n, gen) if k < 2 else zipf_indices(rs, n, 1.2, gen))
            else:
                cols.append(zipf_indices(rs, n, 1.05, gen))
        keys = np.zeros(gen, dtype=np.uint64)
        for k in range(w.d):
            keys += cols[k].astype(np.uint64) * strides[k]
        try:
            return unique_first(keys, want)
        except RuntimeError:
            gen *= 2


def sparse_values(w: Workload, n: int, seed: int) -> np.ndarray:
    rs = np.random.default_rng(seed)
    if w.loss == "bernoulli-odds":
        return np.ones(n, dtype=np.float32)
    if w.name == "c4":
        return (1.0 + rs.poisson(2.0, n)).astype(np.float32)
    v = rs.poisson(3.0, n)
    v[v == 0] = 1  # condition on >= 1: no explicit zeros (tensor.cpp:35)
    return np.log1p(v).astype(np.float32)


def c5_device_data(w: Workload, seed: int = 1005, oversample: float = 1.36,
                   bucket_limit: int = 1_500_000_000, device=None):
    """C5 on the GPU (torch as ingest plumbing, off the hot path): per-mode
    Zipf(1.05) indices by inverse CDF, u64 linear keys, the first `nnz`
    distinct keys in generation order, returned sorted; values
    log(1 + Poisson(3)) conditioned on Poisson >= 1 (no explicit zeros,
    tensor.cpp:35).  Deduplication: candidate keys are split into key-range
    buckets of < bucket_limit elements (torch sorts < 2^31 elements; buckets
    never share a key), each bucket is stably sorted so the first element of a
    run of equal keys is its first occurrence, and the exact count is reached
    by bisection on the first-occurrence position."""
    import torch
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    target = w.nnz
    strides = [1]
    for n in w.dims[:-1]:
        strides.append(strides[-1] * n)
    cdfs = []
    for n in w.dims:
        wt = 1.0 / torch.arange(1, n + 1, dtype=torch.float64, device=dev) ** 1.05
        c = torch.cumsum(wt, 0)
        cdfs.append(c / c[-1])
    sign = torch.tensor(-(2 ** 63), dtype=torch.int64, device=dev)
    gen = int(target * oversample)
    while True:
        keys = torch.zeros(gen, dtype=torch.int64, device=dev)
        chunk = 1 << 27
        for b in range(0, gen, chunk):
            e = min(gen, b + chunk)
            for k, n in enumerate(w.dims):
                u = torch.rand(e - b, dtype=torch.float64, device=dev, generator=g)
                ik = torch.searchsorted(cdfs[k], u, right=True).clamp_(max=n - 1)
                keys[b:e] += ik * strides[k]  # wraps mod 2^64 (N > 2^63 for C5)
                del u, ik
        keys.bitwise_xor_(sign)  # u64 order as signed order
        nb = -(-gen // bucket_limit)
        if nb > 1:
            probe = keys[torch.randint(0, gen, (1 << 20,), device=dev, generator=g)]
            qs = torch.quantile(probe.to(torch.float64),
                                torch.linspace(0, 1, nb + 1, dtype=torch.float64, device=dev)[1:-1])
            pivots = [int(v) for v in qs.tolist()]
        else:
            pivots = []
        bounds = [None] + pivots + [None]
        uniqs, firsts = [], []
        for bi in range(len(bounds) - 1):
            m = torch.ones(gen, dtype=torch.bool, device=dev)
            if bounds[bi] is not None:
                m &= keys >= bounds[bi]
            if bounds[bi + 1] is not None:
                m &= keys < bounds[bi + 1]
            pos = torch.nonzero(m).squeeze(1)
            kb = keys[pos]
            del m
            sk, order = torch.sort(kb, stable=True)
            del kb
            pos = pos[order]
            del order
            st = torch.ones(sk.numel(), dtype=torch.bool, device=dev)
            st[1:] = sk[1:] != sk[:-1]
            uniqs.append(sk[st])
            firsts.append(pos[st])
            del sk, pos, st
        del keys
        uniq = torch.cat(uniqs)
        first = torch.cat(firsts)
        del uniqs, firsts
        if uniq.numel() >= target:
            break
        del uniq, first
        gen = int(gen * 1.3)
    lo, hi = 0, gen  # smallest T with count(first < T) == target
    while lo < hi:
        mid = (lo + hi) // 2
        if int((first < mid).sum()) >= target:
            hi = mid
        else:
            lo = mid + 1
    sel = uniq[first < lo]
    del uniq, first
    assert sel.numel() == target
    sel.bitwise_xor_(sign)  # back to the u64 bit pattern (still ascending as u64)
    lam = torch.full((target,), 3.0, dtype=torch.float32, device=dev)
    v = torch.poisson(lam, generator=g)
    del lam
    v.clamp_(min=1.0)
    vals = torch.log1p(v)
    del v
    return sel, vals
