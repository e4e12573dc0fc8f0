"""Measurement: ideal-LRU (Che approximation) L2 hit rate of the C5 pick launch's row touches from the
generated tensor's real per-mode row marginals, for several cache sizes (128-byte [A | G] lines; each
pick also brings one record line)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1906_01687_b200 import workloads as WL

w = WL.get("c5")
keys, vals = WL.c5_device_data(w)
del vals
k = keys  # u64 linear keys as int64 bit patterns (first mode fastest; N > 2^63 for C5)
ps = []
rem = k
n0, n1, n2 = w.dims
s01 = n0 * n1
hi = (rem >> 32) & 0xFFFFFFFF
lo = rem & 0xFFFFFFFF
# i2 = key // (n0 * n1) as an unsigned division: a float64 estimate from the two halves,
# corrected exactly with wrapped int64 arithmetic
kd = hi.to(torch.float64) * 4294967296.0 + lo.to(torch.float64)
i2 = torch.floor(kd / float(s01)).to(torch.int64)
r = rem - i2 * s01                          # wraps mod 2^64 consistently -> exact remainder +- s01
i2 = torch.where(r < 0, i2 - 1, i2); r = torch.where(r < 0, r + s01, r)
i2 = torch.where(r >= s01, i2 + 1, i2); r = torch.where(r >= s01, r - s01, r)
i1 = r // n0
i0 = r - i1 * n0
assert int(i0.min()) >= 0 and int(i0.max()) < n0 and int(i1.max()) < n1 and int(i2.max()) < n2 and int(i2.min()) >= 0
nnz = k.numel()
for idx, n in ((i0, n0), (i1, n1), (i2, n2)):
    c = torch.bincount(idx, minlength=n).to(torch.float64)
    ps.append(torch.sort(c / nnz, descending=True).values)
    print(f"mode of {n} rows: top row {float(ps[-1][0]):.4f}, top-32 {float(ps[-1][:32].sum()):.4f}, "
          f"top-1e4 {float(ps[-1][:10000].sum()):.4f}, top-1e5 {float(ps[-1][:100000].sum()):.4f}, "
          f"rows with >=1 nz {int((c > 0).sum())}")

def occ(T, rec):
    s = T if rec else 0.0
    for p in ps:
        s += float((1 - torch.exp(-p * T)).sum())
    return s

for mb in (16, 32, 45, 64, 90, 126):
    C = mb * (1 << 20) / 128
    for rec in (True, False):
        lo_, hi_ = 1.0, 1e10
        for _ in range(70):
            mid = (lo_ * hi_) ** 0.5
            if occ(mid, rec) > C: hi_ = mid
            else: lo_ = mid
        hits = [float((p * (1 - torch.exp(-p * lo_))).sum()) for p in ps]
        # the 32 hottest rows per mode are privatised but still read: they hit anyway
        print(f"LRU {mb:4d} MB, record lines {'in' if rec else 'out of'} the cache: window {lo_:.3g} picks, "
              f"row hit rates {hits[0]:.3f} {hits[1]:.3f} {hits[2]:.3f}, mean {sum(hits)/3:.3f}")
