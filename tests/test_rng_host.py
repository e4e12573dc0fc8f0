"""The RngStream state the device generators consume (gcpb_rng_seed /
gcpb_rng_split, host-only) against the reference's RngStream
(rng.cpp:33-47): the first draw of a seeded stream and of split children."""
import pytest

M64 = (1 << 64) - 1
PHI = 0x9e3779b97f4a7c15


def mix64(z):
    z &= M64
    z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & M64
    z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & M64
    return z ^ (z >> 31)


@pytest.mark.parametrize("seed", [0, 1, 7, 12345, 2**63 + 5])
@pytest.mark.parametrize("label", [0, 3, 2**40])
def test_seed_and_split_match_reference(ref, seed, label):
    from paper_1906_01687_b200 import gcp as g
    r = g.RngStream(seed)
    assert r.counter == 0
    assert mix64(r.key + PHI) == ref.rng(seed).next_u64()
    c = r.split(label)
    assert mix64(c.key + PHI) == ref.rng(seed).split(label).next_u64()
