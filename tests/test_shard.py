"""CPU: the rectangle partitioning of bench.py --strong (shard.rect_shard): for the BASELINE
configs at 1/2/4/8 GPUs the rectangles are disjoint, equal and cover every (batch, kv-head)
unit; slicing keeps ALiBi slopes aligned with the shard's q heads."""
import pytest
import torch

from paper_2412_05496_b200 import shard


@pytest.mark.parametrize("B,Hkv", [(4, 16), (1, 32), (2, 8), (64, 32)])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_rectangles_cover_units(B, Hkv, world):
    seen = {}
    sizes = set()
    for r in range(world):
        b0, b1, h0, h1 = shard.rect_shard(B, Hkv, world, r)
        sizes.add((b1 - b0) * (h1 - h0))
        for b in range(b0, b1):
            for h in range(h0, h1):
                assert (b, h) not in seen
                seen[(b, h)] = r
    assert len(seen) == B * Hkv and len(sizes) == 1


def test_unsplittable_raises():
    with pytest.raises(ValueError):
        shard.rect_shard(3, 1, 2, 0)


def test_slice_and_slopes():
    import paper_2412_05496_b200 as fa
    B, Hq, Hkv, L, D, G = 2, 8, 4, 4, 2, 2
    q = torch.arange(B * Hq * L * D).reshape(B, Hq, L, D)
    k = torch.arange(B * Hkv * L * D).reshape(B, Hkv, L, D)
    sh = shard.rect_shard(B, Hkv, 2, 1)  # kv heads 2..3 -> q heads 4..7
    qs, ks, vs, dos = shard.slice_job(q, k, k, q, G, sh)
    assert torch.equal(qs, q[:, 4:8]) and torch.equal(ks, k[:, 2:4]) and qs.is_contiguous()
    s = shard.shard_score(fa.alibi(fa.alibi_slopes(Hq)), G, sh)
    assert list(s.slopes) == fa.alibi_slopes(Hq)[4:8]
