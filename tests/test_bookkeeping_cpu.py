"""Integer bookkeeping (bit-exact): KV page slots, SWA ring, conv ring, split-KV plan."""
import pytest

from oracle import bookkeeping as bk
from paper_2604_19877_b200.dist import shard_batch
from paper_2604_19877_b200.model import choose_split


def test_fa_slots_page_boundaries():
    bt = [7, 3, 9]
    assert [bk.fa_slot(bt, p, 64) for p in (0, 63, 64, 127, 128)] == [(7, 0), (7, 63), (3, 0), (3, 63), (9, 0)]


def test_swa_ring_wraps():
    bt = [5, 2]  # window 128, page 64
    assert bk.swa_slot(bt, 0, 128, 64) == (5, 0)
    assert bk.swa_slot(bt, 127, 128, 64) == (2, 63)
    assert bk.swa_slot(bt, 128, 128, 64) == (5, 0)
    assert bk.swa_slot(bt, 200, 128, 64) == (2, 8)
    ring = bk.swa_ring_contents(300, 128)
    assert sorted(ring) == list(range(300 - 128, 300))  # exactly the live window
    assert bk.swa_attended(300, 128) == list(range(173, 301))
    assert bk.swa_attended(5, 128) == list(range(0, 6))


def test_conv_ring():
    assert bk.conv_ring_contents(2, 4) == [0, 1, None, None]
    c = bk.conv_ring_contents(10, 4)
    assert c[bk.conv_ring_slot(9, 4)] == 9 and c[bk.conv_ring_slot(8, 4)] == 8 and c[bk.conv_ring_slot(7, 4)] == 7
    assert c[bk.conv_ring_slot(10, 4)] is None  # the next write's slot


@pytest.mark.parametrize("pages,rows", [(1, 1), (64, 512), (513, 184), (9, 1)])
def test_choose_split(pages, rows):
    sp, ms = choose_split(pages, rows)
    assert sp >= 1 and ms * sp >= pages and (ms - 1) * sp < pages


@pytest.mark.parametrize("B,W", [(64, 8), (7, 3), (3, 8)])
def test_shard_batch_partition(B, W):
    spans = [shard_batch(B, W, r) for r in range(W)]
    assert sum(c for _, c in spans) == B
    assert [s for s, _ in spans] == [sum(c for _, c in spans[:r]) for r in range(W)]
    assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
