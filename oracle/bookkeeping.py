"""Integer bookkeeping oracle (KV paging, SWA ring, conv ring) — TEST INFRASTRUCTURE ONLY.

Restates, in plain Python, where every token's K/V and conv input must live so
the GPU layouts can be checked bit-exactly (SURVEY.md §4 items 2-3, §8a rows
a7/a11).  The paper fixes only the semantics: FA keeps a KV cache growing with
the context, SWA "attends only to the w most recent positions" (R/PAPER.md:1561),
GDN/KDA keep a short conv buffer (R/PAPER.md:834-843).  The slot functions
below are this runtime's pinned encoding of those semantics (include/sn_abi.h).
"""
from __future__ import annotations


def fa_slot(block_table_row, pos: int, page_size: int):
    """Paged FA cache: position p lives in page block_table[p // page] at offset p % page."""
    return block_table_row[pos // page_size], pos % page_size


def swa_slot(block_table_row, pos: int, window: int, page_size: int):
    """SWA ring: position p lives at ring slot p % w, i.e. page block_table[(p % w) // page]."""
    s = pos % window
    return block_table_row[s // page_size], s % page_size


def swa_attended(pos: int, window: int):
    """Positions a query at `pos` attends to: j in (pos - w, pos]."""
    return list(range(max(0, pos - window + 1), pos + 1))


def swa_ring_contents(length: int, window: int):
    """After `length` tokens, ring slot s holds the newest position p < length with p % w == s
    (or None if never written)."""
    out = [None] * window
    for p in range(length):
        out[p % window] = p
    return out


def conv_ring_slot(pos: int, width: int) -> int:
    """Conv ring: the input of position p lives at slot p % W; a decode step at
    position t reads slots (t-1..t-W+1) % W and writes slot t % W."""
    return pos % width


def conv_ring_contents(length: int, width: int):
    """Ring after `length` inputs (prefill of `length` tokens): slot s holds the newest position p
    in [length-W+1, length-1] with p % W == s, or None (zero) if that position is < 0 or the
    slot belongs to the next write."""
    out = [None] * width
    for d in range(1, width):
        p = length - d
        out[p % width] = p if p >= 0 else None
    return out
