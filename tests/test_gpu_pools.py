"""Stream ordering of the HBM memory pool (pools.py): a block returned on
one stream while a kernel there still reads it, then handed out on another
stream, is not overwritten before that kernel ran."""
import pytest

pytestmark = pytest.mark.gpu


def test_block_reuse_across_streams_waits_for_the_old_stream():
    import torch

    from paper_2503_22227_b200.pools import MemoryPool

    pool = MemoryPool(1, unit_mb=16, cap_mb=16)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    nbytes = 1 << 20
    with torch.cuda.stream(s1):
        h = pool.ask(nbytes)
        blk = h.words()
        blk.fill_(7)
        out = torch.empty_like(blk)
        torch.cuda._sleep(100_000_000)  # s1 stays busy for tens of ms
        out.copy_(blk)                  # the last reader of the block
        pool.ret(h)                     # returned while s1 still runs
    with torch.cuda.stream(s2):
        h2 = pool.ask(nbytes)
        assert (h2.origin, h2.offset) == (h.origin, h.offset)  # the same block
        h2.words().fill_(9)             # must run after s1's copy
    torch.cuda.synchronize()
    assert bool((out == 7).all())
    assert bool((h2.words() == 9).all())


def test_same_stream_reuse_needs_no_wait():
    import torch

    from paper_2503_22227_b200.pools import MemoryPool

    pool = MemoryPool(1, unit_mb=16, cap_mb=16)
    h = pool.ask(4096)
    h.words().fill_(1)
    pool.ret(h)
    h2 = pool.ask(4096)
    assert h2.offset == h.offset
    h2.words().fill_(2)
    torch.cuda.synchronize()
    assert bool((h2.words() == 2).all())
