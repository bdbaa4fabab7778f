"""Host logic: which grid shapes the device crowd accepts (A* key packing,
astar.cuh make_key2 / key_col_bits) and BatchedEnv's per-slot views."""

import pytest


def test_key_col_bits():
    from paper_2505_00690_b200.crowd import key_col_bits
    assert key_col_bits(256, 256) == 10
    assert key_col_bits(1024, 1024) == 10
    assert key_col_bits(1200, 100) == 11          # Traverse preset strip (presets.py:50-60)
    assert key_col_bits(100, 1200) == 7           # row gets 13 bits
    assert key_col_bits(2000, 300) == 11


def test_check_grid_shape():
    from paper_2505_00690_b200.crowd import check_grid_shape
    for nx, ny in ((256, 256), (512, 512), (1024, 1024), (1200, 100), (100, 1200), (1500, 60),
                   (1800, 400)):
        check_grid_shape(nx, ny)
    for nx, ny in ((1025, 1024), (2048, 1024), (2100, 10), (10, 2100), (1800, 600)):
        with pytest.raises(NotImplementedError):
            check_grid_shape(nx, ny)


def test_slot_seq():
    from paper_2505_00690_b200.envcore import _SlotSeq
    q = _SlotSeq(3, lambda i: i * 10)
    assert len(q) == 3 and q[0] == 0 and q[-1] == 20 and list(q) == [0, 10, 20] and q[1:] == [10, 20]
    with pytest.raises(IndexError):
        q[3]
