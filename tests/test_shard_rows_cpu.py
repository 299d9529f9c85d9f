"""The library's row partition (wgp_shard_rows, host only): every rank count
covers [0, n) with disjoint contiguous blocks of whole 128-row tiles, and the
vector leading dimension holds nranks equal blocks (the in-place all-gather
layout)."""
import pytest

import paper_2405_18328_b200 as wg


@pytest.mark.parametrize("n", [1, 127, 128, 129, 300, 2048, 41157, 391386, 1844352])
@pytest.mark.parametrize("nranks", [1, 2, 3, 4, 8])
def test_partition(n, nranks):
    parts = [wg.shard_rows(n, r, nranks) for r in range(nranks)]
    ld = parts[0][2]
    assert all(p[2] == ld for p in parts)
    assert ld >= -(-n // 128) * 128 and ld % nranks == 0
    blk = ld // nranks if nranks > 1 else ld
    covered = 0
    for r, (a, b, _) in enumerate(parts):
        assert a == min(n, r * blk) if nranks > 1 else a == 0
        assert a <= b and (a == b or a % 128 == 0)
        assert a == covered or a == b
        covered = max(covered, b)
    assert covered == n
    assert parts[0][1] - parts[0][0] == min(n, blk)


def test_bad_arguments():
    with pytest.raises(ValueError):
        wg.shard_rows(10, 2, 2)
    with pytest.raises(ValueError):
        wg.shard_rows(0, 0, 1)
