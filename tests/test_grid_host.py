"""Host logic of levels x row shards (no GPU): the row split every rank of a
grid agrees on, and the neighbour list ridc_pipe_connect_shard expects."""

from paper_1209_4297_b200.distributed import shard_neighbours, shard_rows


def test_shard_rows_partition():
    for ny in (2, 7, 12, 37, 4096):
        for S in range(2, min(ny, 9) + 1):
            rows = [shard_rows(ny, s, S) for s in range(S)]
            assert rows[0][0] == 0 and rows[-1][1] == ny
            assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))   # contiguous, no gaps
            sizes = [r1 - r0 for r0, r1 in rows]
            assert min(sizes) >= 1 and max(sizes) - min(sizes) <= 1     # balanced


def test_shard_neighbours_order_and_wrap():
    # middle level, middle shard: every neighbour exists
    assert shard_neighbours(1, 1, 3, 3) == [(0, 1), (0, 0), (0, 2), (2, 1), (2, 0), (2, 2), (1, 0), (1, 2)]
    # shard 0 wraps to the last shard (y periodic); the lowest level has no producers
    assert shard_neighbours(0, 0, 4, 2) == [None, None, None, (1, 0), (1, 3), (1, 1), (0, 3), (0, 1)]
    # the top level has no consumers; with two shards both diagonals are the other shard
    assert shard_neighbours(1, 1, 2, 2) == [(0, 1), (0, 0), (0, 0), None, None, None, (1, 0), (1, 0)]


def test_every_link_has_a_matching_end():
    """A producer's delivery into (j+1, s-+1) must be that consumer's (j, s+-1) producer
    entry: the grid's links pair up."""
    L, S = 4, 3
    for j in range(L):
        for s in range(S):
            nb = shard_neighbours(j, s, S, L)
            if nb[4] is not None:   # I deliver my first row into (j+1, s-1)'s ghost row n+1 ...
                assert shard_neighbours(*nb[4], S, L)[2] == (j, s)   # ... whose (j, s+1) producer is me
            if nb[5] is not None:
                assert shard_neighbours(*nb[5], S, L)[1] == (j, s)
            assert shard_neighbours(*nb[6], S, L)[7] == (j, s)
