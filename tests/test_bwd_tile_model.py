"""Model of k_bwd_tile's work partition (csrc/k_train.cu), on the CPU.

The tiled backward cuts each table's sorted occurrence list into fixed tiles
of TR rows.  Inside a tile a row's occurrences form a segment; a segment that
is the whole row is finished by the tile, otherwise the tile leaves a piece in
slot 0 (the row holds the tile's first occurrence) or slot 1 (the row starts
inside the tile and runs past it), and the row's last arriving piece folds
the pieces of tiles kf..kl.  The rules below are the kernel's, written with
numpy: every occurrence must be summed exactly once, no two pieces may share a
(tile, slot), and every unique row must be finished exactly once -- for Zipf
heads spanning many tiles, tiles holding one row only, rows starting exactly
at a tile edge and a ragged last tile.
"""
import numpy as np
import pytest


def _partition(uid, TR):
    n = len(uid)
    U = int(uid.max()) + 1
    seg_off = np.searchsorted(uid, np.arange(U + 1))
    NT = (n + TR - 1) // TR
    whole_rows, pieces = [], {}
    for k in range(NT):
        lo = k * TR
        u = uid[lo:lo + TR]
        nact = len(u)
        prev = uid[lo - 1] if lo > 0 else -1
        nxt = uid[lo + nact] if lo + nact < n else -1
        prevu = np.concatenate([[prev], u[:-1]])
        nextu = np.concatenate([u[1:], [nxt]])
        first = prevu != u
        last = nextu != u
        last[nact - 1] = True                      # a segment ends at the tile's edge
        tail_open = nextu[nact - 1] == u[nact - 1]
        whole = first & ~((u == u[nact - 1]) & tail_open)
        r0 = 0
        for r1 in np.nonzero(last)[0]:
            row = int(u[r0])
            occ = list(range(lo + r0, lo + r1 + 1))
            if whole[r0]:
                whole_rows.append((row, occ))
            else:
                slo = seg_off[row]
                kf = slo // TR
                ps = 1 if (k == kf and slo != kf * TR) else 0
                assert (k, ps) not in pieces, (k, ps)
                pieces[(k, ps)] = (row, occ)
            r0 = r1 + 1
    return seg_off, whole_rows, pieces


@pytest.mark.parametrize("n,R,alpha,TR", [(4096, 3, 1.05, 32), (4096, 40_000_000, 1.05, 32),
                                          (20_000, 2000, 0.8, 32), (5000, 1000, 1.2, 7),
                                          (1000, 1, 1.0, 32), (33, 5, 1.0, 32), (64, 64, 0.0, 32)])
def test_every_occurrence_once_and_pieces_disjoint(n, R, alpha, TR):
    rng = np.random.default_rng(n + R)
    p = 1.0 / np.arange(1, R + 1) ** alpha
    p /= p.sum()
    ids = np.sort(rng.choice(R, size=n, p=p))
    _, uid = np.unique(ids, return_inverse=True)
    seg_off, whole_rows, pieces = _partition(uid, TR)
    U = len(seg_off) - 1
    seen = np.zeros(n, int)
    finished = np.zeros(U, int)
    for row, occ in whole_rows:
        seen[occ] += 1
        finished[row] += 1
        assert occ == list(range(seg_off[row], seg_off[row + 1]))   # the whole row, in order
    for row in range(U):   # the last arriver's fold over tiles kf..kl
        kf, kl = seg_off[row] // TR, (seg_off[row + 1] - 1) // TR
        if kf == kl:
            continue
        got = []
        for kk in range(kf, kl + 1):
            ps = 1 if (kk == kf and seg_off[row] != kf * TR) else 0
            prow, occ = pieces.pop((kk, ps))
            assert prow == row
            got += occ
        assert got == list(range(seg_off[row], seg_off[row + 1]))   # pieces in tile order = occurrence order
        seen[got] += 1
        finished[row] += 1
    assert not pieces                     # no orphan piece
    assert (seen == 1).all() and (finished == 1).all()


def _owners(uid, TR):
    """k_bwd_rows' owner rule: tile k owns the row at its tail iff that row
    continues past the tile's end and starts inside the tile (seg_off >= lo)."""
    n = len(uid)
    seg_off = np.searchsorted(uid, np.arange(int(uid.max()) + 2))
    NT = (n + TR - 1) // TR
    own = {}
    for k in range(NT):
        lo, nrows = k * TR, min(TR, n - k * TR)
        if lo + nrows >= n:
            continue
        u, un = uid[lo + nrows - 1], uid[lo + nrows]
        if u == un and seg_off[u] >= lo:
            assert u not in own
            own[int(u)] = (k, (seg_off[u + 1] - 1) // TR)
    return seg_off, own


@pytest.mark.parametrize("n,R,alpha,TR", [(4096, 3, 1.05, 16), (4096, 40_000_000, 1.05, 16),
                                          (20_000, 2000, 0.8, 32), (5000, 1000, 1.2, 7),
                                          (1000, 1, 1.0, 32), (33, 5, 1.0, 32), (64, 64, 0.0, 32)])
def test_two_phase_owner_finishes_every_spanning_row_once(n, R, alpha, TR):
    """Two-phase backward: every row spanning tiles [kf, kl] has exactly one
    owner, its first tile kf, which folds the pieces of kf..kl; rows inside
    one tile have none (k_bwd_tile finishes them)."""
    rng = np.random.default_rng(n * 7 + R)
    p = 1.0 / np.arange(1, R + 1) ** alpha
    p /= p.sum()
    ids = np.sort(rng.choice(R, size=n, p=p))
    _, uid = np.unique(ids, return_inverse=True)
    seg_off, own = _owners(uid, TR)
    _, _, pieces = _partition(uid, TR)
    for row in range(len(seg_off) - 1):
        kf, kl = seg_off[row] // TR, (seg_off[row + 1] - 1) // TR
        if kf == kl:
            assert row not in own
        else:
            assert own[row] == (kf, kl)
            for kk in range(kf, kl + 1):   # the pieces it folds exist and are this row's
                ps = 1 if (kk == kf and seg_off[row] != kf * TR) else 0
                assert pieces.pop((kk, ps))[0] == row
    assert not pieces
