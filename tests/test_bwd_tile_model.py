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
