"""Pins of the oracle's packing-policy suite beside the guillotine reading: the literal
Alg. 2 InnerFree (maximal empty rectangle by the histogram-stack method, reading D14),
skyline bottom-left (D15) and first-fit shelves (D16). Pinned against brute force (every rectangle of
small grids; every skyline position), closed forms (identical squares), hand-worked instances and the
plan invariants shared with the guillotine packer. CPU only."""
import numpy as np
import pytest

import oracle
from test_oracle_index import _boxes_wh, _check_plan

POLICIES = [oracle.POLICY_MAXRECT, oracle.POLICY_SKYLINE, oracle.POLICY_SHELF]


def _brute_mer(occ):
    """Largest all-free rectangle by enumerating every rectangle (2-D prefix sums)."""
    H, W = occ.shape
    ps = np.zeros((H + 1, W + 1), np.int64)
    ps[1:, 1:] = np.cumsum(np.cumsum(occ != 0, 0), 1)
    best = 0
    for y0 in range(H):
        for y1 in range(y0 + 1, H + 1):
            for x0 in range(W):
                for x1 in range(x0 + 1, W + 1):
                    if ps[y1, x1] - ps[y0, x1] - ps[y1, x0] + ps[y0, x0] == 0:
                        best = max(best, (y1 - y0) * (x1 - x0))
    return best


@pytest.mark.parametrize("seed", range(12))
def test_max_empty_rect_is_the_largest_free_rectangle(seed):
    rng = np.random.default_rng(seed)
    H, W = int(rng.integers(1, 9)), int(rng.integers(1, 10))
    occ = (rng.random((H, W)) < [0.1, 0.3, 0.5][seed % 3]).astype(np.uint8)
    x, y, w, h = oracle.max_empty_rect(occ)
    assert w * h == _brute_mer(occ)
    if w * h:
        assert not occ[y:y + h, x:x + w].any()


def test_max_empty_rect_hand_examples():
    occ = np.zeros((5, 7), np.uint8)
    assert oracle.max_empty_rect(occ) == (0, 0, 7, 5)
    occ[:, 0] = 1                                       # a fresh bin: column 0 reserved
    assert oracle.max_empty_rect(occ) == (1, 0, 6, 5)
    occ[0:2, 1:4] = 1                                   # a 3x2 box at the top-left: right strip 3x5 vs bottom 6x3
    assert oracle.max_empty_rect(occ) == (1, 2, 6, 3)    # 18 > 15
    assert oracle.max_empty_rect(np.ones((3, 3), np.uint8)) == (0, 0, 0, 0)


def test_maxrect_first_fit_over_the_bins_maximal_empty_rectangles():
    """Replay: every placed box sits at the top-left of the maximal empty rectangle of its bin (taken
    just before it), fits it (unrotated preferred), and no earlier bin's rectangle admitted it."""
    rng = np.random.default_rng(7)
    W, H, g = 48, 40, 1
    n = 70
    bx = _boxes_wh([(int(rng.integers(2, 20)), int(rng.integers(2, 20))) for _ in range(n)])
    order = rng.permutation(n).astype(np.int32)
    pl, nb = oracle.pack(bx, order, W, H, 6, g, oracle.POLICY_MAXRECT)
    occ = np.zeros((6, H + g, W), np.uint8)
    occ[:, :, 0] = 1
    for i in order:
        pw, ph = int(bx[i, 8]) + g, int(bx[i, 9]) + g
        fits = lambda r: (r[2] >= pw and r[3] >= ph) or (r[2] >= ph and r[3] >= pw)  # noqa: E731
        b, x, y, rot = pl[i]
        for k in range(b if b >= 0 else 6):
            assert not fits(oracle.max_empty_rect(occ[k]))
        if b < 0:
            continue
        r = oracle.max_empty_rect(occ[b])
        assert fits(r) and (x, y) == (r[0], r[1]) and rot == (not (r[2] >= pw and r[3] >= ph))
        uw, uh = (ph, pw) if rot else (pw, ph)
        occ[b, y:y + uh, x:x + uw] = 1
    _check_plan(bx, pl, W, H, g, nb)


def test_skyline_hand_example():
    # bin 21 x 10 (+1 gutter row), footprints 6x4, 8x3, 7x5, 5x2: the first two side by side on the
    # floor (x 1..6, 7..14); the 7-wide one no longer fits the floor (15 + 7 > 21) and rests lowest on
    # the 8x3 box (y 3, leftmost x 7); the 5x2 one fits the floor at x 15
    bx = _boxes_wh([(5, 3), (7, 2), (6, 4), (4, 1)])
    order = np.arange(4, dtype=np.int32)
    pl, nb = oracle.pack(bx, order, 21, 10, 1, 1, oracle.POLICY_SKYLINE)
    assert pl.tolist() == [[0, 1, 0, 0], [0, 7, 0, 0], [0, 7, 3, 0], [0, 15, 0, 0]] and nb == 1


def test_skyline_position_is_the_lowest_then_leftmost():
    """Brute force over every x: the chosen y is the minimum of max(heights[x..x+w)) and x the leftmost."""
    rng = np.random.default_rng(4)
    W, H = 40, 30
    n = 60
    bx = _boxes_wh([(int(rng.integers(2, 12)), int(rng.integers(2, 12))) for _ in range(n)])
    order = np.arange(n, dtype=np.int32)
    pl, nb = oracle.pack(bx, order, W, H, 8, 1, oracle.POLICY_SKYLINE)
    heights = {}
    for i in order:
        b, x, y, rot = pl[i]
        if b < 0:
            continue
        hg = heights.setdefault(int(b), np.array([H + 1] + [0] * (W - 1)))
        w, h = int(bx[i, 8]) + 1, int(bx[i, 9]) + 1
        uw, uh = (h, w) if rot else (w, h)
        cand = [(int(hg[c:c + uw].max()), c) for c in range(1, W - uw + 1) if hg[c:c + uw].max() + uh <= H + 1]
        assert (y, x) == min(cand)
        if rot:   # rotated only when the unrotated footprint rests nowhere in this bin
            assert not [c for c in range(1, W - w + 1) if hg[c:c + w].max() + h <= H + 1]
        hg[x:x + uw] = y + uh
    _check_plan(bx, pl, W, H, 1, nb)


def test_shelf_hand_example():
    # bin 30 x 20 (+1), footprints 9x9, 8x7, 11x7, 13x6 in height order: shelf 0 (y 0, height 9) takes
    # the first three at x 1, 10, 18 (ends at 29); the 13-wide one fits neither way on shelf 0 and opens
    # shelf 1 at y 9
    bx = _boxes_wh([(8, 8), (7, 6), (10, 6), (12, 5)])
    order = oracle.sort(bx, np.zeros(4), oracle.ORDER_HEIGHT)
    assert order.tolist() == [0, 1, 2, 3]
    pl, nb = oracle.pack(bx, order, 30, 20, 1, 1, oracle.POLICY_SHELF)
    assert pl.tolist() == [[0, 1, 0, 0], [0, 10, 0, 0], [0, 18, 0, 0], [0, 1, 9, 0]] and nb == 1


@pytest.mark.parametrize("policy", [oracle.POLICY_SKYLINE, oracle.POLICY_SHELF])
@pytest.mark.parametrize("a", [1, 5, 8, 13, 20, 31, 40, 62])
@pytest.mark.parametrize("W,H", [(64, 64), (128, 128), (100, 37)])
def test_identical_squares_closed_form(policy, a, W, H):
    g, n = 1, 400
    bx = _boxes_wh([(a, a)] * n)
    pl, _ = oracle.pack(bx, np.arange(n, dtype=np.int32), W, H, 1, g, policy)
    assert int((pl[:, 0] >= 0).sum()) == min(n, ((W - 1) // (a + g)) * ((H + g) // (a + g)))


@pytest.mark.parametrize("policy", POLICIES)
@pytest.mark.parametrize("seed", range(15))
def test_policy_plan_invariants_random(policy, seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(1, 100))
    W, H = [(64, 64), (128, 128), (96, 50)][seed % 3]
    bx = _boxes_wh([(int(rng.integers(1, W)), int(rng.integers(1, H + 4))) for _ in range(n)])
    order = rng.permutation(n).astype(np.int32)
    max_bins = int(rng.integers(1, 10))
    pl, nb = oracle.pack(bx, order, W, H, max_bins, 1, policy)
    _check_plan(bx, pl, W, H, 1, max_bins)
    used = sorted(set(pl[pl[:, 0] >= 0, 0].tolist()))
    assert nb == (used[-1] + 1 if used else 0)
    for i in range(n):   # a box that fits an empty bin in neither orientation is never placed
        w, h = int(bx[i, 8]), int(bx[i, 9])
        if not ((w + 1 <= W - 1 and h + 1 <= H + 1) or (h + 1 <= W - 1 and w + 1 <= H + 1)):
            assert pl[i, 0] == -1
        elif max_bins > n:   # room for one fresh bin per box: every box that fits an empty bin is placed
            assert pl[i, 0] >= 0
