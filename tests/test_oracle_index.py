"""Pins of the oracle's index path (select, regions, boxes, sort, pack) against things other than
itself: brute-force definitions with library sorts, scipy's connected-component labelling, the
paper's/SPEC's worked numbers, closed forms and packing invariants. CPU only."""
import json
import math
import os

import numpy as np
import pytest
import scipy.ndimage as ndi

import oracle
import synth

HERE = os.path.dirname(os.path.abspath(__file__))


def _maps(kind, S=2, F=3, GH=12, GW=20, seed=1):
    return synth.importance_maps(S, F, GH, GW, seed, kind)


# ------------------------------------------------------------------------------------ select

def _brute_topk(imp, k):
    flat = imp.reshape(-1).astype(np.float64)
    ids = np.arange(flat.size)
    order = np.lexsort((ids, -flat))  # importance desc, id asc (reading D2)
    sel = np.zeros(flat.size, np.uint8)
    sel[order[:k]] = 1
    return sel.reshape(imp.shape)


@pytest.mark.parametrize("kind", ["blobs", "levels", "equal", "checker", "noisy"])
@pytest.mark.parametrize("k", [0, 1, 37, 480, 1440])
def test_select_topk_matches_full_sort(kind, k):
    imp = _maps(kind)
    sel = oracle.select(imp, 320, 180, oracle.MODE_TOPK, k)
    assert np.array_equal(sel, _brute_topk(imp, k))
    assert sel.sum() == min(k, imp.size)


def test_select_all_ties_take_lowest_ids():
    imp = np.full((1, 2, 3, 4), 0.25, np.float32)
    sel = oracle.select(imp, 64, 48, oracle.MODE_TOPK, 5)
    assert np.array_equal(np.flatnonzero(sel.reshape(-1)), np.arange(5))


def test_select_capacity_example_spec():
    # capacity floor(512*512*4/256) = 4096; 5000 random MBs -> sort-and-truncate
    cap = (512 * 512 * 4) // (16 * 16)
    assert cap == 4096
    rng = np.random.default_rng(5)
    imp = rng.random((1, 1, 50, 100), dtype=np.float32)  # 5000 MBs
    sel = oracle.select(imp, 1600, 800, oracle.MODE_TOPK, cap)
    assert np.array_equal(sel, _brute_topk(imp, cap))
    sel10 = oracle.select(imp[:, :, :1, :10], 160, 16, oracle.MODE_TOPK, cap)  # 10 MBs, all returned
    assert sel10.sum() == 10


def test_select_nan_lowest_and_signed_zero():
    imp = np.array([[[[0.0, -0.0, np.nan, -1.0, 2.0]]]], np.float32)
    # order: 2.0 (id4), 0.0 (id0) == -0.0 (id1) tie -> id0 first, then id1, then -1.0, NaN last
    assert np.flatnonzero(oracle.select(imp, 80, 16, 0, 1).reshape(-1)).tolist() == [4]
    assert np.flatnonzero(oracle.select(imp, 80, 16, 0, 2).reshape(-1)).tolist() == [0, 4]
    assert np.flatnonzero(oracle.select(imp, 80, 16, 0, 3).reshape(-1)).tolist() == [0, 1, 4]
    assert np.flatnonzero(oracle.select(imp, 80, 16, 0, 4).reshape(-1)).tolist() == [0, 1, 3, 4]


@pytest.mark.parametrize("cap", [-1, 0, 50])
def test_select_threshold(cap):
    imp = _maps("blobs")
    sel = oracle.select(imp, 320, 180, oracle.MODE_THRESHOLD, cap, tau=0.5)
    ref = (imp >= 0.5).astype(np.uint8)
    if cap >= 0:
        # cap by the same queue order: top-cap of the thresholded set
        masked = np.where(ref > 0, imp, -np.inf)
        ref = _brute_topk(masked, min(cap, int(ref.sum())))
    assert np.array_equal(sel, ref)


@pytest.mark.parametrize("k,cap", [(100, 40), (40, 100), (0, 5), (300, 0)])
def test_select_capacity_cap_topk(k, cap):
    # the capacity N bounds the selection on top of the configured k
    imp = _maps("levels")
    sel = oracle.select(imp, 320, 180, oracle.MODE_TOPK, k, cap=cap)
    assert np.array_equal(sel, _brute_topk(imp, min(k, cap)))


def test_select_capacity_cap_threshold_and_scope():
    imp = _maps("blobs")
    sel = oracle.select(imp, 320, 180, oracle.MODE_THRESHOLD, -1, tau=0.3, cap=25)
    masked = np.where(imp >= 0.3, imp, -np.inf)
    assert np.array_equal(sel, _brute_topk(masked, 25))
    sel = oracle.select(imp, 320, 180, oracle.MODE_TOPK, 30, scope=oracle.SCOPE_PER_FRAME, cap=7)
    for s in range(imp.shape[0]):
        for f in range(imp.shape[1]):
            assert np.array_equal(sel[s, f], _brute_topk(imp[s:s + 1, f:f + 1], 7)[0, 0])


@pytest.mark.parametrize("scope", [oracle.SCOPE_PER_STREAM, oracle.SCOPE_PER_FRAME])
def test_select_scopes(scope):
    imp = _maps("levels")
    k = 17
    sel = oracle.select(imp, 320, 180, oracle.MODE_TOPK, k, scope=scope)
    S, F = imp.shape[:2]
    if scope == oracle.SCOPE_PER_STREAM:
        for s in range(S):
            assert np.array_equal(sel[s], _brute_topk(imp[s:s + 1], k)[0])
    else:
        for s in range(S):
            for f in range(F):
                assert np.array_equal(sel[s, f], _brute_topk(imp[s:s + 1, f:f + 1], k)[0, 0])


# ------------------------------------------------------------------------------------ regions

def _scipy_labels(sel, conn):
    """Connected components by scipy, relabelled in (stream, frame, min raster index) order."""
    st = np.ones((3, 3), int) if conn == 8 else ndi.generate_binary_structure(2, 1)
    out = np.full(sel.shape, -1, np.int64)
    nxt = 0
    for s in range(sel.shape[0]):
        for f in range(sel.shape[1]):
            lab, n = ndi.label(sel[s, f], structure=st)
            firsts = sorted((np.flatnonzero(lab.reshape(-1) == i)[0], i) for i in range(1, n + 1))
            for _, i in firsts:
                out[s, f][lab == i] = nxt
                nxt += 1
    return out, nxt


@pytest.mark.parametrize("conn", [8, 4])
@pytest.mark.parametrize("kind", ["blobs", "noisy", "checker", "full"])
def test_regions_match_scipy(conn, kind):
    imp = _maps(kind, GH=23, GW=40)
    sel = oracle.select(imp, 640, 360, 0, int(0.25 * imp.size))
    if kind == "full":
        sel[:] = 1
    labels, regs = oracle.regions(sel, 640, 360, conn)
    ref, n = _scipy_labels(sel, conn)
    assert len(regs) == n
    assert np.array_equal(labels, ref)
    for r, rec in enumerate(regs):
        s, f, root, mx0, my0, mx1, my1, cnt = rec
        ys, xs = np.nonzero(labels[s, f] == r)
        assert (mx0, my0, mx1, my1, cnt) == (xs.min(), ys.min(), xs.max() + 1, ys.max() + 1, len(xs))
        assert root == np.flatnonzero(labels[s, f].reshape(-1) == r)[0]


def test_regions_spec_examples():
    # {(0,0),(0,1),(5,5)} -> 2 regions of 2 and 1; diagonal -> 2 under 4-conn
    sel = np.zeros((1, 1, 8, 8), np.uint8)
    sel[0, 0, 0, 0] = sel[0, 0, 1, 0] = sel[0, 0, 5, 5] = 1   # (x,y) = (0,0), (0,1), (5,5)
    _, regs = oracle.regions(sel, 128, 128, 4)
    assert sorted(regs[:, 7].tolist()) == [1, 2]
    diag = np.zeros((1, 1, 8, 8), np.uint8)
    diag[0, 0, 0, 0] = diag[0, 0, 1, 1] = 1
    assert len(oracle.regions(diag, 128, 128, 4)[1]) == 2
    assert len(oracle.regions(diag, 128, 128, 8)[1]) == 1


# ------------------------------------------------------------------------------------ boxes

def _one_region_boxes(cells, W=640, H=360, P=4, imp=None):
    GW, GH = synth.grid(W, H)
    sel = np.zeros((1, 1, GH, GW), np.uint8)
    for x, y in cells:
        sel[0, 0, y, x] = 1
    if imp is None:
        imp = np.ones((1, 1, GH, GW), np.float32)
    labels, regs = oracle.regions(sel, W, H, 8)
    return oracle.boxes(imp, labels, regs, W, H, 3, P), sel


def test_bound_spec_examples():
    # SPEC S:256-258 (x, y, w, h) with expand 3, frame 640x360
    (bx, _, _), _ = _one_region_boxes([(0, 0)])
    assert tuple(bx[0, 6:10]) == (0, 0, 19, 19)
    (bx, _, _), _ = _one_region_boxes([(2, 2)])
    assert tuple(bx[0, 6:10]) == (29, 29, 22, 22)
    (bx, _, _), _ = _one_region_boxes([(0, 0), (1, 0)])
    assert tuple(bx[0, 6:10]) == (0, 0, 35, 19)


def test_bound_partial_mb_clamped_to_frame():
    # 640x360: MB row 22 covers y 352..359 only (P:535 ceil reading) -> box bottom clamps at 360
    (bx, _, _), _ = _one_region_boxes([(39, 22)])
    x0, y0, w, h = bx[0, 6:10]
    assert (x0, y0, x0 + w, y0 + h) == (16 * 39 - 3, 16 * 22 - 3, 640, 360)


@pytest.mark.parametrize("width,pieces", [(4, [4]), (5, [3, 2]), (8, [4, 4]), (9, [3, 3, 3]), (10, [4, 3, 3]),
                                          (13, [4, 3, 3, 3])])
def test_partition_piece_sizes(width, pieces):
    # a straight row region `width` MBs wide at P=4 -> ceil(width/4) near-equal pieces, first ones larger
    (bx, _, _), _ = _one_region_boxes([(x, 5) for x in range(width)])
    assert [int(b[4] - b[2]) for b in bx] == pieces
    assert all(b[3] == 5 and b[5] == 6 for b in bx)


def test_partition_rebounds_to_members_and_drops_empty():
    # L-shaped region 8x8 at P=4: the top-right piece holds no members and is dropped
    cells = [(x, 0) for x in range(4)] + [(0, y) for y in range(8)] + [(x, 7) for x in range(8)]
    (bx, dens, own), sel = _one_region_boxes(cells)
    spans = sorted((int(b[2]), int(b[3]), int(b[4]), int(b[5])) for b in bx)
    assert spans == [(0, 0, 4, 4), (0, 4, 4, 8), (4, 7, 8, 8)]  # (4,4)-(8,8) re-bounded to row 7


@pytest.mark.parametrize("kind,P", [("blobs", 4), ("noisy", 2), ("full", 3), ("checker", 4)])
def test_boxes_partition_members_exactly_once(kind, P):
    imp = _maps(kind, S=1, F=2, GH=23, GW=40)
    sel = oracle.select(imp, 640, 360, 0, int(0.3 * imp.size))
    if kind == "full":
        sel[:] = 1
    labels, regs = oracle.regions(sel, 640, 360, 8)
    bx, dens, own = oracle.boxes(imp, labels, regs, 640, 360, 3, P)
    assert np.array_equal(own >= 0, sel > 0)                          # every selected MB owned once
    assert np.array_equal(np.bincount(own[own >= 0], minlength=len(bx)), bx[:, 10])
    for b, rec in enumerate(bx):
        s, f, mx0, my0, mx1, my1, x0, y0, w, h, cnt, r = rec
        assert 0 < mx1 - mx0 <= P and 0 < my1 - my0 <= P
        ys, xs = np.nonzero(own[s, f] == b)                           # re-bounded to its members
        assert (xs.min(), ys.min(), xs.max() + 1, ys.max() + 1) == (mx0, my0, mx1, my1)
        assert np.all(labels[s, f][ys, xs] == r)
        assert (x0, y0) == (max(0, 16 * mx0 - 3), max(0, 16 * my0 - 3))
        assert (x0 + w, y0 + h) == (min(640, 16 * mx1 + 3), min(360, 16 * my1 + 3))
        span = imp[s, f, my0:my1, mx0:mx1].astype(np.float64)
        assert math.isclose(dens[b], math.fsum(span.reshape(-1)) / span.size, rel_tol=1e-14)


def test_density_members_mode_is_mean_over_members():
    # P:691's set notation read as the member MBs of the box (REGEN_DENSITY_MEMBERS)
    imp = _maps("noisy", S=1, F=2, GH=23, GW=40)
    sel = oracle.select(imp, 640, 360, 0, int(0.3 * imp.size))
    labels, regs = oracle.regions(sel, 640, 360, 8)
    bx, dens, own = oracle.boxes(imp, labels, regs, 640, 360, 3, 3, density_mode=oracle.DENSITY_MEMBERS)
    bx0, dens0, own0 = oracle.boxes(imp, labels, regs, 640, 360, 3, 3)
    assert np.array_equal(bx, bx0) and np.array_equal(own, own0)
    differs = 0
    for b, rec in enumerate(bx):
        s, f = rec[0], rec[1]
        vals = imp[s, f][own[s, f] == b].astype(np.float64)
        assert len(vals) == rec[10]
        assert math.isclose(dens[b], math.fsum(vals) / len(vals), rel_tol=1e-14)
        differs += dens[b] != dens0[b]
    assert differs > 0     # boxes that bound unselected MBs get a different density


def test_region_ids_and_box_order_are_creation_order():
    imp = _maps("blobs", S=2, F=2, GH=23, GW=40)
    sel = oracle.select(imp, 640, 360, 0, int(0.2 * imp.size))
    labels, regs = oracle.regions(sel, 640, 360, 8)
    bx, _, _ = oracle.boxes(imp, labels, regs, 640, 360, 3, 4)
    keys = [(int(b[0]), int(b[1]), int(b[11])) for b in bx]
    assert keys == sorted(keys)


# ------------------------------------------------------------------------------------ sort

def test_sort_density_then_index_and_area_policy():
    rng = np.random.default_rng(3)
    n = 300
    dens = rng.integers(0, 20, n).astype(np.float64) / 7.0   # many ties
    bx = np.zeros((n, 12), np.int32)
    bx[:, 8] = rng.integers(1, 70, n)
    bx[:, 9] = rng.integers(1, 70, n)
    order = oracle.sort(bx, dens, oracle.ORDER_DENSITY)
    assert order.tolist() == sorted(range(n), key=lambda i: (-dens[i], i))
    order = oracle.sort(bx, dens, oracle.ORDER_AREA)
    assert order.tolist() == sorted(range(n), key=lambda i: (-int(bx[i, 8]) * int(bx[i, 9]), i))
    order = oracle.sort(bx, dens, oracle.ORDER_HEIGHT)
    assert order.tolist() == sorted(range(n), key=lambda i: (-int(bx[i, 9]), i))


# ------------------------------------------------------------------------------------ pack

def test_inner_free_spec_examples():
    # SPEC S:283-284 and S:285 corrected: vertical {12x10, 8x6} wins the 120-120 tie
    assert oracle.inner_free(16, 16, 10, 10) == [(10, 0, 6, 16), (0, 10, 10, 6)]
    assert oracle.inner_free(16, 16, 16, 16) == []
    assert oracle.inner_free(20, 10, 8, 4) == [(8, 0, 12, 10), (0, 4, 8, 6)]
    # horizontal wins when its larger remainder is strictly larger
    assert oracle.inner_free(16, 17, 10, 10) == [(0, 10, 16, 7), (10, 0, 6, 10)]


def _boxes_wh(whs):
    bx = np.zeros((len(whs), 12), np.int32)
    for i, (w, h) in enumerate(whs):
        bx[i, 8], bx[i, 9] = w, h
    return bx


def test_pack_spec_examples():
    # a 10x10 box in a 16x16 free area -> at the area's origin; 12x20 fits in neither orientation
    bx = _boxes_wh([(10, 10)])
    pl, nb = oracle.pack(bx, np.arange(1, dtype=np.int32), 17, 15, 1, 1)  # free area (1,0,16,16)
    assert pl[0].tolist() == [0, 1, 0, 0] and nb == 1
    bx = _boxes_wh([(12, 20)])
    pl, nb = oracle.pack(bx, np.arange(1, dtype=np.int32), 17, 15, 1, 1)
    assert pl[0, 0] == -1 and nb == 0


def test_pack_handworked_golden():
    g = json.load(open(os.path.join(HERE, "golden", "pack_handworked.json")))
    bx = _boxes_wh(g["boxes_wh_in_order"])
    pl, nb = oracle.pack(bx, np.arange(len(bx), dtype=np.int32), g["bin_w"], g["bin_h"], g["max_bins"], g["gutter"])
    assert pl.tolist() == g["expected_placement"] and nb == g["expected_num_bins"]


@pytest.mark.parametrize("a", [1, 5, 8, 13, 20, 31, 40, 62])
@pytest.mark.parametrize("W,H", [(64, 64), (128, 128), (100, 37)])
def test_pack_identical_squares_closed_form(a, W, H):
    # n identical a x a boxes with gutter g into one bin: floor((W-1)/(a+g)) * floor((H+g)/(a+g)) placed
    g = 1
    n = 400
    bx = _boxes_wh([(a, a)] * n)
    pl, _ = oracle.pack(bx, np.arange(n, dtype=np.int32), W, H, 1, g)
    assert int((pl[:, 0] >= 0).sum()) == min(n, ((W - 1) // (a + g)) * ((H + g) // (a + g)))


def _check_plan(bx, pl, W, H, g, nbins):
    foot = {}
    for i, (b, x, y, rot) in enumerate(pl):
        if b < 0:
            continue
        w, h = int(bx[i, 8]), int(bx[i, 9])
        fw, fh = (h, w) if rot else (w, h)
        assert 1 <= x and x + fw + g <= W and 0 <= y and y + fh + g <= H + g and b < nbins
        foot.setdefault(b, []).append((x, y, fw + g, fh + g))
    for b, rects in foot.items():
        occ = np.zeros((H + g, W), np.int32)
        for x, y, fw, fh in rects:
            occ[y:y + fh, x:x + fw] += 1
        assert occ.max() <= 1, "footprints overlap"
        assert occ[:, 0].max() == 0, "column 0 is reserved"


@pytest.mark.parametrize("seed", range(40))
def test_pack_invariants_random(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 120))
    W, H = [(64, 64), (128, 128), (96, 50)][seed % 3]
    bx = _boxes_wh([(int(rng.integers(1, W)), int(rng.integers(1, H + 4))) for _ in range(n)])
    order = rng.permutation(n).astype(np.int32)
    max_bins = int(rng.integers(1, 12))
    pl, nb = oracle.pack(bx, order, W, H, max_bins, 1)
    _check_plan(bx, pl, W, H, 1, max_bins)
    used = sorted(set(pl[pl[:, 0] >= 0, 0].tolist()))
    assert nb == (used[-1] + 1 if used else 0)
    for i in range(n):  # a box that fits an empty bin in neither orientation is never placed
        w, h = int(bx[i, 8]), int(bx[i, 9])
        if not ((w + 1 <= W - 1 and h + 1 <= H + 1) or (h + 1 <= W - 1 and w + 1 <= H + 1)):
            assert pl[i, 0] == -1
    # lazy bins: a box never opens bin b+1 if it fit in an empty bin b that stayed empty before it
    first_use = {}
    for oi, i in enumerate(order):
        if pl[i, 0] >= 0:
            first_use.setdefault(int(pl[i, 0]), oi)
    fu = [first_use[b] for b in sorted(first_use)]
    assert fu == sorted(fu)


def test_pack_density_beats_area_when_capacity_binds():
    # fig:Puzzle: a large low-density box vs two small high-density boxes, one bin
    W, H = 64, 64
    bx = _boxes_wh([(60, 60), (30, 30), (30, 30)])
    dens = np.array([0.2, 0.9, 0.8])
    imp_sum = dens * np.array([16, 4, 4])
    pl_d, _ = oracle.pack(bx, oracle.sort(bx, dens, oracle.ORDER_DENSITY), W, H, 1, 1)
    pl_a, _ = oracle.pack(bx, oracle.sort(bx, dens, oracle.ORDER_AREA), W, H, 1, 1)
    assert (pl_d[:, 0] >= 0).tolist() == [False, True, True]
    assert (pl_a[:, 0] >= 0).tolist() == [True, False, False]
    assert imp_sum[pl_d[:, 0] >= 0].sum() > imp_sum[pl_a[:, 0] >= 0].sum()
