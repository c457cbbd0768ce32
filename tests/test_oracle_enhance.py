"""Pins of the oracle's per-box enhancement (`ref_enhance`, O7b: crop extraction from the LR bins and
placement of SR(crop) into the HR bins, "stitch the real-content regions into tensors (bins)"),
of its multi-threaded entries, and of the MB-owner grid (reading D9/D13) when boxes stay unplaced.

The enhancement pins use networks whose weights make the SR a closed form:
* delta network: every conv an identity (or channel-fan-out) tap, the residual convs zero, so the
  whole EDSR / tiny model reduces to nearest-neighbour x s -> the HR bin must equal np.repeat of the
  crop at (s*bx, s*by), zero elsewhere;
* shift network: the tiny model's first conv reads the pixel to the right (tap (1, 2)), so the crop's
  last column sees the zero padding of the crop border (D8 isolation) and NOT the next box packed to
  its right in the same bin.
A wrong s*bx offset, a transposed (rotated) crop or a crop read across the bin neighbour fails one
of them."""
import numpy as np
import pytest

import oracle
import synth


def _delta_weights(cfg: synth.SRConfig, shift: bool = False) -> np.ndarray:
    """Flat fp64 weights (network order) reducing the model to nearest x s (see module doc)."""
    parts = []
    shapes = cfg.conv_shapes()
    n_up = 2 if (cfg.n_resblocks > 0 and cfg.scale == 4) else 1
    up_first = 1 + 2 * cfg.n_resblocks + 1
    for i, (ci, co) in enumerate(shapes):
        w = np.zeros((co, ci, 3, 3))
        b = np.zeros(co)
        if cfg.n_resblocks == 0:
            if i == 0:   # 3 -> C: copy RGB into channels 0..2 (optionally shifted by one pixel)
                for c in range(3):
                    w[c, c, 1, 2 if shift else 1] = 1.0
            else:        # C -> 3 s^2: fan channel c out to the s^2 sub-pixels of PixelShuffle(s)
                s = cfg.scale
                for c in range(3):
                    for j in range(s * s):
                        w[c * s * s + j, c, 1, 1] = 1.0
        else:
            if i == 0 or i == len(shapes) - 1:      # head 3->C, tail C->3: identity on RGB
                for c in range(3):
                    w[c, c, 1, 1] = 1.0
            elif up_first <= i < up_first + n_up:   # upsampler stage(s): fan-out for PixelShuffle
                ss = 2 if cfg.scale == 4 else cfg.scale
                for c in range(3):
                    for j in range(ss * ss):
                        w[c * ss * ss + j, c, 1, 1] = 1.0
            # residual convs and the body conv stay zero: r' = r, body = 0 + h (global skip)
        parts += [w.ravel(), b]
    return np.concatenate(parts)


def _scene(seed=0):
    """Three boxes in two 32x24 bins: box 0 unrotated at (1, 0); box 1 rotated, packed right after
    box 0's gutter in the same bin; box 2 unrotated in bin 1. LR bin values random in [0, 1)."""
    rng = np.random.default_rng(seed)
    bin_w, bin_h = 32, 24
    lr = rng.random((2, bin_h, bin_w, 3))
    bx = np.zeros((3, 12), np.int32)
    bx[:, 8:10] = [[11, 7], [5, 13], [9, 9]]   # w, h of each box (pixel box size)
    pl = np.array([[0, 1, 0, 0],               # footprint 11 x 7
                   [0, 13, 2, 1],              # rotated: footprint h x w = 13 wide, 5 tall
                   [1, 4, 6, 0]], np.int32)
    return lr, bx, pl, bin_w, bin_h


def _footprint(bx, pl, b):
    w, h = int(bx[b, 8]), int(bx[b, 9])
    return (h, w) if pl[b, 3] else (w, h)


@pytest.mark.parametrize("cfg", [synth.SRConfig(2, 8, 0, 1.0, False), synth.SRConfig(3, 8, 0, 1.0, False),
                                 synth.SRConfig(3, 8, 1, 1.0, False), synth.SRConfig(4, 8, 1, 1.0, False),
                                 synth.SRConfig(2, 4, 2, 0.5, False)])
def test_enhance_delta_network_is_nearest_upsampling_of_each_crop(cfg):
    lr, bx, pl, bw, bh = _scene()
    s = cfg.scale
    hr = oracle.enhance(cfg, _delta_weights(cfg), lr, bx, pl)
    expect = np.zeros_like(hr)
    for b in range(len(bx)):
        fw, fh = _footprint(bx, pl, b)
        bin_, x, y = pl[b, :3]
        crop = lr[bin_, y:y + fh, x:x + fw]
        expect[bin_, s * y:s * (y + fh), s * x:s * (x + fw)] = np.repeat(np.repeat(crop, s, 0), s, 1)
    np.testing.assert_allclose(hr, expect, rtol=0, atol=1e-15)


def test_enhance_crop_border_is_zero_padded_not_the_bin_neighbour():
    cfg = synth.SRConfig(2, 8, 0, 1.0, False)
    lr, bx, pl, bw, bh = _scene(1)
    hr = oracle.enhance(cfg, _delta_weights(cfg, shift=True), lr, bx, pl)
    s = 2
    for b in range(len(bx)):
        fw, fh = _footprint(bx, pl, b)
        bin_, x, y = pl[b, :3]
        crop = lr[bin_, y:y + fh, x:x + fw]
        shifted = np.zeros_like(crop)
        shifted[:, :-1] = crop[:, 1:]          # reads x+1; the last column sees the zero padding
        np.testing.assert_allclose(hr[bin_, s * y:s * (y + fh), s * x:s * (x + fw)],
                                   np.repeat(np.repeat(shifted, s, 0), s, 1), rtol=0, atol=1e-15)
    # box 0's right neighbour in bin 0 (box 1) is non-zero, so reading across the seam would show
    assert lr[0, 0:7, 12].any()


def test_enhance_box_range_and_unplaced_boxes():
    cfg = synth.SRConfig(3, 8, 0, 1.0, False)
    lr, bx, pl, bw, bh = _scene(2)
    w = _delta_weights(cfg)
    full = oracle.enhance(cfg, w, lr, bx, pl)
    part = oracle.enhance(cfg, w, lr, bx, pl, 1, 2)
    fw, fh = _footprint(bx, pl, 1)
    sl = (0, slice(3 * 2, 3 * (2 + fh)), slice(3 * 13, 3 * (13 + fw)))
    np.testing.assert_array_equal(part[sl], full[sl])
    part[sl] = 0
    assert not part.any()                     # only box 1 written
    pl2 = pl.copy()
    pl2[2, 0] = -1                            # unplaced: contributes nothing
    un = oracle.enhance(cfg, w, lr, bx, pl2)
    assert not un[1].any() and np.array_equal(un[0], full[0])


def test_enhance_and_scatter_multithreaded_are_bit_identical():
    wl = synth.small(synth.CONFIGS["c2"], F=2)
    cfg = synth.SRConfig(3, 8, 1, 1.0, True)
    imp = synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 3)
    fr = synth.frames_rgb8(wl.S, wl.F, wl.H, wl.W, 3)
    ip = oracle.index_path(imp, wl.W, wl.H, wl.k // 3, partition_mb=4, bin_w=128, bin_h=128, max_bins=64)
    lr = oracle.gather(fr, ip["boxes"], ip["placement"], 128, 128, ip["num_bins"], True)
    w64 = oracle.sr_weights_for(cfg, synth.sr_weights(cfg, 1))
    n = min(len(ip["boxes"]), 10)
    a = oracle.enhance(cfg, w64, lr, ip["boxes"], ip["placement"], 0, n)
    b = oracle.enhance(cfg, w64, lr, ip["boxes"], ip["placement"], 0, n, threads=4)
    assert np.array_equal(a, b)
    s1 = oracle.scatter(fr, ip["boxes"], ip["placement"], ip["owner"], a, 3, 128, 128)
    s4 = oracle.scatter(fr, ip["boxes"], ip["placement"], ip["owner"], a, 3, 128, 128, threads=3)
    assert np.array_equal(s1, s4)


def test_mb_owner_with_unplaced_boxes_matches_definition():
    """Reading D9/D13: owner[mb] = the box holding mb as a member if that box was placed, else -1.
    Checked against a direct re-derivation from labels, box spans and placements, with max_bins small
    enough that many boxes stay unplaced."""
    W, H = 320, 180
    GW, GH = synth.grid(W, H)
    imp = synth.importance_maps(2, 3, GH, GW, 5, "noisy")
    ip = oracle.index_path(imp, W, H, int(0.25 * imp.size), partition_mb=3, bin_w=64, bin_h=64, max_bins=3)
    pl = ip["placement"]
    assert (pl[:, 0] < 0).sum() > 5 and (pl[:, 0] >= 0).sum() > 5
    expect = np.full(ip["labels"].shape, -1, np.int32)
    covered = np.zeros(ip["labels"].shape, np.int32)
    for b, row in enumerate(ip["boxes"]):
        s, f, mx0, my0, mx1, my1 = (int(v) for v in row[:6])
        region = int(row[11])
        span = ip["labels"][s, f, my0:my1, mx0:mx1] == region
        covered[s, f, my0:my1, mx0:mx1] += span
        if pl[b, 0] >= 0:
            expect[s, f, my0:my1, mx0:mx1][span] = b
    np.testing.assert_array_equal(covered, (ip["labels"] >= 0).astype(np.int32))   # each member exactly once
    np.testing.assert_array_equal(ip["owner"], expect)
    assert (ip["owner"][ip["sel"] == 0] == -1).all()
