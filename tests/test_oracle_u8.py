"""Pins of the oracle's u8 output (reading D20, SURVEY §8(c) "u8 output (clamp, round-half-even)")
against things other than itself: the fp64 O8 frames (pinned in test_oracle_pixels.py against
torch's F.interpolate) rounded by numpy's half-to-even `np.round`, hand-worked tie rows, constant
frames (a closed form) and the clamp at both ends."""
import numpy as np
import pytest

import oracle


def _bilinear_only(frames, scale):
    S, F, H, W = frames.shape[:4]
    owner = -np.ones((S, F, (H + 15) // 16, (W + 15) // 16), np.int32)
    hr64 = oracle.scatter(frames, np.zeros((0, 12), np.int32), np.zeros((0, 4), np.int32), owner,
                          np.zeros(0), scale, 16, 16)
    return owner, hr64, oracle.quantize_u8(frames, owner, hr64, scale)


@pytest.mark.parametrize("scale", [2, 3, 4])
def test_bilinear_codes_are_the_fp64_values_rounded_half_to_even(scale):
    rng = np.random.default_rng(scale)
    frames = rng.integers(0, 256, (1, 2, 32, 48, 3), dtype=np.uint8)
    _, hr64, q = _bilinear_only(frames, scale)
    x = hr64 * 255.0
    frac = x - np.floor(x)
    clear = np.abs(frac - 0.5) > 1e-9          # away from a tie the fp64 value decides unambiguously
    np.testing.assert_array_equal(q[clear], np.round(x[clear]).astype(np.uint8))
    tie = ~clear                               # exact ties (only for even s): the even neighbour
    if scale % 2 == 0:
        assert tie.sum() > 100, "random frames should produce exact .5 ties at even scales"
    else:
        assert tie.sum() == 0, "odd s cannot tie: the weight numerators 2j+1-s are even, so 255 v = M / s^2"
    lo = np.floor(x[tie]).astype(np.int64)
    np.testing.assert_array_equal(q[tie].astype(np.int64), np.where(lo % 2 == 0, lo, lo + 1))


def test_hand_worked_tie_row():
    """s = 2, LR row (0, 2, 0, 2, ...): HR column X samples (X + 0.5)/2 - 0.5. X = 1 -> 0.25 between
    codes 0 and 2 -> 0.5 (tie -> 0); X = 2 -> 0.75 -> 1.5 (tie -> 2); X = 0 clamps to column 0 -> 0;
    X = 3 -> 1.25 between 2 and 0 -> 1.5 -> 2; X = 4 -> 1.75 -> 0.5 -> 0."""
    W = 16
    row = np.tile(np.array([0, 2], np.uint8), W // 2)
    frames = np.repeat(row[None, None, None, :, None], 16, axis=2).repeat(3, axis=4)   # [1][1][16][16][3]
    _, _, q = _bilinear_only(frames, 2)
    np.testing.assert_array_equal(q[0, 5, :6, 0], [0, 0, 2, 2, 0, 0])
    # and the last HR column clamps to the last LR column (code 2)
    assert q[0, 5, -1, 0] == 2


def test_constant_frames_give_the_constant_code():
    frames = np.full((1, 1, 16, 32, 3), 77, np.uint8)
    for s in (2, 3, 4):
        _, _, q = _bilinear_only(frames, s)
        assert (q == 77).all()


def test_pasted_pixels_clamp_and_round_half_to_even():
    S, F, H, W, s = 1, 1, 16, 16, 2
    owner = np.zeros((S, F, 1, 1), np.int32)          # the one MB is owned: every pixel is pasted
    frames = np.zeros((S, F, H, W, 3), np.uint8)
    vals = np.array([-0.3, 1.7, 0.5, 0.25, 1.0, 0.0, 2.5 / 255.0, 100.2 / 255.0, np.nextafter(0.5, 1.0)])
    hr = np.zeros((1, s * H, s * W, 3))
    hr.reshape(-1)[:len(vals)] = vals
    q = oracle.quantize_u8(frames, owner, hr, s).reshape(-1)[:len(vals)]
    # 0.5*255 = 127.5 exactly: tie -> 128 (even); 0.25*255 = 63.75 -> 64; 2.5/255*255 rounds to 2.5
    # in fp64 (tie -> 2) unless the product is inexact, which np.round then decides the same way
    exp = np.round(np.clip(vals, 0.0, 1.0) * 255.0).astype(np.uint8)
    np.testing.assert_array_equal(q, exp)
    np.testing.assert_array_equal(q[:6], [0, 255, 128, 64, 255, 0])
    assert q[7] == 100 and q[8] == 128
