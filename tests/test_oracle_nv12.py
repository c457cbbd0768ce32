"""Pins of the oracle's NV12 -> RGB8 conversion (reading D19: BT.601 limited range,
8-bit integer form, nearest chroma) against the BT.601 definition itself: the inverse of the forward
Y'CbCr matrix (Kr = 0.299, Kb = 0.114, 219/224 quantisation levels) computed by numpy.linalg.inv, the
reference colours of the limited range, and the NV12 plane layout (a known 2x2-block chroma image
round-trips to its colours). CPU only."""
import numpy as np

import oracle

KR, KB = 0.299, 0.114
KG = 1.0 - KR - KB


def _forward():
    """BT.601 R'G'B' in [0, 255] -> limited-range Y'CbCr offsets (Y-16, Cb-128, Cr-128)."""
    y = np.array([KR, KG, KB]) * 219.0 / 255.0
    cb = (np.array([0.0, 0.0, 1.0]) - np.array([KR, KG, KB])) / (2 * (1 - KB)) * 224.0 / 255.0
    cr = (np.array([1.0, 0.0, 0.0]) - np.array([KR, KG, KB])) / (2 * (1 - KR)) * 224.0 / 255.0
    return np.stack([y, cb, cr])


def _nv12(Y, U, V):
    """One frame from full-res Y [H][W] and quarter-res U, V [H/2][W/2]."""
    H, W = Y.shape
    uv = np.stack([U, V], -1).reshape(H // 2, W)
    return np.concatenate([Y.reshape(-1), uv.reshape(-1)]).astype(np.uint8)


def test_reference_colours():
    H, W = 2, 4
    for (y, u, v), rgb in [((16, 128, 128), (0, 0, 0)), ((235, 128, 128), (255, 255, 255)),
                           ((126, 128, 128), (128, 128, 128))]:
        out = oracle.nv12_to_rgb8(_nv12(np.full((H, W), y), np.full((1, 2), u), np.full((1, 2), v)), W, H)
        assert (out.reshape(-1, 3) == rgb).all(), ((y, u, v), out.reshape(-1, 3)[0])


def test_matches_the_inverse_bt601_matrix_within_one_level():
    inv = np.linalg.inv(_forward())                      # (Y-16, Cb-128, Cr-128) -> R'G'B'
    rng = np.random.default_rng(0)
    n = 4000
    yuv = np.stack([rng.integers(16, 236, n), rng.integers(16, 241, n), rng.integers(16, 241, n)], 1)
    H, W = 2, 2
    frames = np.stack([_nv12(np.full((H, W), a), np.full((1, 1), b), np.full((1, 1), c)) for a, b, c in yuv])
    got = oracle.nv12_to_rgb8(frames, W, H)[:, 0, 0].astype(np.int64)
    exact = (yuv - [16, 128, 128]) @ inv.T
    ref = np.clip(np.rint(exact), 0, 255)
    assert np.abs(got - ref).max() <= 1                 # the 8-bit integer form's rounding error


def test_chroma_layout_round_trip():
    """A known RGB image with constant colour per 2x2 block -> forward BT.601 -> NV12 -> oracle: the
    colours come back within 2 levels; swapping U/V or the chroma index would not."""
    rng = np.random.default_rng(1)
    H, W = 6, 8
    blocks = rng.integers(40, 216, size=(H // 2, W // 2, 3))
    rgb = np.repeat(np.repeat(blocks, 2, 0), 2, 1)
    ycc = rgb.astype(np.float64) @ _forward().T + [16, 128, 128]
    Y = np.rint(ycc[..., 0]).astype(np.uint8)
    U = np.rint(ycc[::2, ::2, 1]).astype(np.uint8)
    V = np.rint(ycc[::2, ::2, 2]).astype(np.uint8)
    out = oracle.nv12_to_rgb8(_nv12(Y, U, V), W, H).astype(np.int64)
    assert np.abs(out - rgb).max() <= 2
    swapped = oracle.nv12_to_rgb8(_nv12(Y, V, U), W, H).astype(np.int64)
    assert np.abs(swapped - rgb).max() > 10
