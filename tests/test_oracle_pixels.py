"""Pins of the oracle's pixel path (gather, SR, scatter) against torch fp64 library routines,
closed forms and round-trip identities. CPU only."""
import numpy as np
import pytest
import torch
import torch.nn.functional as Fnn

import oracle
import synth


def test_input_quantisation_all_256_values():
    # reading D9: v = u8/255 in fp32, rounded to bf16 for the bf16 path
    u = torch.arange(256, dtype=torch.float32)
    v32 = u / 255.0
    v16 = v32.to(torch.bfloat16).to(torch.float64)
    for i in range(256):
        assert oracle.input_value(i, False) == float(v32[i])
        assert oracle.input_value(i, True) == float(v16[i])


def test_round_bf16_matches_torch():
    x = np.random.default_rng(0).standard_normal(10000).astype(np.float32) * 3
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(oracle.round_bf16(x), ref)


@pytest.mark.parametrize("cin,cout,h,w", [(3, 8, 7, 5), (16, 12, 9, 11), (5, 3, 1, 1), (4, 4, 1, 6)])
def test_conv3x3_matches_torch(cin, cout, h, w):
    rng = np.random.default_rng(cin * 100 + cout)
    x = rng.standard_normal((cin, h, w))
    wt = rng.standard_normal((cout, cin, 3, 3))
    b = rng.standard_normal(cout)
    ref = Fnn.conv2d(torch.from_numpy(x)[None], torch.from_numpy(wt), torch.from_numpy(b), padding=1)[0].numpy()
    np.testing.assert_allclose(oracle.conv3x3(x, wt, b), ref, rtol=1e-12, atol=1e-12)


def test_conv3x3_delta_kernel_is_identity():
    x = np.random.default_rng(1).standard_normal((3, 6, 9))
    wt = np.zeros((3, 3, 3, 3))
    for c in range(3):
        wt[c, c, 1, 1] = 1.0
    assert np.array_equal(oracle.conv3x3(x, wt, np.zeros(3)), x)


@pytest.mark.parametrize("s", [2, 3, 4])
def test_pixel_shuffle_matches_torch(s):
    x = np.random.default_rng(s).standard_normal((5 * s * s, 4, 7))
    ref = torch.pixel_shuffle(torch.from_numpy(x)[None], s)[0].numpy()
    assert np.array_equal(oracle.pixel_shuffle(x, s), ref)


def _torch_sr(cfg, w64, crop):
    """The network of reading D11 composed from torch fp64 library ops (independent of the C loops)."""
    x = torch.from_numpy(crop)[None]
    off = 0
    params = []
    for ci, co in cfg.conv_shapes():
        wt = torch.from_numpy(w64[off: off + co * ci * 9].reshape(co, ci, 3, 3))
        off += co * ci * 9
        b = torch.from_numpy(w64[off: off + co])
        off += co
        params.append((wt, b))
    conv = lambda t, p: Fnn.conv2d(t, p[0], p[1], padding=1)
    if cfg.n_resblocks == 0:
        return torch.pixel_shuffle(conv(torch.relu(conv(x, params[0])), params[1]), cfg.scale)[0].numpy()
    h = conv(x, params[0])
    r = h
    i = 1
    for _ in range(cfg.n_resblocks):
        t = torch.relu(conv(r, params[i]))
        r = r + cfg.res_scale * conv(t, params[i + 1])
        i += 2
    u = conv(r, params[i]) + h
    i += 1
    for _ in range(2 if cfg.scale == 4 else 1):
        u = torch.pixel_shuffle(conv(u, params[i]), 2 if cfg.scale == 4 else cfg.scale)
        i += 1
    return conv(u, params[i])[0].numpy()


@pytest.mark.parametrize("cfg", [synth.SRConfig(2, 16, 0, 1.0, False), synth.SRConfig(3, 8, 2, 1.0, True),
                                 synth.SRConfig(2, 8, 1, 0.5, True), synth.SRConfig(4, 4, 1, 1.0, False)])
def test_sr_crop_matches_torch_composition(cfg):
    w = synth.sr_weights(cfg, 7)
    w64 = oracle.sr_weights_for(cfg, w)
    crop = np.random.default_rng(2).random((3, 9, 13))
    np.testing.assert_allclose(oracle.sr_crop(cfg, w64, crop), _torch_sr(cfg, w64, crop), rtol=1e-10, atol=1e-12)


def test_sr_weights_bf16_rounding_only_weights():
    cfg = synth.SRConfig(2, 16, 0, 1.0, True)
    w = synth.sr_weights(cfg, 0)
    w64 = oracle.sr_weights_for(cfg, w)
    n0 = 16 * 3 * 9
    assert np.array_equal(w64[:n0], oracle.round_bf16(w[:n0]).astype(np.float64))
    assert np.array_equal(w64[n0:n0 + 16], w[n0:n0 + 16].astype(np.float64))  # bias untouched


def test_scatter_without_selection_is_torch_bilinear():
    # reading D10: bilinear = F.interpolate(align_corners=False), fp64
    fr = synth.frames_rgb8(1, 2, 20, 28, 3)
    for s in (2, 3, 4):
        own = np.full((1, 2, 2, 2), -1, np.int32)
        out = oracle.scatter(fr, np.zeros((0, 12), np.int32), np.zeros((0, 4), np.int32), own,
                             np.zeros((1, 1, 1, 3)), s, 8, 8)
        x = torch.from_numpy(fr[0].astype(np.float64) / 255.0).permute(0, 3, 1, 2)
        ref = Fnn.interpolate(x, scale_factor=s, mode="bilinear", align_corners=False).permute(0, 2, 3, 1).numpy()
        np.testing.assert_allclose(out, ref, rtol=0, atol=1e-12)


def test_scatter_constant_image_stays_constant():
    fr = np.full((1, 1, 17, 23, 3), 77, np.uint8)
    own = np.full((1, 1, 2, 2), -1, np.int32)
    out = oracle.scatter(fr, np.zeros((0, 12), np.int32), np.zeros((0, 4), np.int32), own, np.zeros(1), 3, 8, 8)
    np.testing.assert_allclose(out, 77 / 255.0, rtol=0, atol=1e-15)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_gather_scatter_round_trip_with_identity_sr(seed):
    """Gather -> nearest x s ("identity SR") -> scatter reproduces the quantised source pixels on every
    owned MB (pins the rotation map of gather against the un-rotation of scatter) and the bilinear
    value everywhere else."""
    W, H, s = 200, 120, 3
    GW, GH = synth.grid(W, H)
    imp = synth.importance_maps(1, 3, GH, GW, seed, "noisy")
    fr = synth.frames_rgb8(1, 3, H, W, seed)
    ip = oracle.index_path(imp, W, H, int(0.3 * imp.size), partition_mb=3, bin_w=64, bin_h=64, max_bins=40)
    assert ip["placement"][:, 3].any(), "instance should exercise rotation"
    lr = oracle.gather(fr, ip["boxes"], ip["placement"], 64, 64, ip["num_bins"], False)
    hr = np.repeat(np.repeat(lr, s, axis=1), s, axis=2)
    out = oracle.scatter(fr, ip["boxes"], ip["placement"], ip["owner"], hr, s, 64, 64)
    own = ip["owner"][0]
    src = np.repeat(np.repeat(fr[0].astype(np.float32) / np.float32(255.0), s, axis=1), s, axis=2)
    mbmask = np.repeat(np.repeat(own >= 0, 16 * s, axis=1), 16 * s, axis=2)[:, : s * H, : s * W]
    np.testing.assert_array_equal(out[mbmask], src[mbmask].astype(np.float64))
    bil = oracle.scatter(fr, ip["boxes"], ip["placement"], np.full_like(ip["owner"], -1), hr, s, 64, 64)
    np.testing.assert_array_equal(out[~mbmask], bil[~mbmask])
    assert (ip["owner"] >= 0).sum() > 0 and (ip["owner"] >= 0).sum() <= (ip["sel"] > 0).sum()


def test_gather_zero_outside_boxes_and_rotation_geometry():
    # one 3x2 box placed rotated: bin footprint 2 wide, 3 tall; rotated(p,q) = src(x0+q, y0+h-1-p)
    fr = np.arange(1 * 1 * 4 * 6 * 3, dtype=np.uint8).reshape(1, 1, 4, 6, 3)
    bx = np.zeros((1, 12), np.int32)
    bx[0, 6:10] = [1, 1, 3, 2]           # x0=1, y0=1, w=3, h=2
    pl = np.array([[0, 5, 2, 1]], np.int32)
    lr = oracle.gather(fr, bx, pl, 8, 8, 1, False)
    for q in range(3):
        for p in range(2):
            sx, sy = 1 + q, 1 + 2 - 1 - p
            np.testing.assert_array_equal(lr[0, 2 + q, 5 + p], np.float32(fr[0, 0, sy, sx]) / np.float32(255.0))
    mask = np.zeros((8, 8), bool)
    mask[2:5, 5:7] = True
    assert np.all(lr[0][~mask] == 0)
