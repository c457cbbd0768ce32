"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no selection, packing, SR or blending): only
random inputs with the shapes, value distributions and structure of the paper's workloads
(DESIGN.md §4 "input recipe"), and the per-config size tables of BASELINE.json.

* importance maps: per-MB fp32 scores with Gaussian hot-spot blobs + uniform noise, normalised
  to max 1 — the paper's "eregions are a small portion of the frame" (P:271-277, 10-25% area);
  variants: 10 integer levels (massive ties), noise-heavy, all-equal, checkerboard,
  full-frame.
* frames: RGB8 HWC uniform random (SR latency is pixel-value agnostic).
* Y residuals (temporal reuse, §3.2.2): int16, sparse moving objects + noise + occasional scene cuts.
* SR weights: torch.nn.Conv2d default init U(+-1/sqrt(fan_in)) for weights and biases (reading D11).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

MB = 16


def grid(w: int, h: int, mb: int = MB) -> tuple[int, int]:
    """(GW, GH) macroblock grid, partial MBs included (1920x1080 -> 120x68)."""
    return (w + mb - 1) // mb, (h + mb - 1) // mb


def _rng(seed: int, *keys: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, *keys])))


def importance_maps(S: int, F: int, GH: int, GW: int, seed: int = 0, kind: str = "blobs", s0: int = 0) -> np.ndarray:
    """fp32 [S][F][GH][GW] importance scores of streams s0 .. s0+S-1 (each stream seeded by its global
    index, so any shard of a multi-stream workload sees the same maps)."""
    out = np.zeros((S, F, GH, GW), np.float32)
    yy, xx = np.mgrid[0:GH, 0:GW].astype(np.float64)
    for s in range(S):
        rng = _rng(seed, 1, s0 + s)
        for f in range(F):
            if kind == "equal":
                out[s, f] = 0.5
                continue
            if kind == "checker":
                out[s, f] = ((yy + xx) % 2 == 0).astype(np.float32)
                continue
            if kind == "full":
                out[s, f] = 1.0
                continue
            nblob = max(1, math.ceil(GH * GW / 150)) * (4 if kind == "noisy" else 1)
            m = np.zeros((GH, GW))
            for _ in range(nblob):
                cy, cx = rng.uniform(0, GH), rng.uniform(0, GW)
                sig = rng.uniform(1.0, 3.5)
                amp = rng.uniform(0.5, 1.0)
                m += amp * np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / (2 * sig * sig))
            m += rng.uniform(0.0, 0.6 if kind == "noisy" else 0.1, size=(GH, GW))
            m /= m.max()
            if kind == "levels":
                m = np.minimum(np.floor(m * 10.0), 9.0)  # 10 importance levels 0..9
            out[s, f] = m.astype(np.float32)
    return out


def frames_rgb8(S: int, F: int, H: int, W: int, seed: int = 0, s0: int = 0) -> np.ndarray:
    """uint8 [S][F][H][W][3] RGB frames of streams s0 .. s0+S-1 (seeded by global stream index)."""
    out = np.empty((S, F, H, W, 3), np.uint8)
    for s in range(S):
        rng = _rng(seed, 2, s0 + s)
        out[s] = rng.integers(0, 256, size=(F, H, W, 3), dtype=np.uint8)
    return out


def residuals_y(S: int, F: int, H: int, W: int, seed: int = 0, s0: int = 0, scene_cut: float = 0.1) -> np.ndarray:
    """int16 [S][F][H][W] Y-channel residuals of streams s0 .. s0+S-1 (the decoder's residual tap,
    P:598 footnote): mostly zero (the codec predicted the block well), a few small moving objects
    whose pixels carry signed residuals U(+-10..60) with holes (so they split into several small
    components), sparse noise on 0.05% of the pixels, and with probability `scene_cut` per frame a
    large textured block (a big change that the 1/Area operator weighs little)."""
    out = np.zeros((S, F, H, W), np.int16)
    for s in range(S):
        rng = _rng(seed, 4, s0 + s)
        n_obj = int(rng.integers(3, 13))
        pos = rng.uniform([0, 0], [W, H], size=(n_obj, 2))
        vel = rng.uniform(-4, 4, size=(n_obj, 2))
        size = rng.integers(3, 25, size=(n_obj, 2))
        for f in range(F):
            r = out[s, f]
            for o in range(n_obj):
                x0, y0 = int(pos[o, 0]) % W, int(pos[o, 1]) % H
                w, h = int(size[o, 0]), int(size[o, 1])
                blk = r[y0:y0 + h, x0:x0 + w]
                mag = rng.integers(10, 61, size=blk.shape) * rng.choice([-1, 1], size=blk.shape)
                keep = rng.random(blk.shape) < 0.8
                blk[keep] = mag[keep]
                pos[o] += vel[o]
            noise = rng.random((H, W)) < 0.0005
            r[noise] = rng.integers(-30, 31, size=int(noise.sum()))
            if rng.random() < scene_cut:
                bw, bh = int(rng.integers(W // 4, W // 2)), int(rng.integers(H // 4, H // 2))
                bx, by = int(rng.integers(0, W - bw)), int(rng.integers(0, H - bh))
                r[by:by + bh, bx:bx + bw] = rng.integers(-40, 41, size=(bh, bw))
    return out


def frames_nv12(S: int, F: int, H: int, W: int, seed: int = 0, s0: int = 0) -> np.ndarray:
    """uint8 [S][F][H*W*3/2] NV12 frames (decoder output): limited-range Y in [16, 235], U/V in [16, 240],
    uniform random (SR cost is content-agnostic)."""
    out = np.empty((S, F, H * W * 3 // 2), np.uint8)
    for s in range(S):
        rng = _rng(seed, 5, s0 + s)
        out[s, :, : H * W] = rng.integers(16, 236, size=(F, H * W), dtype=np.uint8)
        out[s, :, H * W:] = rng.integers(16, 241, size=(F, H * W // 2), dtype=np.uint8)
    return out


@dataclasses.dataclass(frozen=True)
class SRConfig:
    scale: int
    channels: int
    n_resblocks: int  # 0 => tiny 2-conv model
    res_scale: float = 1.0
    bf16: bool = True

    def conv_shapes(self) -> list[tuple[int, int]]:
        """(Cin, Cout) per conv in network order (the weight-buffer order of include/regen.h)."""
        C, s = self.channels, self.scale
        if self.n_resblocks == 0:
            return [(3, C), (C, 3 * s * s)]
        shapes = [(3, C)]
        shapes += [(C, C)] * (2 * self.n_resblocks)
        shapes += [(C, C)]
        if s == 4:
            shapes += [(C, 4 * C), (C, 4 * C)]
        else:
            shapes += [(C, C * s * s)]
        shapes += [(C, 3)]
        return shapes

    def n_weights(self) -> int:
        return sum(co * ci * 9 + co for ci, co in self.conv_shapes())


def sr_weights(cfg: SRConfig, seed: int = 0) -> np.ndarray:
    """Flat fp32 weights: per conv W[Cout][Cin][3][3] then bias[Cout], network order."""
    rng = _rng(seed, 3)
    parts = []
    for ci, co in cfg.conv_shapes():
        bound = 1.0 / math.sqrt(ci * 9)
        parts.append(rng.uniform(-bound, bound, size=co * ci * 9))
        parts.append(rng.uniform(-bound, bound, size=co))
    return np.concatenate(parts).astype(np.float32)


@dataclasses.dataclass(frozen=True)
class Workload:
    """One selection group: S streams x F frames of W x H, selected by top-k over the group."""
    name: str
    S: int
    F: int
    W: int
    H: int
    pct: float  # top-pct% MBs of the group
    bin_w: int
    bin_h: int
    partition_mb: int
    sr: SRConfig
    max_bins: int
    groups: int = 0   # selection groups in the whole job (S streams each); 0 = one per rank (weak scaling)

    @property
    def GW(self) -> int:
        return grid(self.W, self.H)[0]

    @property
    def GH(self) -> int:
        return grid(self.W, self.H)[1]

    @property
    def n_mbs(self) -> int:
        return self.S * self.F * self.GH * self.GW

    @property
    def k(self) -> int:
        # integer floor(pct% * M), pct given with <= 2 decimals
        return (round(self.pct * 100) * self.n_mbs) // 10000


# BASELINE.json configs (frame count F=30 where unstated: 1-s chunk). A Workload is one
# selection group (the scope of the cross-stream top-N); `groups` > 0 fixes the job's stream count
# (groups x S streams, sharded over the ranks: strong scaling), 0 gives every rank one group (weak).
CONFIGS = {
    "c1": Workload("c1_320x180_x2_tiny_fp32", 1, 8, 320, 180, 10.0, 64, 64, 3,
                   SRConfig(2, 16, 0, 1.0, bf16=False), 64),
    "c2": Workload("c2_360p_x3_edsr8x32_bf16", 1, 30, 640, 360, 20.0, 128, 128, 4,
                   SRConfig(3, 32, 8, 1.0, bf16=True), 512),
    "c3": Workload("c3_8x360p_x3_edsr8x32_bf16", 8, 30, 640, 360, 20.0, 128, 128, 4,
                   SRConfig(3, 32, 8, 1.0, bf16=True), 2048),
    # C4: 64 streams = 8 selection groups of 8 streams (one paper edge server's load)
    "c4": Workload("c4_64x360p_x3_top15_8groups", 8, 30, 640, 360, 15.0, 128, 128, 4,
                   SRConfig(3, 32, 8, 1.0, bf16=True), 2048, groups=8),
    "c4g": Workload("c4_group8_360p_x3_top15", 8, 30, 640, 360, 15.0, 128, 128, 4,
                    SRConfig(3, 32, 8, 1.0, bf16=True), 2048),
    # C5: 16 streams of 720p in 8 selection groups of 2 streams (a 2-stream group at the 50% end of
    # the ratio sweep already needs ~3k bins of C=64 activations); ratio set per run (5..50%)
    "c5": Workload("c5_16x720p_x2_edsr16x64_bf16", 2, 30, 1280, 720, 5.0, 128, 128, 4,
                   SRConfig(2, 64, 16, 1.0, bf16=True), 5632, groups=8),
}
C5_RATIOS = (5.0, 10.0, 15.0, 20.0, 25.0, 35.0, 50.0)


def small(w: Workload, F: int | None = None, S: int | None = None) -> Workload:
    """Same workload with fewer frames/streams (parity-test sizes)."""
    return dataclasses.replace(w, F=F if F is not None else w.F, S=S if S is not None else w.S)
