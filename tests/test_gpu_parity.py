"""GPU parity: the CUDA path through the C-ABI (paper_2407_16990_b200) vs the CPU oracle, on the same
seeded inputs. Integer outputs (selection, labels, regions, boxes incl. fp64 density bits, order,
placements, bin count, MB owners) must be bit-exact; pixels within 1e-4 (fp32 model) or 2e-2 (bf16
model) max-abs (BASELINE.json north_star)."""
import dataclasses
import os

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {True: 2e-2, False: 1e-4}


def _rg():
    import paper_2407_16990_b200 as rg
    return rg


def _pipeline(wl, weights, **kw):
    rg = _rg()
    return rg.Pipeline(S=wl.S, F=wl.F, W=wl.W, H=wl.H, k=kw.pop("k", wl.k), bin_w=wl.bin_w, bin_h=wl.bin_h,
                       max_bins=wl.max_bins, partition_mb=wl.partition_mb, scale=wl.sr.scale,
                       channels=wl.sr.channels, n_resblocks=wl.sr.n_resblocks, weights=weights, bf16=wl.sr.bf16,
                       res_scale=wl.sr.res_scale, **kw)


def _oracle_index(wl, imp, **kw):
    return oracle.index_path(imp, wl.W, wl.H, kw.pop("k", wl.k), partition_mb=wl.partition_mb, bin_w=wl.bin_w,
                             bin_h=wl.bin_h, max_bins=wl.max_bins, **kw)


def _assert_index_equal(g, o):
    assert g["status"] == 0
    np.testing.assert_array_equal(g["sel"], o["sel"])
    np.testing.assert_array_equal(g["labels"], o["labels"])
    assert g["num_regions"] == len(o["regions"])
    gr = g["regions"]
    np.testing.assert_array_equal(np.stack([gr[f] for f in gr.dtype.names], 1), o["regions"])
    assert g["num_boxes"] == len(o["boxes"])
    gb = g["boxes"]
    cols = ["stream", "frame", "mx0", "my0", "mx1", "my1", "x0", "y0", "w", "h", "n_members", "region"]
    np.testing.assert_array_equal(np.stack([gb[c] for c in cols], 1), o["boxes"])
    np.testing.assert_array_equal(gb["density"].view(np.uint64), o["density"].view(np.uint64))
    np.testing.assert_array_equal(g["order"], o["order"])
    np.testing.assert_array_equal(np.stack([gb["bin"], gb["bx"], gb["by"], gb["rotated"]], 1), o["placement"])
    assert g["num_bins"] == o["num_bins"]
    np.testing.assert_array_equal(g["owner"], o["owner"])


def _run_index(wl, imp, weights, **kw):
    p = _pipeline(wl, weights, **kw)
    d_imp = torch.from_numpy(imp).cuda()
    p.select(d_imp)
    p.pack_step(d_imp)
    return p, p.host_results()


INDEX_CASES = [
    ("c1", "blobs", {}),
    ("c2f4", "blobs", {}),
    ("c2f4", "levels", {}),
    ("c2f4", "equal", {}),
    ("c2f4", "checker", {}),
    ("c2f4", "noisy", {}),
    ("c2f4", "full", {"k": 40 * 23 * 4}),
    ("c2f4", "noisy", {"connectivity": 4}),
    ("c2f4", "levels", {"mode": 1, "tau": 5.0, "k": -1}),
    ("c2f4", "blobs", {"mode": 1, "tau": 0.4, "k": 900}),
    ("c2f4", "levels", {"scope": 2, "k": 37}),
    ("c2f4", "blobs", {"scope": 1, "k": 500}),
    ("c2f4", "blobs", {"order": 1}),
    ("c3f2", "blobs", {}),
    ("c5f2", "noisy", {}),
    ("c2f4", "levels", {"cap": 700}),                       # capacity N below k
    ("c2f4", "blobs", {"mode": 1, "tau": 0.3, "k": -1, "cap": 450}),
    ("c2f4", "noisy", {"density": 1}),                      # REGEN_DENSITY_MEMBERS
    ("c2f4", "blobs", {"order": 2}),                        # REGEN_ORDER_HEIGHT
]


def _wl(name):
    if name == "c2f4":
        return synth.small(synth.CONFIGS["c2"], F=4)
    if name == "c3f2":
        return synth.small(synth.CONFIGS["c3"], F=2)
    if name == "c5f2":
        return synth.small(synth.CONFIGS["c5"], F=2)
    return synth.CONFIGS[name]


@pytest.mark.parametrize("name,kind,kw", INDEX_CASES)
def test_index_path_bit_exact(name, kind, kw):
    wl = _wl(name)
    imp = synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 11, kind)
    w = synth.sr_weights(wl.sr, 0)
    okw = dict(kw)
    conv = okw.pop("connectivity", 8)
    order = okw.pop("order", 0)
    dens = okw.pop("density", 0)
    _, g = _run_index(wl, imp, w, **kw)
    o = _oracle_index(wl, imp, conn=conv, order_policy=order, density_mode=dens, **okw)
    _assert_index_equal(g, o)


POLICY_CASES = [(pol, name, kind, extra) for pol in (1, 2, 3)
                for name, kind, extra in [("c2f4", "blobs", {}), ("c2f4", "noisy", {}), ("c3f2", "blobs", {}),
                                          ("c1", "blobs", {}), ("c2f4", "noisy", {"max_bins": 6})]] + \
               [(3, "c2f4", "blobs", {"order": 2}), (2, "c2f4", "levels", {"order": 1})]


@pytest.mark.parametrize("policy,name,kind,extra", POLICY_CASES)
def test_index_path_policies_bit_exact(policy, name, kind, extra):
    """MAXRECT (literal Alg. 2, D14), SKYLINE (D15) and SHELF (D16) placements on the GPU
    (pack_policies.cu) equal the oracle's, including unplaced boxes when the bins run out."""
    wl = _wl(name)
    if "max_bins" in extra:
        wl = dataclasses.replace(wl, max_bins=extra["max_bins"])
    imp = synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 19, kind)
    order = extra.get("order", 0)
    _, g = _run_index(wl, imp, synth.sr_weights(wl.sr, 0), policy=policy, order=order)
    o = _oracle_index(wl, imp, policy=policy, order_policy=order)
    if "max_bins" in extra:
        assert (o["placement"][:, 0] < 0).any()
    _assert_index_equal(g, o)


@pytest.mark.parametrize("P", [1, 2, 7])
def test_index_path_partition_sizes(P):
    """Block mode (partition_mb = 1: every selected MB its own box, SURVEY §8(f)1 'Block') and the
    other partition limits of the survey's fill study, bit-exact against the oracle."""
    wl = dataclasses.replace(synth.small(synth.CONFIGS["c2"], F=3), partition_mb=P)
    imp = synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 13, "noisy")
    _, g = _run_index(wl, imp, synth.sr_weights(wl.sr, 0))
    o = _oracle_index(wl, imp)
    _assert_index_equal(g, o)


@pytest.mark.parametrize("cfg,F,P,pct,kind", [("c2", 30, 1, 20.0, "blobs"),     # 5520 boxes (Block mode)
                                              ("c5", 14, 4, 50.0, "blobs"),     # 720p 50%: ~5.8k boxes, ~2.3k bins
                                              ("c4g", 30, 2, 15.0, "noisy")])
def test_index_path_large_pools_bit_exact(cfg, F, P, pct, kind):
    """Beyond PACK_BINS_FROM boxes the packer switches to per-bin area lists with dominance summaries
    (pack.cu pack_bins); placements stay bit-exact against the oracle's linear first-fit scan."""
    wl = dataclasses.replace(synth.small(synth.CONFIGS[cfg], F=F), partition_mb=P, pct=pct)
    imp = synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 17, kind)
    _, g = _run_index(wl, imp, synth.sr_weights(wl.sr, 0))
    o = _oracle_index(wl, imp)
    assert len(o["boxes"]) > 5000
    _assert_index_equal(g, o)


def test_index_path_small_max_bins_leaves_unplaced():
    wl = dataclasses.replace(synth.small(synth.CONFIGS["c2"], F=3), max_bins=5)
    imp = synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 2)
    _, g = _run_index(wl, imp, synth.sr_weights(wl.sr, 0))
    o = _oracle_index(wl, imp)
    assert (o["placement"][:, 0] < 0).any()
    _assert_index_equal(g, o)


def test_index_path_zero_k_and_empty():
    wl = synth.small(synth.CONFIGS["c2"], F=2)
    imp = synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 2)
    _, g = _run_index(wl, imp, synth.sr_weights(wl.sr, 0), k=0)
    assert g["num_regions"] == 0 and g["num_boxes"] == 0 and g["num_bins"] == 0
    assert (g["owner"] < 0).all() and g["sel"].sum() == 0


@pytest.mark.parametrize("bf16", [True, False])
def test_stitch_bins_bit_exact(bf16):
    rg = _rg()
    wl = synth.small(synth.CONFIGS["c2"], F=3)
    wl = dataclasses.replace(wl, sr=dataclasses.replace(wl.sr, bf16=bf16))
    imp = synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 4, "noisy")
    fr = synth.frames_rgb8(wl.S, wl.F, wl.H, wl.W, 4)
    p, g = _run_index(wl, imp, synth.sr_weights(wl.sr, 0))
    o = _oracle_index(wl, imp)
    nb = o["num_bins"]
    dt = torch.bfloat16 if bf16 else torch.float32
    lr = torch.zeros((wl.max_bins, wl.bin_h, wl.bin_w, 4), dtype=dt, device="cuda")
    rg.stitch_bins(p.geom, p.pack, rg.DTYPE_BF16 if bf16 else rg.DTYPE_FP32, torch.from_numpy(fr).cuda(), p.boxes,
                   p.max_boxes, p.counts[1:2], p.num_bins, lr, p.ws)
    ref = oracle.gather(fr, o["boxes"], o["placement"], wl.bin_w, wl.bin_h, nb, bf16)
    got = lr[:nb, :, :, :3].float().cpu().numpy().astype(np.float64)
    np.testing.assert_array_equal(got, ref)
    assert (lr[:nb, :, :, 3] == 0).all()


def _check_pixels(wl, seed=5, kind="blobs", box_sample=None, frame_sample=None):
    imp = synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, seed, kind)
    fr = synth.frames_rgb8(wl.S, wl.F, wl.H, wl.W, seed)
    w = synth.sr_weights(wl.sr, seed)
    p = _pipeline(wl, w)
    imp_t, fr_t = torch.from_numpy(imp).cuda(), torch.from_numpy(fr).cuda()
    out = p.run(imp_t, fr_t, fused=False).clone()            # regen_enhance_packed + regen_scatter_blend
    out_fused = p.run(imp_t, fr_t, out=torch.empty_like(out))  # regen_enhance_scatter
    assert torch.equal(out_fused, out), "regen_enhance_scatter differs from the separate calls"
    # the two halves (regen_enhance_owned + regen_scatter_bilinear, in either order) cover every HR
    # pixel exactly once (NaN-filled buffer) and equal the fused call
    for order in (0, 1):
        out_split = torch.full_like(out, float("nan"))
        if order == 0:
            p.enhance_owned(fr_t, out=out_split)
            p.scatter_bilinear(fr_t, out=out_split)
        else:
            p.scatter_bilinear(fr_t, out=out_split)
            p.enhance_owned(fr_t, out=out_split)
        assert torch.equal(out_split, out), "regen_enhance_owned + regen_scatter_bilinear differ from the fused call"
    if (wl.sr.bf16 and wl.sr.n_resblocks > 0 and not os.environ.get("REGEN_NO_FOLD")
            and not os.environ.get("REGEN_FORCE_SIMT")):
        # the SR half split again (regen_enhance_partials + regen_fold_combine_frames): bit-identical
        out_split = torch.full_like(out, float("nan"))
        p.scatter_bilinear(fr_t, out=out_split)
        p.enhance_partials(fr_t)
        p.fold_combine(out=out_split)
        assert torch.equal(out_split, out), "regen_enhance_partials + regen_fold_combine_frames differ"
    g = p.host_results()
    o = _oracle_index(wl, imp)
    _assert_index_equal(g, o)
    nb = o["num_bins"]
    lr = oracle.gather(fr, o["boxes"], o["placement"], wl.bin_w, wl.bin_h, nb, wl.sr.bf16)
    w64 = oracle.sr_weights_for(wl.sr, w)
    nbox = len(o["boxes"])
    boxes_to_check = range(nbox) if box_sample is None else box_sample(nbox)
    hr_g = p.hr_bins[:nb].float().cpu().numpy()
    tol = TOL[wl.sr.bf16]
    s = wl.sr.scale
    worst = 0.0
    for b in boxes_to_check:
        bin_, bx, by, rot = o["placement"][b]
        if bin_ < 0:
            continue
        hr = oracle.enhance(wl.sr, w64, lr, o["boxes"], o["placement"], b, b + 1)
        w_, h_ = o["boxes"][b, 8], o["boxes"][b, 9]
        fw, fh = (h_, w_) if rot else (w_, h_)
        sl = (bin_, slice(s * by, s * (by + fh)), slice(s * bx, s * (bx + fw)))
        d = np.abs(hr_g[sl][..., :3] - hr[sl])
        worst = max(worst, float(d.max()))
        assert d.max() <= tol, f"box {b}: max err {d.max()}"
    # HR bin pixels outside every box are zero
    f_lo, f_hi = (0, wl.S * wl.F) if frame_sample is None else frame_sample
    if box_sample is None:
        hr_all = oracle.enhance(wl.sr, w64, lr, o["boxes"], o["placement"])
        ref = oracle.scatter(fr, o["boxes"], o["placement"], o["owner"], hr_all, s, wl.bin_w, wl.bin_h, f_lo, f_hi)
        got = out.reshape(-1, *out.shape[2:])[f_lo:f_hi].float().cpu().numpy()
        d = np.abs(got - ref)
        assert d.max() <= tol, f"frames: max err {d.max()}"
    return worst


def test_pixels_c1_fp32_full():
    _check_pixels(synth.CONFIGS["c1"])


def test_pixels_c2_bf16_small():
    _check_pixels(synth.small(synth.CONFIGS["c2"], F=2), box_sample=lambda n: range(0, n, max(1, n // 12)))


def test_pixels_tiny_fp32_x3_full_frames():
    wl = dataclasses.replace(synth.small(synth.CONFIGS["c2"], F=2), sr=synth.SRConfig(3, 16, 0, 1.0, False))
    _check_pixels(wl)


@pytest.mark.parametrize("sr,bin_w", [(synth.SRConfig(3, 16, 0, 1.0, True), 128),   # tiny model: no tcgen05 tail
                                      (synth.SRConfig(3, 8, 1, 1.0, True), 128),    # C % 16 != 0
                                      (synth.SRConfig(3, 32, 1, 1.0, True), 96)])   # bin_w % 128 != 0
def test_bf16_configs_without_tensor_core_kernels_fail_loudly(sr, bin_w):
    """No silent dispatch: a BF16 model with a conv the tcgen05 kernels do not tile is rejected by
    regen_sr_create with REGEN_E_UNSUPPORTED instead of running on the CUDA-core kernel."""
    rg = _rg()
    with pytest.raises(rg.RegenError, match="unsupported"):
        rg.SRNet(sr.scale, sr.channels, sr.n_resblocks, synth.sr_weights(sr, 0), True, 1.0, bin_w)


def test_pixels_small_edsr_bf16_full_frames():
    wl = dataclasses.replace(synth.small(synth.CONFIGS["c2"], F=1), sr=synth.SRConfig(3, 16, 1, 1.0, True))
    _check_pixels(wl, kind="noisy")


def test_pixels_small_edsr_fp32_x4_and_x2():
    for s in (4, 2):
        wl = dataclasses.replace(synth.small(synth.CONFIGS["c2"], F=1), sr=synth.SRConfig(s, 8, 1, 0.5, False))
        _check_pixels(wl, box_sample=lambda n: range(0, n, max(1, n // 10)))


@pytest.mark.parametrize("s,C,nres", [(2, 32, 1), (4, 32, 1), (2, 64, 1), (3, 48, 1)])
def test_pixels_bf16_tensor_core_shapes(s, C, nres):
    """tcgen05 SLIDE/PLAIN mappings at every tile count: x2 (HR rows of 2 tiles), x4 (2x stage of 2
    tiles, tail of 4 tiles), C=64 (N=192 windows, 2 PLAIN chunks), C=48."""
    wl = dataclasses.replace(synth.small(synth.CONFIGS["c2"], F=1), sr=synth.SRConfig(s, C, nres, 1.0, True))
    _check_pixels(wl, kind="noisy", box_sample=lambda n: range(0, n, max(1, n // 6)))


def _kernels_of(fn):
    rg = _rg()
    rg.trace_read()
    rg.trace_enable(True)
    try:
        fn()
        torch.cuda.synchronize()
    finally:
        rg.trace_enable(False)
    return {name for name, _ in rg.trace_read()}


def test_sr_tensor_core_matches_simt_path(monkeypatch):
    """The same batch through the tcgen05 kernels and, in a handle created under the explicit
    REGEN_FORCE_SIMT=1 switch, through the CUDA-core kernel: the launched kernels prove which path
    ran, both stay within the bf16 tolerance of the oracle and of each other."""
    wl = synth.small(synth.CONFIGS["c2"], F=2)
    sample = lambda n: range(1, n, max(1, n // 5))  # noqa: E731
    imp = synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 9)
    fr = torch.from_numpy(synth.frames_rgb8(wl.S, wl.F, wl.H, wl.W, 9)).cuda()
    w = synth.sr_weights(wl.sr, 9)
    outs = {}
    for mode in ("tc", "simt"):
        if mode == "simt":
            monkeypatch.setenv("REGEN_FORCE_SIMT", "1")
        p = _pipeline(wl, w)
        d_imp = torch.from_numpy(imp).cuda()
        names = _kernels_of(lambda: p.run(d_imp, fr))
        if mode == "tc":
            assert "resblock" in names and "conv_fold_frames" in names and "conv_simt" not in names, names
        else:
            assert "conv_simt" in names and not any(n.startswith(("resblock", "conv_fold", "conv_head")) for n in names), names
        outs[mode] = p.out.float().clone()
        assert _check_pixels(wl, seed=9, box_sample=sample) <= TOL[True]
    assert float((outs["tc"] - outs["simt"]).abs().max()) <= TOL[True]


@pytest.mark.parametrize("s,C", [(3, 32), (2, 32), (4, 16), (3, 64)])
def test_upsampler_tail_fold_matches_oracle_and_literal_path(s, C, monkeypatch):
    """The UP∘TAIL fold (upfold.cu) and the literal upsampler + tail both stay within the
    bf16 tolerance of the oracle on the same boxes (REGEN_NO_FOLD=1 selects the literal path)."""
    wl = dataclasses.replace(synth.small(synth.CONFIGS["c2"], F=1), sr=synth.SRConfig(s, C, 1, 1.0, True))
    sample = lambda n: range(0, n, max(1, n // 8))  # noqa: E731
    worst_fold = _check_pixels(wl, seed=11, kind="noisy", box_sample=sample)
    monkeypatch.setenv("REGEN_NO_FOLD", "1")
    worst_lit = _check_pixels(wl, seed=11, kind="noisy", box_sample=sample)
    assert worst_fold <= TOL[True] and worst_lit <= TOL[True]


def test_stitch_bin_with_more_boxes_than_the_smem_cache():
    """A 1024 x 128 bin of one-MB boxes holds more than the stitch's 128-entry SMEM box cache: the boxes
    past it are read from their records; every pixel still matches the oracle (fp32 tiny model)."""
    wl = dataclasses.replace(synth.small(synth.CONFIGS["c1"], F=6), bin_w=1024, bin_h=128, pct=40.0,
                             partition_mb=1, max_bins=8)
    imp = synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 31, "noisy")
    o = _oracle_index(wl, imp)
    per_bin = np.bincount(o["placement"][:, 0][o["placement"][:, 0] >= 0])
    assert per_bin.max() > 128, per_bin
    assert _check_pixels(wl, seed=31, kind="noisy") <= TOL[False]


def test_no_selection_gives_the_pure_bilinear_frames():
    """k = 0: no region, no box, no bin; every HR pixel is the D10 bilinear value (the enhance call runs
    over zero bins)."""
    wl = synth.small(synth.CONFIGS["c2"], F=2)
    imp = synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 3)
    fr = synth.frames_rgb8(wl.S, wl.F, wl.H, wl.W, 3)
    p = _pipeline(wl, synth.sr_weights(wl.sr, 0), k=0)
    out = p.run(torch.from_numpy(imp).cuda(), torch.from_numpy(fr).cuda())
    g = p.host_results()
    assert g["num_boxes"] == 0 and g["num_bins"] == 0
    ref = oracle.scatter(fr, np.zeros((0, 12), np.int32), np.zeros((0, 4), np.int32), np.full(g["owner"].shape, -1,
                         np.int32), np.zeros(1), wl.sr.scale, wl.bin_w, wl.bin_h)
    got = out.float().cpu().numpy().reshape(ref.shape)
    assert np.abs(got - ref).max() <= 2e-2 * 0.5


@pytest.mark.parametrize("W,H", [(200, 120), (328, 184)])
def test_odd_frame_sizes_whole_path(W, H):
    """Frame widths that are not a multiple of 8 (the bilinear pass takes its row kernel) and partial
    MBs on both axes, through the whole bf16 path: index path bit-exact, every HR pixel in tolerance."""
    wl = dataclasses.replace(synth.small(synth.CONFIGS["c2"], F=2), W=W, H=H, pct=25.0,
                             sr=synth.SRConfig(3, 16, 1, 1.0, True))
    _check_pixels(wl, seed=6, kind="noisy")
