"""Exhaustive pixel parity at BASELINE sizes, in the launch configuration bench.py times (two pipelines
on two streams, the steps captured into one CUDA graph and replayed): EVERY placed box's SR pixels
and EVERY HR pixel of every frame against the oracle (fp64; its multi-threaded entries, bit-identical
to the single-threaded ones, spread the boxes and frames over the host cores), within the bf16
tolerance 2e-2 of north_star. Plus one test per asynchronous status bit (include/regen.h
REGEN_ST_*): the overflow is reported and the outputs are truncated deterministically."""
import dataclasses

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL_BF16 = 2e-2


def _rg():
    import paper_2407_16990_b200 as rg
    return rg


def _make(wl, w, **kw):
    rg = _rg()
    return lambda: rg.Pipeline(S=wl.S, F=wl.F, W=wl.W, H=wl.H, k=wl.k, bin_w=wl.bin_w, bin_h=wl.bin_h,
                               max_bins=wl.max_bins, partition_mb=wl.partition_mb, scale=wl.sr.scale,
                               channels=wl.sr.channels, n_resblocks=wl.sr.n_resblocks, weights=w,
                               bf16=wl.sr.bf16, res_scale=wl.sr.res_scale, **kw)


def _every_pixel(wl, seed, **pipe_kw):
    from paper_2407_16990_b200.schedule import PipelinedRunner
    imp_h = synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, seed)
    fr_h = synth.frames_rgb8(wl.S, wl.F, wl.H, wl.W, seed)
    w = synth.sr_weights(wl.sr, seed)
    r = PipelinedRunner(_make(wl, w, **pipe_kw), "cuda", n_pipes=3, n_front=2)
    imp, fr = torch.from_numpy(imp_h).cuda(), torch.from_numpy(fr_h).cuda()
    r.run_eager(imp, fr, 2)
    torch.cuda.synchronize()
    for q in r.pipes:
        q.out.fill_(float("nan"))
    g = r.capture(imp, fr, 3)
    g.replay()
    torch.cuda.synchronize()
    out = r.pipes[0].out.float().cpu().numpy().reshape(-1, wl.sr.scale * wl.H, wl.sr.scale * wl.W, 3)
    assert torch.equal(r.pipes[0].out, r.pipes[1].out)
    res = r.pipes[0].host_results()
    o = oracle.index_path(imp_h, wl.W, wl.H, wl.k, partition_mb=wl.partition_mb, bin_w=wl.bin_w, bin_h=wl.bin_h,
                          max_bins=wl.max_bins, policy=pipe_kw.get("policy", 0), order_policy=pipe_kw.get("order", 0))
    assert res["status"] == 0 and res["num_bins"] == o["num_bins"]
    np.testing.assert_array_equal(res["owner"], o["owner"])
    np.testing.assert_array_equal(np.stack([res["boxes"][c] for c in ("bin", "bx", "by", "rotated")], 1),
                                  o["placement"])
    cores = oracle.host_cores()
    lr = oracle.gather(fr_h, o["boxes"], o["placement"], wl.bin_w, wl.bin_h, o["num_bins"], wl.sr.bf16)
    hr = oracle.enhance(wl.sr, oracle.sr_weights_for(wl.sr, w), lr, o["boxes"], o["placement"], threads=cores)
    worst = 0.0
    n = wl.S * wl.F
    for f0 in range(0, n, 4):    # 4 frames of fp64 HR at a time
        f1 = min(n, f0 + 4)
        ref = oracle.scatter(fr_h, o["boxes"], o["placement"], o["owner"], hr, wl.sr.scale, wl.bin_w, wl.bin_h,
                             f0, f1, threads=cores)
        d = float(np.abs(out[f0:f1] - ref).max())
        worst = max(worst, d)
        assert d <= TOL_BF16, f"frames [{f0}, {f1}): max abs err {d}"
    return worst, int((o["placement"][:, 0] >= 0).sum())


def test_c2_every_box_every_hr_pixel():
    """C2 (BASELINE configs[1], the bench workload): all ~630 placed boxes, all 30 x 1920 x 1080 HR pixels."""
    worst, nbox = _every_pixel(synth.CONFIGS["c2"], 21)
    assert nbox > 500
    print(f"C2: {nbox} boxes, every HR pixel within {worst:.3e}")


def test_c3_two_frames_every_box_every_hr_pixel():
    """C3 (8 streams, one selection group) at 2 frames per stream: every box and HR pixel."""
    worst, nbox = _every_pixel(synth.small(synth.CONFIGS["c3"], F=2), 22)
    assert nbox > 200


def test_c4_group_two_frames_every_box_every_hr_pixel():
    """C4's selection group (8 streams, top-15%) at 2 frames per stream: every box and HR pixel."""
    worst, nbox = _every_pixel(synth.small(synth.CONFIGS["c4"], F=2), 23)
    assert nbox > 150


def test_c5_group_two_frames_every_box_every_hr_pixel():
    """C5's selection group (2 streams of 720p -> 1440p x2, EDSR 16 x 64: the unfused C = 64 convs and
    the p = 2 fold) at 2 frames per stream and a 10% ratio: every box and HR pixel."""
    import dataclasses as dc
    worst, nbox = _every_pixel(dc.replace(synth.small(synth.CONFIGS["c5"], F=2), pct=10.0), 24)
    assert nbox > 50


@pytest.mark.parametrize("policy,order", [(1, 0), (2, 0), (3, 2)])
def test_policy_packings_through_the_whole_path(policy, order):
    """The SR and paste-back do not depend on the packer: bins filled by the MAXRECT / SKYLINE / SHELF
    policies give every HR pixel within tolerance too (C2 geometry, 3 frames)."""
    worst, nbox = _every_pixel(synth.small(synth.CONFIGS["c2"], F=3), 25, policy=policy, order=order)
    assert nbox > 40


# ----------------------------------------------------------------------------- status bits

def _wl_small():
    return synth.small(synth.CONFIGS["c2"], F=3)


def test_status_region_overflow_truncates_records():
    rg = _rg()
    wl = _wl_small()
    imp_h = synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 3, "noisy")
    p = _make(wl, synth.sr_weights(wl.sr, 0))()
    imp = torch.from_numpy(imp_h).cuda()
    rg.select_mbs(p.geom, p.sel, imp, p.bitmap, p.labels, p.regions, 3, p.counts[0:1], p.status, p.ws)
    torch.cuda.synchronize()
    o = oracle.index_path(imp_h, wl.W, wl.H, wl.k, partition_mb=wl.partition_mb, bin_w=wl.bin_w, bin_h=wl.bin_h,
                          max_bins=wl.max_bins)
    assert int(p.status.item()) & rg.ST_REGION_OVERFLOW
    assert int(p.counts[0].item()) == len(o["regions"]) > 3          # the true count is reported
    got = np.frombuffer(p.regions[: 3 * 32].cpu().numpy().tobytes(), rg.REGION_DTYPE)
    np.testing.assert_array_equal(np.stack([got[f] for f in got.dtype.names], 1), o["regions"][:3])


def test_status_box_overflow_truncates_boxes_deterministically():
    rg = _rg()
    wl = _wl_small()
    imp_h = synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 4)
    p = _make(wl, synth.sr_weights(wl.sr, 0), max_boxes=5)()
    imp = torch.from_numpy(imp_h).cuda()
    p.select(imp)
    p.pack_step(imp)
    g = p.host_results()
    o = oracle.index_path(imp_h, wl.W, wl.H, wl.k, partition_mb=wl.partition_mb, bin_w=wl.bin_w, bin_h=wl.bin_h,
                          max_bins=wl.max_bins)
    assert g["status"] & rg.ST_BOX_OVERFLOW and not g["status"] & rg.ST_REGION_OVERFLOW
    assert g["num_boxes"] == len(o["boxes"]) > 5
    cols = ["stream", "frame", "mx0", "my0", "mx1", "my1", "x0", "y0", "w", "h", "n_members", "region"]
    np.testing.assert_array_equal(np.stack([g["boxes"][c] for c in cols], 1), o["boxes"][:5])
    # the first 5 boxes are sorted and packed exactly as the oracle packs those 5
    order = oracle.sort(o["boxes"][:5], o["density"][:5])
    pl, nb = oracle.pack(o["boxes"][:5], order, wl.bin_w, wl.bin_h, wl.max_bins)
    np.testing.assert_array_equal(g["order"], order)
    np.testing.assert_array_equal(np.stack([g["boxes"][c] for c in ("bin", "bx", "by", "rotated")], 1), pl)
    own = o["box_of_mb"].copy()
    own[own >= 5] = -1
    np.testing.assert_array_equal(g["owner"], oracle.mb_owner(own, pl))


@pytest.mark.parametrize("F", [3, 30])   # 3 frames: the pool path; 30 frames (5520 boxes): the per-bin path
def test_status_freelist_overflow_keeps_a_valid_plan(monkeypatch, F):
    rg = _rg()
    wl = dataclasses.replace(synth.small(synth.CONFIGS["c2"], F=F), partition_mb=1)   # Block mode: many boxes
    imp_h = synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 5, "noisy")
    monkeypatch.setenv("REGEN_PACK_POOL_LIMIT", "1")         # one live free area (per bin on the bins path)
    p = _make(wl, synth.sr_weights(wl.sr, 0))()
    imp = torch.from_numpy(imp_h).cuda()
    p.select(imp)
    p.pack_step(imp)
    g = p.host_results()
    assert g["status"] & rg.ST_FREELIST_OVERFLOW
    bx = g["boxes"]
    placed = bx["bin"] >= 0
    assert placed.sum() > 0
    # the plan stays valid: footprints inside their bins and pairwise disjoint
    occ = np.zeros((g["num_bins"], wl.bin_h + 1, wl.bin_w), np.int32)
    for b in np.flatnonzero(placed):
        fw, fh = (bx["h"][b], bx["w"][b]) if bx["rotated"][b] else (bx["w"][b], bx["h"][b])
        x, y = bx["bx"][b], bx["by"][b]
        assert x >= 1 and x + fw + 1 <= wl.bin_w and y + fh + 1 <= wl.bin_h + 1
        occ[bx["bin"][b], y:y + fh + 1, x:x + fw + 1] += 1
    assert occ.max() == 1
    monkeypatch.delenv("REGEN_PACK_POOL_LIMIT")
    p.select(imp)
    p.pack_step(imp)
    assert p.host_results()["status"] == 0                    # the default pool holds this instance


def test_boxes_at_the_bin_border_finite_deterministic_and_exact():
    """Regression (found by bench.py's e2e check on C5 at 15%): the head conv's packed-dx MMA used to read
    one pixel past the bin row for pixel W-2 (a box touching the reserved right gutter); stale SMEM there
    can hold NaN patterns and 0 * NaN = NaN. C5 group, 15%, 10 frames: no NaN, two runs bit-identical,
    and the boxes that end at column W-2 match the oracle."""
    import dataclasses as dc
    rg = _rg()
    wl = dc.replace(synth.CONFIGS["c5"], pct=15.0, F=10)
    imp_h = synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 0)
    fr_h = synth.frames_rgb8(wl.S, wl.F, wl.H, wl.W, 0)
    w = synth.sr_weights(wl.sr, 0)
    p = _make(wl, w)()
    imp, fr = torch.from_numpy(imp_h).cuda(), torch.from_numpy(fr_h).cuda()
    a = p.run(imp, fr, fused=False).clone()
    b = p.run(imp, fr, fused=False).clone()
    assert not torch.isnan(a.float()).any() and torch.equal(a, b)
    g = p.host_results()
    bx = g["boxes"]
    fw = np.where(bx["rotated"] == 1, bx["h"], bx["w"])
    edge = np.flatnonzero((bx["bin"] >= 0) & (bx["bx"] + fw == wl.bin_w - 1))
    assert len(edge) > 0
    o = oracle.index_path(imp_h, wl.W, wl.H, wl.k, partition_mb=wl.partition_mb, bin_w=wl.bin_w, bin_h=wl.bin_h,
                          max_bins=wl.max_bins)
    lr = oracle.gather(fr_h, o["boxes"], o["placement"], wl.bin_w, wl.bin_h, o["num_bins"], True)
    w64 = oracle.sr_weights_for(wl.sr, w)
    hr_g = p.hr_bins.float().cpu().numpy()
    s = wl.sr.scale
    sample = edge[:: max(1, len(edge) // 4)][:4]
    pl = o["placement"].copy()
    keep = np.zeros(len(pl), bool)
    keep[sample] = True
    pl[~keep, 0] = -1                      # the sampled boxes only, one oracle call over the host cores
    hr = oracle.enhance(wl.sr, w64, lr, o["boxes"], pl, threads=oracle.host_cores())
    for bi in sample:
        b_, x_, y_, rot = o["placement"][bi]
        ww, hh = (o["boxes"][bi, 9], o["boxes"][bi, 8]) if rot else (o["boxes"][bi, 8], o["boxes"][bi, 9])
        sl = (b_, slice(s * y_, s * (y_ + hh)), slice(s * x_, s * (x_ + ww)))
        assert np.abs(hr_g[sl][..., :3] - hr[sl]).max() <= TOL_BF16
