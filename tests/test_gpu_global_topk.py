"""GPU parity of the exact cross-rank global top-N (include/regen.h regen_topk_*,
global_topk.py): ranks are simulated on one GPU (each "rank" a Pipeline over its own streams, the
all-reduce between the rounds a device sum of their histograms, the rounds run in lock step), and the
selection of every rank, its regions and the rest of its index path must equal the oracle's GLOBAL
selection over the union of the streams, bit for bit."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _rg():
    import paper_2407_16990_b200 as rg
    return rg


def _pipe(wl, S):
    rg = _rg()
    return rg.Pipeline(S=S, F=wl.F, W=wl.W, H=wl.H, k=0, bin_w=wl.bin_w, bin_h=wl.bin_h, max_bins=wl.max_bins,
                       partition_mb=wl.partition_mb, scale=wl.sr.scale, channels=wl.sr.channels,
                       n_resblocks=wl.sr.n_resblocks, weights=synth.sr_weights(wl.sr, 0), bf16=True)


def _simulated_ranks(wl, splits, k_total, kind, seed=3):
    """splits: stream ranges per simulated rank. Returns [(s0, s1, pipe, imp_host)] after the global
    selection and pack_step of every rank."""
    rg = _rg()
    from paper_2407_16990_b200.global_topk import GlobalTopK
    ranks = []
    for s0, s1 in splits:
        imp = synth.importance_maps(s1 - s0, wl.F, wl.GH, wl.GW, seed, kind, s0=s0)
        p = _pipe(wl, s1 - s0)
        ranks.append((s0, s1, p, imp, torch.from_numpy(imp).cuda(), GlobalTopK("cuda")))
    for _, _, _, _, _, g in ranks:
        rg.topk_init(k_total, g.state)
    for _ in range(4):
        for s0, _, p, _, d_imp, g in ranks:
            g.hist.zero_()
            rg.topk_histogram(p.geom, s0, d_imp, g.state, g.hist)
        total = sum(g.hist for *_, g in ranks)          # the all-reduce of the round
        for *_, g in ranks:
            g.hist.copy_(total)
            rg.topk_pick(g.hist, g.state)
    for s0, _, p, _, d_imp, g in ranks:
        g.select(p, d_imp, s0)
        p.pack_step(d_imp)
    return ranks


@pytest.mark.parametrize("splits,kind,frac", [
    ([(0, 4), (4, 8)], "blobs", 0.15),
    ([(0, 3), (3, 5), (5, 8)], "levels", 0.2),       # uneven ranks, massive ties
    ([(0, 4), (4, 8)], "equal", 0.1),                 # all ties: lowest global ids win
    ([(0, 4), (4, 8)], "blobs", 0.0),                 # N = 0
    ([(0, 2), (2, 8)], "noisy", 1.0),                 # N = every MB
])
def test_global_topk_over_simulated_ranks_matches_oracle(splits, kind, frac):
    wl = synth.small(synth.CONFIGS["c4"], F=3)
    n_all = splits[-1][1]
    k_total = int(frac * n_all * wl.F * wl.GH * wl.GW)
    ranks = _simulated_ranks(wl, splits, k_total, kind)
    imp_all = synth.importance_maps(n_all, wl.F, wl.GH, wl.GW, 3, kind)
    sel_all = oracle.select(imp_all, wl.W, wl.H, oracle.MODE_TOPK, k_total)
    assert sel_all.sum() == min(k_total, imp_all.size)
    for s0, s1, p, imp, _, _ in ranks:
        g = p.host_results()
        assert g["status"] == 0
        sel = sel_all[s0:s1]
        np.testing.assert_array_equal(g["sel"], sel)
        # the rest of the rank's index path: the oracle's steps on the rank's slice of the global selection
        labels, regs = oracle.regions(sel, wl.W, wl.H, 8)
        np.testing.assert_array_equal(g["labels"], labels)
        bx, dens, box_of = oracle.boxes(imp, labels, regs, wl.W, wl.H, 3, wl.partition_mb)
        order = oracle.sort(bx, dens)
        pl, nb = oracle.pack(bx, order, wl.bin_w, wl.bin_h, wl.max_bins)
        assert g["num_boxes"] == len(bx) and g["num_bins"] == nb
        np.testing.assert_array_equal(np.stack([g["boxes"][c] for c in ("bin", "bx", "by", "rotated")], 1), pl)
        np.testing.assert_array_equal(g["owner"], oracle.mb_owner(box_of, pl))


def test_global_topk_single_rank_equals_regen_select_mbs():
    """With one rank the protocol is the local GLOBAL-scope selection of regen_select_mbs."""
    from paper_2407_16990_b200.global_topk import global_select
    wl = synth.small(synth.CONFIGS["c4"], F=4)
    imp = synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 9, "levels")
    d_imp = torch.from_numpy(imp).cuda()
    a, b = _pipe(wl, wl.S), _pipe(wl, wl.S)
    a.sel.k = wl.k
    a.select(d_imp)
    global_select([(b, 0, d_imp)], wl.k, "cuda")
    ga, gb = a.host_results(), b.host_results()
    np.testing.assert_array_equal(ga["sel"], gb["sel"])
    np.testing.assert_array_equal(ga["labels"], gb["labels"])


def test_select_before_the_rounds_reports_incomplete():
    rg = _rg()
    from paper_2407_16990_b200.global_topk import GlobalTopK
    wl = synth.small(synth.CONFIGS["c4"], F=2)
    imp = torch.from_numpy(synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 1)).cuda()
    p = _pipe(wl, wl.S)
    g = GlobalTopK("cuda")
    rg.topk_init(100, g.state)
    g.select(p, imp, 0)
    r = p.host_results()
    assert r["status"] & rg.ST_TOPK_INCOMPLETE and r["sel"].sum() == 0
