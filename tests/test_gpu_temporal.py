"""GPU parity of the temporal MB-importance reuse (include/regen.h
regen_temporal_select / regen_reuse_importance) against the oracle: Phi bit for bit (the exact sum of
the 1/area terms), and the float-decided integers (per-stream budgets, selected frames, reuse map)
exactly, on synthetic Y residuals at 360p and 720p, several thresholds and budgets, and the
degenerate cases (no foreground anywhere, one frame, budget below the stream count)."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _run(res, thr, budget):
    import paper_2407_16990_b200 as rg
    S, F, H, W = res.shape
    t = rg.TemporalReuse(S, F, W, H, threshold=thr)
    t.run(torch.from_numpy(res).cuda(), budget)
    torch.cuda.synchronize()
    return t


@pytest.mark.parametrize("S,F,H,W,thr,budget,seed", [
    (2, 30, 360, 640, 8, 12, 0),
    (8, 30, 360, 640, 8, 64, 1),
    (3, 30, 720, 1280, 16, 20, 2),
    (4, 30, 180, 320, 0, 200, 3),       # everything above threshold 0 that is non-zero; budget > S*F
    (5, 7, 90, 160, 30, 3, 4),          # budget below the stream count: anchors only
    (1, 1, 64, 64, 8, 1, 5),            # one frame: no dPhi at all
])
def test_temporal_select_matches_oracle(S, F, H, W, thr, budget, seed):
    res = synth.residuals_y(S, F, H, W, seed)
    t = _run(res, thr, budget)
    o = oracle.temporal_select(res, thr, budget)
    np.testing.assert_array_equal(t.phi.cpu().numpy().view(np.uint64), o["phi"].view(np.uint64))
    np.testing.assert_array_equal(t.frames.cpu().numpy(), o["frames_per_stream"])
    np.testing.assert_array_equal(t.selected.cpu().numpy(), o["selected"])
    np.testing.assert_array_equal(t.reuse.cpu().numpy(), o["reuse"])


def test_temporal_select_without_foreground():
    res = np.zeros((3, 10, 48, 64), np.int16)
    t = _run(res, 8, 9)
    o = oracle.temporal_select(res, 8, 9)
    assert (t.phi.cpu().numpy() == 0).all()
    np.testing.assert_array_equal(t.frames.cpu().numpy(), o["frames_per_stream"])
    np.testing.assert_array_equal(t.selected.cpu().numpy(), o["selected"])
    assert t.selected.cpu().numpy().sum() == 3                 # no change: the anchors only


def test_reuse_importance_copies_the_source_maps():
    S, F, H, W = 2, 30, 360, 640
    res = synth.residuals_y(S, F, H, W, 7)
    t = _run(res, 8, 10)
    GW, GH = synth.grid(W, H)
    pred = synth.importance_maps(S, F, GH, GW, 7)
    out = torch.empty((S, F, GH, GW), dtype=torch.float32, device="cuda")
    t.reuse_maps(torch.from_numpy(pred).cuda(), out)
    ru = t.reuse.cpu().numpy()
    ref = np.stack([pred[s][ru[s]] for s in range(S)])
    np.testing.assert_array_equal(out.cpu().numpy(), ref)
