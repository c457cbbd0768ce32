"""CPU oracle for the RegenHance hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) may import
this package. The product path (paper_2407_16990_b200) never imports it and shares no code with
it: the arithmetic lives in regen_oracle.c (plain C, fp64, one function per step of the paper,
each citing PAPER.md lines); this file only marshals numpy arrays through ctypes and composes
the steps in the paper's order (Alg. 1, §3.3).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "regen_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

MODE_TOPK, MODE_THRESHOLD = 0, 1
SCOPE_GLOBAL, SCOPE_PER_STREAM, SCOPE_PER_FRAME = 0, 1, 2
ORDER_DENSITY, ORDER_AREA, ORDER_HEIGHT = 0, 1, 2
DENSITY_SPAN, DENSITY_MEMBERS = 0, 1


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread", "-ffp-contract=off",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            _lib = ctypes.CDLL(_LIB)
            _lib.ref_input_value.restype = ctypes.c_double
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _i64p():
    return ctypes.c_int64(0)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round fp32 values to bf16 (round to nearest even), returned as fp32."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


# ----------------------------------------------------------------------------------- steps

def select(importance: np.ndarray, W: int, H: int, mode: int, k: int, tau: float = 0.0,
           scope: int = SCOPE_GLOBAL, mb: int = 16, cap: int = -1) -> np.ndarray:
    """O2: uint8 [S][F][GH][GW] selection mask (cap >= 0: capacity N of P:663)."""
    imp = np.ascontiguousarray(importance, np.float32)
    S, F = imp.shape[:2]
    sel = np.zeros(imp.shape, np.uint8)
    rc = lib().ref_select(S, F, W, H, mb, mode, ctypes.c_int64(k), ctypes.c_float(tau), scope, ctypes.c_int64(cap),
                          _p(imp), _p(sel))
    assert rc == 0
    return sel


def regions(sel: np.ndarray, W: int, H: int, conn: int = 8, mb: int = 16):
    """O3 (Alg.1 l.3): labels int32 [S][F][GH][GW], regions int32 [n][8]."""
    sel = np.ascontiguousarray(sel, np.uint8)
    S, F = sel.shape[:2]
    labels = np.empty(sel.shape, np.int32)
    cap = int(sel.sum()) + 1
    regs = np.zeros((cap, 8), np.int32)
    n = _i64p()
    rc = lib().ref_regions(S, F, W, H, mb, conn, _p(sel), _p(labels), _p(regs), ctypes.c_int64(cap), ctypes.byref(n))
    assert rc == 0
    return labels, regs[: n.value].copy()


def boxes(importance: np.ndarray, labels: np.ndarray, regs: np.ndarray, W: int, H: int,
          expand: int = 3, partition_mb: int = 4, mb: int = 16, density_mode: int = DENSITY_SPAN):
    """O4 (Alg.1 l.4-6): boxes int32 [n][12], density f64 [n], box_of_mb int32 [S][F][GH][GW]."""
    imp = np.ascontiguousarray(importance, np.float32)
    labels = np.ascontiguousarray(labels, np.int32)
    regs = np.ascontiguousarray(regs, np.int32)
    S, F = imp.shape[:2]
    cap = int((labels >= 0).sum()) + 1
    bx = np.zeros((cap, 12), np.int32)
    dens = np.zeros(cap, np.float64)
    owner = np.empty(labels.shape, np.int32)
    n = _i64p()
    rc = lib().ref_boxes(S, F, W, H, mb, expand, partition_mb, density_mode, _p(imp), _p(labels), _p(regs),
                         ctypes.c_int64(len(regs)), _p(bx), _p(dens), ctypes.c_int64(cap), ctypes.byref(n), _p(owner))
    assert rc == 0
    return bx[: n.value].copy(), dens[: n.value].copy(), owner


def sort(bx: np.ndarray, density: np.ndarray, policy: int = ORDER_DENSITY) -> np.ndarray:
    """O5a (Alg.1 l.6): int32 permutation, packing order."""
    bx = np.ascontiguousarray(bx, np.int32)
    density = np.ascontiguousarray(density, np.float64)
    order = np.zeros(max(len(bx), 1), np.int32)
    lib().ref_sort(ctypes.c_int64(len(bx)), _p(bx), _p(density), policy, _p(order))
    return order[: len(bx)].copy()


POLICY_GUILLOTINE, POLICY_MAXRECT, POLICY_SKYLINE, POLICY_SHELF = 0, 1, 2, 3
_PACK_FN = {POLICY_GUILLOTINE: "ref_pack", POLICY_MAXRECT: "ref_pack_maxrect", POLICY_SKYLINE: "ref_pack_skyline",
            POLICY_SHELF: "ref_pack_shelf"}


def pack(bx: np.ndarray, order: np.ndarray, bin_w: int, bin_h: int, max_bins: int, gutter: int = 1,
         policy: int = POLICY_GUILLOTINE):
    """O5b (Alg.1 l.7-21, Alg.2): placement int32 [n][4] (bin,bx,by,rot), num_bins. policy: the
    guillotine reading (D6), or MAXRECT (D14), SKYLINE (D15), SHELF (D16)."""
    bx = np.ascontiguousarray(bx, np.int32)
    order = np.ascontiguousarray(order, np.int32)
    pl = np.zeros((max(len(bx), 1), 4), np.int32)
    nb = ctypes.c_int32(0)
    rc = getattr(lib(), _PACK_FN[policy])(ctypes.c_int64(len(bx)), _p(bx), _p(order), bin_w, bin_h, max_bins,
                                          gutter, _p(pl), ctypes.byref(nb))
    assert rc == 0
    return pl[: len(bx)].copy(), int(nb.value)


def max_empty_rect(occ: np.ndarray) -> tuple[int, int, int, int]:
    """Alg. 2 (reading D14) on a [Hg][W] occupancy grid (nonzero = used): (x, y, w, h)."""
    o = np.ascontiguousarray(occ != 0, np.uint8)
    out = np.zeros(4, np.int32)
    lib().ref_max_empty_rect(_p(o), o.shape[1], o.shape[0], _p(out))
    return tuple(int(v) for v in out)


def inner_free(fw: int, fh: int, uw: int, uh: int) -> list[tuple[int, int, int, int]]:
    """Alg. 2 InnerFree under reading D6: remainders (dx, dy, w, h) in listed order."""
    out = np.zeros(8, np.int32)
    n = lib().ref_inner_free(fw, fh, uw, uh, _p(out))
    return [tuple(int(v) for v in out[4 * i: 4 * i + 4]) for i in range(n)]


def mb_owner(box_of_mb: np.ndarray, placement: np.ndarray) -> np.ndarray:
    """Owner box of each selected MB whose box was placed, else -1 (reading D9)."""
    own = box_of_mb.copy()
    sel = own >= 0
    if len(placement):
        placed = placement[:, 0] >= 0
        own[sel] = np.where(placed[own[sel]], own[sel], -1)
    return own


def input_value(u: int, bf16: bool) -> float:
    return lib().ref_input_value(ctypes.c_uint8(u), int(bf16))


def gather(frames: np.ndarray, bx: np.ndarray, placement: np.ndarray, bin_w: int, bin_h: int,
           num_bins: int, bf16: bool) -> np.ndarray:
    """O6: LR bins fp64 [num_bins][bin_h][bin_w][3]."""
    fr = np.ascontiguousarray(frames, np.uint8)
    S, F, H, W = fr.shape[:4]
    lr = np.zeros((max(num_bins, 0), bin_h, bin_w, 3), np.float64)
    lib().ref_gather(S, F, W, H, _p(fr), ctypes.c_int64(len(bx)), _p(np.ascontiguousarray(bx, np.int32)),
                     _p(np.ascontiguousarray(placement, np.int32)), bin_w, bin_h, num_bins, int(bf16), _p(lr))
    return lr


def sr_weights_for(cfg, weights: np.ndarray) -> np.ndarray:
    """fp64 weights as the network uses them: conv weights rounded to bf16 for the bf16 path
    (reading D11: weight quantisation is part of the bf16 model, biases stay fp32)."""
    w = np.asarray(weights, np.float32).copy()
    if cfg.bf16:
        off = 0
        for ci, co in cfg.conv_shapes():
            n = co * ci * 9
            w[off: off + n] = round_bf16(w[off: off + n])
            off += n + co
    return w.astype(np.float64)


def conv3x3(x: np.ndarray, w: np.ndarray, b: np.ndarray) -> np.ndarray:
    """[Cin][H][W] fp64 -> [Cout][H][W], zero padding 1."""
    x = np.ascontiguousarray(x, np.float64)
    w = np.ascontiguousarray(w, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    Cin, Hh, Ww = x.shape
    Cout = w.shape[0]
    out = np.zeros((Cout, Hh, Ww), np.float64)
    lib().ref_conv3x3(_p(x), Cin, Hh, Ww, _p(w), _p(b), Cout, _p(out))
    return out


def pixel_shuffle(x: np.ndarray, s: int) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    Cin, Hh, Ww = x.shape
    out = np.zeros((Cin // (s * s), Hh * s, Ww * s), np.float64)
    lib().ref_pixel_shuffle(_p(x), Cin, Hh, Ww, s, _p(out))
    return out


def sr_crop(cfg, w64: np.ndarray, crop: np.ndarray) -> np.ndarray:
    """O7 on one crop: [3][h][w] fp64 -> [3][s h][s w]."""
    crop = np.ascontiguousarray(crop, np.float64)
    _, Hh, Ww = crop.shape
    out = np.zeros((3, Hh * cfg.scale, Ww * cfg.scale), np.float64)
    rc = lib().ref_sr_crop(cfg.scale, cfg.channels, cfg.n_resblocks, ctypes.c_double(cfg.res_scale),
                           _p(np.ascontiguousarray(w64, np.float64)), _p(crop), Hh, Ww, _p(out))
    assert rc == 0
    return out


def host_cores() -> int:
    """Host cores this process may run on (the thread count of the multi-threaded entries)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def enhance(cfg, w64: np.ndarray, lr: np.ndarray, bx: np.ndarray, placement: np.ndarray,
            box_lo: int = 0, box_hi: int | None = None, threads: int = 1) -> np.ndarray:
    """O7b: HR bins fp64 [num_bins][s bin_h][s bin_w][3] (boxes [box_lo, box_hi) only).
    threads > 1: ref_enhance_mt (the same per-box function over POSIX threads, bit-identical)."""
    nb, bh, bw = lr.shape[:3]
    s = cfg.scale
    hr = np.zeros((nb, s * bh, s * bw, 3), np.float64)
    box_hi = len(bx) if box_hi is None else box_hi
    args = [s, cfg.channels, cfg.n_resblocks, ctypes.c_double(cfg.res_scale),
            _p(np.ascontiguousarray(w64, np.float64)), _p(np.ascontiguousarray(lr, np.float64)),
            bw, bh, nb, ctypes.c_int64(len(bx)), _p(np.ascontiguousarray(bx, np.int32)),
            _p(np.ascontiguousarray(placement, np.int32)), ctypes.c_int64(box_lo), ctypes.c_int64(box_hi), _p(hr)]
    rc = lib().ref_enhance_mt(*args, int(threads)) if threads > 1 else lib().ref_enhance(*args)
    assert rc == 0
    return hr


def scatter(frames: np.ndarray, bx: np.ndarray, placement: np.ndarray, owner: np.ndarray, hr: np.ndarray,
            scale: int, bin_w: int, bin_h: int, f_lo: int = 0, f_hi: int | None = None, mb: int = 16,
            threads: int = 1) -> np.ndarray:
    """O8: HR frames fp64 [f_hi-f_lo][s H][s W][3] of the flat (stream, frame) range.
    threads > 1: ref_scatter_mt (same per-frame function over POSIX threads, bit-identical)."""
    fr = np.ascontiguousarray(frames, np.uint8)
    S, F, H, W = fr.shape[:4]
    f_hi = S * F if f_hi is None else f_hi
    out = np.zeros((f_hi - f_lo, scale * H, scale * W, 3), np.float64)
    hr = np.ascontiguousarray(hr, np.float64)
    if hr.size == 0:
        hr = np.zeros(1, np.float64)
    args = [S, F, W, H, mb, scale, _p(fr), _p(np.ascontiguousarray(bx, np.int32)),
            _p(np.ascontiguousarray(placement, np.int32)), _p(np.ascontiguousarray(owner, np.int32)),
            _p(hr), bin_w, bin_h, ctypes.c_int64(f_lo), ctypes.c_int64(f_hi), _p(out)]
    if threads > 1:
        lib().ref_scatter_mt(*args, int(threads))
    else:
        lib().ref_scatter(*args)
    return out


def quantize_u8(frames: np.ndarray, owner: np.ndarray, hr_frames: np.ndarray, scale: int, f_lo: int = 0,
                f_hi: int | None = None, mb: int = 16) -> np.ndarray:
    """D20 u8 output of O8's frames [f_lo, f_hi): pasted pixels rhe(clamp(v,0,1)*255) of the fp64
    value, bilinear pixels D10 * 255 exactly (integer weights over (2s)^2), round half to even."""
    fr = np.ascontiguousarray(frames, np.uint8)
    S, F, H, W = fr.shape[:4]
    f_hi = S * F if f_hi is None else f_hi
    hr = np.ascontiguousarray(hr_frames, np.float64)
    assert hr.shape == (f_hi - f_lo, scale * H, scale * W, 3)
    out = np.zeros(hr.shape, np.uint8)
    rc = lib().ref_quantize_u8(S, F, W, H, mb, scale, _p(fr), _p(np.ascontiguousarray(owner, np.int32)), _p(hr),
                               ctypes.c_int64(f_lo), ctypes.c_int64(f_hi), _p(out))
    assert rc == 0
    return out


# ----------------------------------------------------------------------------------- pipeline

def index_path(importance: np.ndarray, W: int, H: int, k: int, *, mode: int = MODE_TOPK, tau: float = 0.0,
               scope: int = SCOPE_GLOBAL, conn: int = 8, expand: int = 3, partition_mb: int = 4,
               bin_w: int = 128, bin_h: int = 128, max_bins: int = 4096, gutter: int = 1,
               order_policy: int = ORDER_DENSITY, cap: int = -1, density_mode: int = DENSITY_SPAN,
               policy: int = POLICY_GUILLOTINE) -> dict:
    """Selection -> regions -> boxes -> sort -> pack, in Alg. 1's order."""
    sel = select(importance, W, H, mode, k, tau, scope, cap=cap)
    labels, regs = regions(sel, W, H, conn)
    bx, dens, box_of = boxes(importance, labels, regs, W, H, expand, partition_mb, density_mode=density_mode)
    order = sort(bx, dens, order_policy)
    pl, nbins = pack(bx, order, bin_w, bin_h, max_bins, gutter, policy)
    return dict(sel=sel, labels=labels, regions=regs, boxes=bx, density=dens, box_of_mb=box_of,
                order=order, placement=pl, num_bins=nbins, owner=mb_owner(box_of, pl))


def run_workload(wl, importance: np.ndarray, frames: np.ndarray, weights: np.ndarray,
                 box_range: tuple[int, int] | None = None, frame_range: tuple[int, int] | None = None) -> dict:
    """The whole hot path of one selection group (synth.Workload), oracle side."""
    ip = index_path(importance, wl.W, wl.H, wl.k, partition_mb=wl.partition_mb, bin_w=wl.bin_w,
                    bin_h=wl.bin_h, max_bins=wl.max_bins)
    lr = gather(frames, ip["boxes"], ip["placement"], wl.bin_w, wl.bin_h, ip["num_bins"], wl.sr.bf16)
    w64 = sr_weights_for(wl.sr, weights)
    lo, hi = box_range if box_range is not None else (0, len(ip["boxes"]))
    hr = enhance(wl.sr, w64, lr, ip["boxes"], ip["placement"], lo, hi)
    f_lo, f_hi = frame_range if frame_range is not None else (0, wl.S * wl.F)
    out = scatter(frames, ip["boxes"], ip["placement"], ip["owner"], hr, wl.sr.scale, wl.bin_w, wl.bin_h, f_lo, f_hi)
    ip.update(lr=lr, hr=hr, out=out)
    return ip


def nv12_to_rgb8(nv12: np.ndarray, W: int, H: int) -> np.ndarray:
    """f4 (reading D19): uint8 NV12 frames [..., H*W*3/2] -> RGB8 [..., H, W, 3]."""
    a = np.ascontiguousarray(nv12, np.uint8)
    lead = a.shape[:-1]
    frames = int(np.prod(lead)) if lead else 1
    out = np.zeros(lead + (H, W, 3), np.uint8)
    lib().ref_nv12_to_rgb8(ctypes.c_int64(frames), W, H, _p(a), _p(out))
    return out


# ----------------------------------------------------------------------------------- temporal reuse
# SURVEY §8(f)3, §3.2.2 P:584-609. Phi (CCL + exact sum) is C (ref_phi_inv_area); the series, CDF
# pick and budget allocation are plain Python floats (IEEE fp64, one operation at a time in the
# order written), the order the CUDA kernel follows (readings D18 in DESIGN.md).

def phi_inv_area(res_frame: np.ndarray, thr: int) -> tuple[float, int]:
    """The 1/Area operator of one frame: (Phi, number of components)."""
    r = np.ascontiguousarray(res_frame, np.int16)
    H, W = r.shape
    n = ctypes.c_int64(0)
    f = lib().ref_phi_inv_area
    f.restype = ctypes.c_double
    return float(f(W, H, _p(r), int(thr), ctypes.byref(n))), int(n.value)


def phi_series(residual: np.ndarray, thr: int) -> np.ndarray:
    """Phi of every frame: [S][F] fp64 from the [S][F][H][W] int16 Y residuals."""
    S, F = residual.shape[:2]
    return np.array([[phi_inv_area(residual[s, f], thr)[0] for f in range(F)] for s in range(S)], np.float64)


def delta_series(phi: list[float]) -> tuple[list[float], float, list[float], list[float]]:
    """(|dPhi_i| for i = 0..F-2, T = their sum, S = Norm(|dPhi|) (L1), CDF M[k] = sum_{i<k} S_i
    for k = 1..F-1 (M[0] = 0)): dPhi_i = Phi_{i+1} - Phi_i belongs to frame i+1."""
    F = len(phi)
    a = [abs(phi[i + 1] - phi[i]) for i in range(F - 1)]
    T = 0.0
    for x in a:
        T = T + x
    Sn = [x / T if T > 0.0 else 0.0 for x in a]
    M = [0.0] * F
    m = 0.0
    for k in range(1, F):
        m = m + Sn[k - 1]
        M[k] = m
    return a, T, Sn, M


def allocate_budget(totals: list[float], budget: int, F: int) -> list[int]:
    """Frames per stream: each stream keeps its anchor frame; the rest of the budget is shared
    by the ratio sum_i |dPhi_ij| / sum_j sum_i |dPhi_ij| with the largest-remainder rule (ties: lower
    stream), each capped at F. The budget is clamped to [S, S*F]."""
    S = len(totals)
    B = min(max(budget, S), S * F)
    rest = B - S
    Tsum = 0.0
    for t in totals:
        Tsum = Tsum + t
    q = [(float(rest) * t) / Tsum if Tsum > 0.0 else float(rest) / float(S) for t in totals]
    fl = [math.floor(x) for x in q]
    rem = [q[j] - fl[j] for j in range(S)]
    n = [1 + fl[j] for j in range(S)]
    left = rest - sum(fl)
    for j in sorted(range(S), key=lambda j: (-rem[j], j))[:max(left, 0)]:
        n[j] += 1
    return [min(x, F) for x in n]


def cdf_pick(M: list[float], n: int, F: int) -> list[int]:
    """Frame 0 (the anchor) and, for N = n - 1 even intervals of the CDF's y axis, the
    smallest frame k >= 1 with M[k] >= (t + 0.5) / N; duplicates collapse."""
    sel = {0}
    N = n - 1
    for t in range(N):
        y = (t + 0.5) / N
        for k in range(1, F):
            if M[k] >= y:
                sel.add(k)
                break
    return sorted(sel)


def temporal_select(residual: np.ndarray, thr: int, budget: int) -> dict:
    """The whole §3.2.2 step for one chunk: phi [S][F], selected [S][F] u8, reuse [S][F] (the nearest
    selected frame at or before f), frames_per_stream [S]."""
    S, F = residual.shape[:2]
    phi = phi_series(residual, thr)
    series = [delta_series(list(phi[s])) for s in range(S)]
    n = allocate_budget([t for _, t, _, _ in series], budget, F)
    selected = np.zeros((S, F), np.uint8)
    reuse = np.zeros((S, F), np.int32)
    for s in range(S):
        for f in cdf_pick(series[s][3], n[s], F):
            selected[s, f] = 1
        last = 0
        for f in range(F):
            last = f if selected[s, f] else last
            reuse[s, f] = last
    return dict(phi=phi, selected=selected, reuse=reuse, frames_per_stream=np.array(n, np.int32))
