"""Python binding of libregen (include/regen.h): the B200 region-aware enhancement hot path of
RegenHance (arXiv 2407.16990).

Argument marshalling only: every step of the path runs in the CUDA kernels of libregen.so; this
module converts torch CUDA tensors to raw pointers, passes the current CUDA stream, and owns the
buffers of a `Pipeline`. There is no CPU fallback: importing fails loudly if libregen.so cannot be
loaded, and every call raises on a non-OK status.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libregen.so")

REGEN_OK, REGEN_E_INVALID, REGEN_E_CAPACITY, REGEN_E_CUDA, REGEN_E_UNSUPPORTED = range(5)
MODE_TOPK, MODE_THRESHOLD = 0, 1
SCOPE_GLOBAL, SCOPE_PER_STREAM, SCOPE_PER_FRAME = 0, 1, 2
ORDER_DENSITY, ORDER_AREA, ORDER_HEIGHT = 0, 1, 2
POLICY_GUILLOTINE, POLICY_MAXRECT, POLICY_SKYLINE, POLICY_SHELF = 0, 1, 2, 3
DENSITY_SPAN, DENSITY_MEMBERS = 0, 1
FORMAT_RGB8, FORMAT_NV12 = 0, 1
DTYPE_BF16, DTYPE_FP32, DTYPE_U8 = 0, 1, 2   # U8: output frames only (D20)
CALL_SELECT, CALL_PACK, CALL_ENHANCE, CALL_SCATTER, CALL_ENHANCE_SCATTER, CALL_TEMPORAL = 0, 1, 2, 3, 4, 5
ST_REGION_OVERFLOW, ST_BOX_OVERFLOW, ST_FREELIST_OVERFLOW, ST_TOPK_INCOMPLETE = 1, 2, 4, 8
TOPK_STATE_BYTES, TOPK_DIGITS = 24, 1 << 16

EXPORTED = ["regen_select_mbs", "regen_pack_regions", "regen_sr_create", "regen_sr_destroy", "regen_stitch_bins",
            "regen_enhance_packed", "regen_scatter_blend", "regen_workspace_size", "regen_capacity_mbs",
            "regen_status_string", "regen_last_error", "regen_abi_version", "regen_enhance_kernel_count",
            "regen_enhance_scatter", "regen_trace_enable", "regen_trace_read", "regen_trace_filter",
            "regen_enhance_owned", "regen_scatter_bilinear", "regen_topk_init", "regen_topk_histogram",
            "regen_topk_pick", "regen_select_mbs_global", "regen_temporal_select", "regen_reuse_importance",
            "regen_nv12_to_rgb8", "regen_enhance_partials", "regen_fold_combine_frames"]


class Geom(ctypes.Structure):
    _fields_ = [("S", ctypes.c_int32), ("F", ctypes.c_int32), ("frame_w", ctypes.c_int32),
                ("frame_h", ctypes.c_int32), ("mb", ctypes.c_int32), ("format", ctypes.c_int32)]


class SelectParams(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("scope", ctypes.c_int32), ("k", ctypes.c_int64), ("tau", ctypes.c_float),
                ("connectivity", ctypes.c_int32), ("cap", ctypes.c_int64)]


class PackParams(ctypes.Structure):
    _fields_ = [("bin_w", ctypes.c_int32), ("bin_h", ctypes.c_int32), ("max_bins", ctypes.c_int32),
                ("expand", ctypes.c_int32), ("partition_mb", ctypes.c_int32), ("gutter", ctypes.c_int32),
                ("order", ctypes.c_int32), ("policy", ctypes.c_int32), ("density", ctypes.c_int32)]


class SRConfig(ctypes.Structure):
    _fields_ = [("scale", ctypes.c_int32), ("channels", ctypes.c_int32), ("n_resblocks", ctypes.c_int32),
                ("dtype", ctypes.c_int32), ("res_scale", ctypes.c_float), ("bin_w", ctypes.c_int32)]


REGION_DTYPE = np.dtype([("stream", "<i4"), ("frame", "<i4"), ("root", "<i4"), ("mx0", "<i4"), ("my0", "<i4"),
                         ("mx1", "<i4"), ("my1", "<i4"), ("n_members", "<i4")])
BOX_DTYPE = np.dtype([("stream", "<i4"), ("frame", "<i4"), ("mx0", "<i4"), ("my0", "<i4"), ("mx1", "<i4"),
                      ("my1", "<i4"), ("x0", "<i4"), ("y0", "<i4"), ("w", "<i4"), ("h", "<i4"),
                      ("n_members", "<i4"), ("region", "<i4"), ("density", "<f8"), ("bin", "<i4"), ("bx", "<i4"),
                      ("by", "<i4"), ("rotated", "<i4"), ("rank", "<i4"), ("reserved", "<i4")])
assert REGION_DTYPE.itemsize == 32 and BOX_DTYPE.itemsize == 80


class RegenError(RuntimeError):
    pass


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libregen.so not built at {LIB_PATH}; run __graft_entry__.build() "
                          f"(python paper_2407_16990_b200/build.py)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    P = ctypes.POINTER
    lib.regen_select_mbs.argtypes = [P(Geom), P(SelectParams), vp, vp, vp, vp, i64, vp, vp, vp, sz, vp]
    lib.regen_pack_regions.argtypes = [P(Geom), P(PackParams), vp, vp, vp, vp, vp, i64, vp, vp, vp, vp, vp, vp, sz,
                                       vp]
    lib.regen_sr_create.argtypes = [P(SRConfig), vp, sz, P(vp)]
    lib.regen_sr_destroy.argtypes = [vp]
    lib.regen_stitch_bins.argtypes = [P(Geom), P(PackParams), i32, vp, vp, i64, vp, vp, vp, vp, sz, vp]
    lib.regen_enhance_packed.argtypes = [vp, P(Geom), P(PackParams), vp, vp, i64, vp, vp, vp, vp, vp, sz, vp]
    lib.regen_scatter_blend.argtypes = [P(Geom), P(PackParams), i32, vp, vp, vp, vp, i32, vp, i32, vp]
    lib.regen_enhance_scatter.argtypes = [vp, P(Geom), P(PackParams), vp, vp, i64, vp, vp, vp, vp, i32, vp, vp, sz,
                                          vp]
    lib.regen_enhance_owned.argtypes = list(lib.regen_enhance_scatter.argtypes)
    lib.regen_scatter_bilinear.argtypes = [P(Geom), i32, vp, vp, vp, i32, vp]
    lib.regen_workspace_size.argtypes = [i32, P(Geom), vp, vp, P(sz)]
    lib.regen_topk_init.argtypes = [i64, vp, vp]
    lib.regen_nv12_to_rgb8.argtypes = [P(Geom), vp, vp, vp]
    lib.regen_enhance_partials.argtypes = [vp, P(Geom), P(PackParams), vp, vp, i64, vp, vp, vp, vp, vp, sz, vp]
    lib.regen_fold_combine_frames.argtypes = [vp, P(Geom), P(PackParams), vp, vp, vp, vp, i32, vp, sz, vp]
    lib.regen_temporal_select.argtypes = [P(Geom), vp, i32, i64, vp, vp, vp, vp, vp, sz, vp]
    lib.regen_reuse_importance.argtypes = [P(Geom), vp, vp, vp, vp]
    lib.regen_topk_histogram.argtypes = [P(Geom), i64, vp, vp, vp, vp]
    lib.regen_topk_pick.argtypes = [vp, vp, vp]
    lib.regen_select_mbs_global.argtypes = [P(Geom), P(SelectParams), i64, vp, vp, vp, vp, vp, i64, vp, vp, vp, sz, vp]
    lib.regen_enhance_kernel_count.argtypes = [vp, P(PackParams), P(i32)]
    lib.regen_trace_enable.argtypes = [i32]
    lib.regen_trace_read.argtypes = [vp, vp, i32, P(i32)]
    lib.regen_trace_filter.argtypes = [ctypes.c_char_p]
    lib.regen_capacity_mbs.argtypes = [i32, i32, i32, i32]
    lib.regen_capacity_mbs.restype = i64
    lib.regen_status_string.restype = ctypes.c_char_p
    lib.regen_last_error.restype = ctypes.c_char_p
    lib.regen_abi_version.restype = i32
    for name in EXPORTED:
        if name not in ("regen_capacity_mbs", "regen_status_string", "regen_last_error", "regen_abi_version"):
            getattr(lib, name).restype = ctypes.c_int
    return lib


lib = _load()


def _check(rc: int, what: str):
    if rc != REGEN_OK:
        raise RegenError(f"{what}: {lib.regen_status_string(rc).decode()}: {lib.regen_last_error().decode()}")


def _ptr(t):
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


TRACE_NAME_LEN = 32


def trace_enable(on: bool = True):
    """Bracket every libregen kernel launch with CUDA events on its stream (regen_trace_enable)."""
    _check(lib.regen_trace_enable(1 if on else 0), "regen_trace_enable")


def trace_filter(prefix: str | None = None):
    """Trace only kernels whose name starts with `prefix` (None = all)."""
    _check(lib.regen_trace_filter(prefix.encode() if prefix else None), "regen_trace_filter")


def trace_read(cap: int = 1 << 16) -> list:
    """[(kernel name, device ms)] of the launches recorded since the last read, in launch order."""
    names = ctypes.create_string_buffer(cap * TRACE_NAME_LEN)
    ms = (ctypes.c_float * cap)()
    n = ctypes.c_int32(0)
    _check(lib.regen_trace_read(names, ms, cap, ctypes.byref(n)), "regen_trace_read")
    raw = names.raw
    return [(raw[i * TRACE_NAME_LEN:(i + 1) * TRACE_NAME_LEN].split(b"\0", 1)[0].decode(), float(ms[i]))
            for i in range(min(n.value, cap))]


def capacity_mbs(bin_w: int, bin_h: int, n_bins: int, mb: int = 16) -> int:
    """max N with MB_size * N <= H * W * B."""
    return int(lib.regen_capacity_mbs(bin_w, bin_h, n_bins, mb))


def workspace_size(which: int, geom: Geom, params=None, sr=None) -> int:
    n = ctypes.c_size_t(0)
    pp = ctypes.byref(params) if params is not None else None
    _check(lib.regen_workspace_size(which, ctypes.byref(geom), pp, sr, ctypes.byref(n)), "workspace_size")
    return int(n.value)


# ----------------------------------------------------------------------------- the four calls

def select_mbs(geom, params, importance, sel_bitmap, labels, regions, max_regions, num_regions, status, ws,
               stream=None):
    _check(lib.regen_select_mbs(ctypes.byref(geom), ctypes.byref(params), _ptr(importance), _ptr(sel_bitmap),
                                _ptr(labels), _ptr(regions), max_regions, _ptr(num_regions), _ptr(status), _ptr(ws),
                                ws.numel() * ws.element_size(), _stream(stream)), "regen_select_mbs")


def pack_regions(geom, params, importance, labels, regions, num_regions, boxes, max_boxes, num_boxes, order,
                 num_bins, mb_owner, status, ws, stream=None):
    _check(lib.regen_pack_regions(ctypes.byref(geom), ctypes.byref(params), _ptr(importance), _ptr(labels),
                                  _ptr(regions), _ptr(num_regions), _ptr(boxes), max_boxes, _ptr(num_boxes),
                                  _ptr(order), _ptr(num_bins), _ptr(mb_owner), _ptr(status), _ptr(ws),
                                  ws.numel() * ws.element_size(), _stream(stream)), "regen_pack_regions")


def topk_init(k, state, stream=None):
    _check(lib.regen_topk_init(k, _ptr(state), _stream(stream)), "regen_topk_init")


def topk_histogram(geom, stream0, importance, state, hist, stream=None):
    _check(lib.regen_topk_histogram(ctypes.byref(geom), stream0, _ptr(importance), _ptr(state), _ptr(hist),
                                    _stream(stream)), "regen_topk_histogram")


def topk_pick(hist, state, stream=None):
    _check(lib.regen_topk_pick(_ptr(hist), _ptr(state), _stream(stream)), "regen_topk_pick")


def select_mbs_global(geom, params, stream0, importance, state, sel_bitmap, labels, regions, max_regions, num_regions,
                      status, ws, stream=None):
    _check(lib.regen_select_mbs_global(ctypes.byref(geom), ctypes.byref(params), stream0, _ptr(importance), _ptr(state),
                                       _ptr(sel_bitmap), _ptr(labels), _ptr(regions), max_regions, _ptr(num_regions),
                                       _ptr(status), _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)),
           "regen_select_mbs_global")


def nv12_to_rgb8(geom, nv12, rgb8, stream=None):
    _check(lib.regen_nv12_to_rgb8(ctypes.byref(geom), _ptr(nv12), _ptr(rgb8), _stream(stream)), "regen_nv12_to_rgb8")


def temporal_select(geom, residual_y, threshold, budget, phi, selected, reuse, frames_per_stream, ws, stream=None):
    _check(lib.regen_temporal_select(ctypes.byref(geom), _ptr(residual_y), threshold, budget, _ptr(phi), _ptr(selected),
                                     _ptr(reuse), _ptr(frames_per_stream), _ptr(ws), ws.numel() * ws.element_size(),
                                     _stream(stream)), "regen_temporal_select")


def reuse_importance(geom, pred, reuse, out, stream=None):
    _check(lib.regen_reuse_importance(ctypes.byref(geom), _ptr(pred), _ptr(reuse), _ptr(out), _stream(stream)),
           "regen_reuse_importance")


class TemporalReuse:
    """Buffers of regen_temporal_select for one chunk of S streams x F frames."""

    def __init__(self, S, F, W, H, threshold=8, device="cuda"):
        import torch
        self.geom = Geom(S, F, W, H, 16)
        self.threshold = threshold
        self.phi = torch.zeros((S, F), dtype=torch.float64, device=device)
        self.selected = torch.zeros((S, F), dtype=torch.uint8, device=device)
        self.reuse = torch.zeros((S, F), dtype=torch.int32, device=device)
        self.frames = torch.zeros(S, dtype=torch.int32, device=device)
        self.ws = torch.empty(workspace_size(CALL_TEMPORAL, self.geom), dtype=torch.uint8, device=device)

    def run(self, residual_y, budget, stream=None):
        temporal_select(self.geom, residual_y, self.threshold, budget, self.phi, self.selected, self.reuse, self.frames,
                        self.ws, stream)

    def reuse_maps(self, pred, out, stream=None):
        reuse_importance(self.geom, pred, self.reuse, out, stream)
        return out


def stitch_bins(geom, params, dtype, frames, boxes, max_boxes, num_boxes, num_bins, lr_bins, ws, stream=None):
    _check(lib.regen_stitch_bins(ctypes.byref(geom), ctypes.byref(params), dtype, _ptr(frames), _ptr(boxes),
                                 max_boxes, _ptr(num_boxes), _ptr(num_bins), _ptr(lr_bins), _ptr(ws),
                                 ws.numel() * ws.element_size(), _stream(stream)), "regen_stitch_bins")


def enhance_packed(sr, geom, params, frames, boxes, max_boxes, num_boxes, num_bins, hr_bins, status, ws,
                   stream=None):
    _check(lib.regen_enhance_packed(sr.handle, ctypes.byref(geom), ctypes.byref(params), _ptr(frames),
                                    _ptr(boxes), max_boxes, _ptr(num_boxes), _ptr(num_bins), _ptr(hr_bins),
                                    _ptr(status), _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)),
           "regen_enhance_packed")


def enhance_scatter(sr, geom, params, frames, boxes, max_boxes, num_boxes, num_bins, mb_owner, out, out_dtype, status,
                    ws, stream=None):
    _check(lib.regen_enhance_scatter(sr.handle, ctypes.byref(geom), ctypes.byref(params), _ptr(frames), _ptr(boxes),
                                     max_boxes, _ptr(num_boxes), _ptr(num_bins), _ptr(mb_owner), _ptr(out), out_dtype,
                                     _ptr(status), _ptr(ws), ws.numel(), _stream(stream)), "regen_enhance_scatter")


def enhance_owned(sr, geom, params, frames, boxes, max_boxes, num_boxes, num_bins, mb_owner, out, out_dtype, status,
                  ws, stream=None):
    _check(lib.regen_enhance_owned(sr.handle, ctypes.byref(geom), ctypes.byref(params), _ptr(frames), _ptr(boxes),
                                   max_boxes, _ptr(num_boxes), _ptr(num_bins), _ptr(mb_owner), _ptr(out), out_dtype,
                                   _ptr(status), _ptr(ws), ws.numel(), _stream(stream)), "regen_enhance_owned")


def scatter_bilinear(geom, scale, frames, mb_owner, out, out_dtype, stream=None):
    _check(lib.regen_scatter_bilinear(ctypes.byref(geom), scale, _ptr(frames), _ptr(mb_owner), _ptr(out), out_dtype,
                                      _stream(stream)), "regen_scatter_bilinear")


def scatter_blend(geom, params, scale, frames, boxes, mb_owner, hr_bins, hr_dtype, out, out_dtype, stream=None):
    _check(lib.regen_scatter_blend(ctypes.byref(geom), ctypes.byref(params), scale, _ptr(frames), _ptr(boxes),
                                   _ptr(mb_owner), _ptr(hr_bins), hr_dtype, _ptr(out), out_dtype, _stream(stream)),
           "regen_scatter_blend")


class SRNet:
    """Owns a regen_sr_create handle (weights repacked on the device)."""

    def __init__(self, scale: int, channels: int, n_resblocks: int, weights: np.ndarray, bf16: bool = True,
                 res_scale: float = 1.0, bin_w: int = 128):
        self.cfg = SRConfig(scale, channels, n_resblocks, DTYPE_BF16 if bf16 else DTYPE_FP32, res_scale, bin_w)
        w = np.ascontiguousarray(weights, np.float32)
        h = ctypes.c_void_p(0)
        _check(lib.regen_sr_create(ctypes.byref(self.cfg), w.ctypes.data_as(ctypes.c_void_p), w.size,
                                   ctypes.byref(h)), "regen_sr_create")
        self.handle = h
        self.dtype = self.cfg.dtype

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and lib is not None:   # lib is None at interpreter shutdown
            lib.regen_sr_destroy(h)
            self.handle = None


class Pipeline:
    """All device buffers of one selection group (S streams x F frames) and the four ABI calls.

    run(importance, frames) executes select -> pack -> enhance -> scatter on the current stream
    without host synchronisation and returns the HR frames tensor (bf16 or fp32)."""

    def __init__(self, *, S, F, W, H, k, bin_w, bin_h, max_bins, partition_mb, scale, channels, n_resblocks,
                 weights, bf16=True, res_scale=1.0, mode=MODE_TOPK, tau=0.0, scope=SCOPE_GLOBAL, connectivity=8,
                 expand=3, gutter=1, order=ORDER_DENSITY, max_boxes=None, out_dtype=None, device="cuda", cap=-1,
                 policy=POLICY_GUILLOTINE, density=DENSITY_SPAN, frame_format=FORMAT_RGB8):
        import torch
        self.torch = torch
        self.geom = Geom(S, F, W, H, 16, frame_format)   # frame_format NV12: every call reads NV12 frames
        self.sel = SelectParams(mode, scope, k, tau, connectivity, cap)
        self.pack = PackParams(bin_w, bin_h, max_bins, expand, partition_mb, gutter, order, policy, density)
        self.sr = SRNet(scale, channels, n_resblocks, weights, bf16, res_scale, bin_w)
        self.scale = scale
        self.GW, self.GH = (W + 15) // 16, (H + 15) // 16
        self.n_mbs = S * F * self.GH * self.GW
        self.max_regions = self.n_mbs
        self.max_boxes = max_boxes if max_boxes is not None else self.n_mbs
        dev = torch.device(device)
        i32, i64, u8 = torch.int32, torch.int64, torch.uint8
        W32 = (self.GW + 31) // 32
        self.bitmap = torch.zeros(S * F * self.GH * W32, dtype=i32, device=dev)
        self.labels = torch.empty(self.n_mbs, dtype=i32, device=dev)
        self.regions = torch.empty(self.max_regions * 32, dtype=u8, device=dev)
        self.counts = torch.zeros(4, dtype=i64, device=dev)        # num_regions, num_boxes
        self.num_bins = torch.zeros(1, dtype=i32, device=dev)
        self.status = torch.zeros(1, dtype=i32, device=dev)
        self.boxes = torch.empty(self.max_boxes * 80, dtype=u8, device=dev)
        self.order = torch.empty(self.max_boxes, dtype=i32, device=dev)
        self.owner = torch.empty(self.n_mbs, dtype=i32, device=dev)
        # the workspace of the calls run() makes; the separate enhance call (HR bins) grows it on first use
        ws = max(workspace_size(CALL_SELECT, self.geom), workspace_size(CALL_PACK, self.geom, self.pack),
                 workspace_size(CALL_ENHANCE_SCATTER, self.geom, self.pack, self.sr.handle))
        self.ws = torch.empty(ws, dtype=u8, device=dev)
        self.hr_dtype = DTYPE_BF16 if bf16 else DTYPE_FP32
        self._hr_shape = (max_bins, scale * bin_h, scale * bin_w, 4)
        self._hr_bins = None   # allocated on first use of the separate enhance/scatter calls
        self.out_dtype = (DTYPE_BF16 if bf16 else DTYPE_FP32) if out_dtype is None else out_dtype
        self.out = torch.empty((S, F, scale * H, scale * W, 3),
                               dtype={DTYPE_BF16: torch.bfloat16, DTYPE_FP32: torch.float32,
                                      DTYPE_U8: torch.uint8}[self.out_dtype], device=dev)

    @property
    def hr_bins(self):
        if self._hr_bins is None:
            t = self.torch
            self._hr_bins = t.empty(self._hr_shape, dtype=t.bfloat16 if self.hr_dtype == DTYPE_BF16 else t.float32,
                                    device=self.out.device)
        return self._hr_bins

    @property
    def num_regions_t(self):
        return self.counts[0:1]

    @property
    def num_boxes_t(self):
        return self.counts[1:2]

    def select(self, importance, stream=None):
        # regen_select_mbs resets the status word on `stream` (the first call of a batch)
        select_mbs(self.geom, self.sel, importance, self.bitmap, self.labels, self.regions, self.max_regions,
                   self.counts[0:1], self.status, self.ws, stream)

    def select_global(self, importance, state, stream0, stream=None):
        """a1+a2 with the selection of a finished cross-rank top-N (regen_select_mbs_global; global_topk.py)."""
        select_mbs_global(self.geom, self.sel, stream0, importance, state, self.bitmap, self.labels, self.regions,
                          self.max_regions, self.counts[0:1], self.status, self.ws, stream)

    def pack_step(self, importance, stream=None):
        pack_regions(self.geom, self.pack, importance, self.labels, self.regions, self.counts[0:1], self.boxes,
                     self.max_boxes, self.counts[1:2], self.order, self.num_bins, self.owner, self.status, self.ws,
                     stream)

    def enhance(self, frames, stream=None):
        need = workspace_size(CALL_ENHANCE, self.geom, self.pack, self.sr.handle)
        if self.ws.numel() < need:
            self.ws = self.torch.empty(need, dtype=self.torch.uint8, device=self.out.device)
        enhance_packed(self.sr, self.geom, self.pack, frames, self.boxes, self.max_boxes, self.counts[1:2],
                       self.num_bins, self.hr_bins, self.status, self.ws, stream)

    def scatter(self, frames, out=None, stream=None):
        out = self.out if out is None else out
        scatter_blend(self.geom, self.pack, self.scale, frames, self.boxes, self.owner, self.hr_bins, self.hr_dtype,
                      out, self.out_dtype, stream)
        return out

    def enhance_scatter(self, frames, out=None, stream=None):
        """a6-a8 in one call (regen_enhance_scatter): HR frames without the HR-bin round trip."""
        out = self.out if out is None else out
        enhance_scatter(self.sr, self.geom, self.pack, frames, self.boxes, self.max_boxes, self.counts[1:2],
                        self.num_bins, self.owner, out, self.out_dtype, self.status, self.ws, stream)
        return out

    def enhance_owned(self, frames, out=None, stream=None):
        """regen_enhance_owned: the SR pixels of the owned MBs only."""
        out = self.out if out is None else out
        enhance_owned(self.sr, self.geom, self.pack, frames, self.boxes, self.max_boxes, self.counts[1:2],
                      self.num_bins, self.owner, out, self.out_dtype, self.status, self.ws, stream)
        return out

    def _split_ws(self):
        need = workspace_size(CALL_ENHANCE, self.geom, self.pack, self.sr.handle)
        if self.ws.numel() < need:
            self.ws = self.torch.empty(need, dtype=self.torch.uint8, device=self.out.device)
        return self.ws

    def enhance_partials(self, frames, stream=None):
        """regen_enhance_partials: the SR up to the UP∘TAIL fold's partial sums (kept in the workspace)."""
        ws = self._split_ws()
        _check(lib.regen_enhance_partials(self.sr.handle, ctypes.byref(self.geom), ctypes.byref(self.pack),
                                          _ptr(frames), _ptr(self.boxes), self.max_boxes, _ptr(self.counts[1:2]),
                                          _ptr(self.num_bins), _ptr(self.owner), _ptr(self.status), _ptr(ws),
                                          ws.numel(), _stream(stream)), "regen_enhance_partials")

    def fold_combine(self, out=None, stream=None):
        """regen_fold_combine_frames: the owned MBs' HR pixels from the partial sums of enhance_partials."""
        out = self.out if out is None else out
        ws = self._split_ws()
        _check(lib.regen_fold_combine_frames(self.sr.handle, ctypes.byref(self.geom), ctypes.byref(self.pack),
                                             _ptr(self.boxes), _ptr(self.num_bins), _ptr(self.owner), _ptr(out),
                                             self.out_dtype, _ptr(ws), ws.numel(), _stream(stream)),
               "regen_fold_combine_frames")
        return out

    def scatter_bilinear(self, frames, out=None, stream=None):
        """regen_scatter_bilinear: the bilinear pixels (MBs without an owner) only."""
        out = self.out if out is None else out
        scatter_bilinear(self.geom, self.scale, frames, self.owner, out, self.out_dtype, stream)
        return out

    def convert_nv12(self, nv12, stream=None):
        """NV12 decoder frames [S][F][H*W*3/2] u8 -> the RGB8 frames tensor the other calls read."""
        t = self.torch
        if getattr(self, "_rgb", None) is None:
            g = self.geom
            self._rgb = t.empty((g.S, g.F, g.frame_h, g.frame_w, 3), dtype=t.uint8, device=self.out.device)
        nv12_to_rgb8(Geom(self.geom.S, self.geom.F, self.geom.frame_w, self.geom.frame_h, 16), nv12, self._rgb, stream)
        return self._rgb

    def run(self, importance, frames, out=None, stream=None, fused=True):
        """select -> pack -> enhance -> scatter; fused=True uses regen_enhance_scatter for the last two."""
        self.select(importance, stream)
        self.pack_step(importance, stream)
        if fused:
            return self.enhance_scatter(frames, out, stream)
        self.enhance(frames, stream)
        return self.scatter(frames, out, stream)

    def enhance_kernels(self) -> int:
        """Kernels one enhance call launches (regen_enhance_kernel_count)."""
        n = ctypes.c_int32(0)
        _check(lib.regen_enhance_kernel_count(self.sr.handle, ctypes.byref(self.pack), ctypes.byref(n)),
               "regen_enhance_kernel_count")
        return int(n.value)

    def launches_per_step(self) -> int:
        """Kernels libregen launches per run(): select 4, pack 7, enhance (counted by the library), scatter 1."""
        return 4 + 7 + self.enhance_kernels() + 1

    # ---- host-side views (sync), for tests and reporting
    def host_results(self) -> dict:
        t = self.torch
        t.cuda.synchronize()
        nr, nb = (int(v) for v in self.counts[:2].cpu())
        regs = np.frombuffer(self.regions[: min(nr, self.max_regions) * 32].cpu().numpy().tobytes(), REGION_DTYPE)
        bx = np.frombuffer(self.boxes[: min(nb, self.max_boxes) * 80].cpu().numpy().tobytes(), BOX_DTYPE)
        S, F = self.geom.S, self.geom.F
        W32 = (self.GW + 31) // 32
        bm = self.bitmap.cpu().numpy().view(np.uint32).reshape(S, F, self.GH, W32)
        sel = np.zeros((S, F, self.GH, self.GW), np.uint8)
        for x in range(self.GW):
            sel[..., x] = (bm[..., x // 32] >> np.uint32(x % 32)) & 1
        return dict(sel=sel, labels=self.labels.cpu().numpy().reshape(S, F, self.GH, self.GW), regions=regs,
                    boxes=bx, order=self.order[: min(nb, self.max_boxes)].cpu().numpy(),
                    num_bins=int(self.num_bins.item()), owner=self.owner.cpu().numpy().reshape(S, F, self.GH, self.GW),
                    status=int(self.status.item()), num_regions=nr, num_boxes=nb)
