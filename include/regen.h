/*
 * regen.h — C-ABI of the B200 (sm_100a) region-aware enhancement hot path of RegenHance
 * (arXiv 2407.16990). Implemented by paper_2407_16990_b200/libregen.so.
 *
 * Citations: P:<line> = PAPER.md line, readings D1..D12 = DESIGN.md §3.
 *
 * Conventions (all calls):
 *  - Pointers prefixed d_ are DEVICE pointers (cudaMalloc / torch CUDA tensors) on the current
 *    device; h_ are host pointers. The caller owns every buffer, including the workspace d_ws
 *    (size from regen_workspace_size). The library owns only the SR handle.
 *  - Every call is stream-ordered on `stream` (a cudaStream_t passed as void*), never
 *    synchronises the host, and is capturable in a CUDA graph.
 *  - Synchronous argument errors (null pointer, bad size/mode, too small workspace) return
 *    REGEN_E_INVALID (or REGEN_E_UNSUPPORTED) before any launch; regen_last_error() gives a
 *    thread-local message. Launch failures return REGEN_E_CUDA.
 *  - Data-dependent overflow (more regions/boxes than the caller's capacity, packer free-list
 *    full) is reported asynchronously by OR-ing REGEN_ST_* bits into *d_status (int32, device);
 *    outputs are then truncated deterministically. Unplaced boxes are NOT an error: their
 *    MBs keep the bilinear value.
 *  - Determinism: identical inputs give bit-identical integer outputs (selection, labels, boxes,
 *    densities, order, placements, owners), independent of launch configuration; they equal the
 *    CPU oracle (oracle/) bit for bit.
 *  - A "call" processes one selection group: S streams x F frames of frame_w x frame_h pixels.
 */
#ifndef REGEN_H_
#define REGEN_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define REGEN_API __attribute__((visibility("default")))
#else
#define REGEN_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  REGEN_OK = 0,
  REGEN_E_INVALID = 1,
  REGEN_E_CAPACITY = 2,
  REGEN_E_CUDA = 3,
  REGEN_E_UNSUPPORTED = 4
} regen_status;

enum { REGEN_MODE_TOPK = 0, REGEN_MODE_THRESHOLD = 1 };
enum { REGEN_SCOPE_GLOBAL = 0, REGEN_SCOPE_PER_STREAM = 1, REGEN_SCOPE_PER_FRAME = 2 };
enum { REGEN_ORDER_DENSITY = 0, REGEN_ORDER_AREA = 1, REGEN_ORDER_HEIGHT = 2 };
/* placement policy of the packer (regen_pack_params.policy): GUILLOTINE = Alg. 1 with InnerFree read
 * as a guillotine split (D6, default); MAXRECT = Alg. 2 literally: one free area per bin, the maximal
 * empty rectangle of the bin's free cells (histogram-stack method), re-computed after
 * every placement (D14); SKYLINE = bottom-left skyline per bin (D15); SHELF = first-fit shelves per
 * bin (D16). The last two are the survey's comparison policies. */
enum { REGEN_POLICY_GUILLOTINE = 0, REGEN_POLICY_MAXRECT = 1, REGEN_POLICY_SKYLINE = 2, REGEN_POLICY_SHELF = 3 };
/* importance density of a box (Alg. 1 l.6): SPAN = mean over every MB of the box's MB span (P:751
 * "all MBs in it", D4, default); MEMBERS = mean over its member MBs only (P:691's set notation). */
enum { REGEN_DENSITY_SPAN = 0, REGEN_DENSITY_MEMBERS = 1 };
/* element types. REGEN_DTYPE_U8 is an output type of the frame-writing calls only (reading D20,
 * SURVEY §8(c)'s "u8 output (clamp, round-half-even)"): a bilinear pixel is the exact D10 value
 * rounded half-to-even to a code (computed in integers: 255 * bilinear(u8/255) = N / (2s)^2 exactly),
 * an enhanced pixel is rhe(255 * clamp(v, 0, 1)) of its value v in the model dtype (exact product). */
enum { REGEN_DTYPE_BF16 = 0, REGEN_DTYPE_FP32 = 1, REGEN_DTYPE_U8 = 2 };
enum { REGEN_CALL_SELECT = 0, REGEN_CALL_PACK = 1, REGEN_CALL_ENHANCE = 2, REGEN_CALL_SCATTER = 3,
       REGEN_CALL_ENHANCE_SCATTER = 4, REGEN_CALL_TEMPORAL = 5 };

/* asynchronous status bits (*d_status) */
enum {
  REGEN_ST_REGION_OVERFLOW = 1,   /* num_regions > max_regions */
  REGEN_ST_BOX_OVERFLOW = 2,      /* num_boxes > max_boxes */
  REGEN_ST_FREELIST_OVERFLOW = 4, /* packer free-area pool full: remaining boxes left unplaced */
  REGEN_ST_TOPK_INCOMPLETE = 8    /* regen_select_mbs_global before the 4 digit rounds: nothing selected */
};

/* Frame geometry. MB grid GW = ceil(frame_w/mb), GH = ceil(frame_h/mb) (D1); mb = 16.
 * format: how every call reads the LR frames d_frames: REGEN_FORMAT_RGB8 [S][F][frame_h][frame_w][3],
 * or REGEN_FORMAT_NV12, the decoder's output: per frame a Y plane [frame_h][frame_w] then the
 * interleaved U,V plane [frame_h/2][frame_w/2][2], converted to RGB8 by BT.601 (D19) inside the gather
 * and the bilinear pass (frame_w % 8 == 0, frame_h % 2 == 0). */
enum { REGEN_FORMAT_RGB8 = 0, REGEN_FORMAT_NV12 = 1 };
typedef struct {
  int32_t S, F;               /* streams, frames per stream in this call */
  int32_t frame_w, frame_h;   /* LR frame size in pixels */
  int32_t mb;                 /* macroblock size, 16 */
  int32_t format;             /* REGEN_FORMAT_RGB8 or REGEN_FORMAT_NV12 */
} regen_geom;

/* Cross-stream MB selection, §3.3.1 P:638-667 (D2). */
typedef struct {
  int32_t mode;          /* REGEN_MODE_TOPK: the k best MBs; REGEN_MODE_THRESHOLD: score >= tau */
  int32_t scope;         /* GLOBAL: one queue over the call; PER_STREAM (Uniform); PER_FRAME */
  int64_t k;             /* TOPK: count per scope segment (>= 0). THRESHOLD: cap (-1 = none) */
  float tau;             /* THRESHOLD only; must not be NaN */
  int32_t connectivity;  /* 8 (default, D3) or 4 */
  int64_t cap;           /* capacity cap N of P:663 (MB_size*N <= H*W*B: regen_capacity_mbs), applied to
                            every scope segment in both modes on top of k; -1 = none */
} regen_select_params;

/* Region-aware bin packing, Alg. 1 P:677-719 (D4-D8, D12). */
typedef struct {
  int32_t bin_w, bin_h;    /* H x W of the bins; bin_w >= 4 */
  int32_t max_bins;        /* B: bins available; boxes beyond stay bilinear */
  int32_t expand;          /* pixels of expansion around a box, 3 */
  int32_t partition_mb;    /* Partition preset size in MBs (D5): 4 for 128-px bins, 3 for 64-px */
  int32_t gutter;          /* zero gutter right/below each box (D8), 1 */
  int32_t order;           /* REGEN_ORDER_DENSITY (Alg. 1 l.6), REGEN_ORDER_AREA (max-area-first) or
                              REGEN_ORDER_HEIGHT (box height desc, for shelves); ties by box index */
  int32_t policy;          /* REGEN_POLICY_* (placement rule, default GUILLOTINE) */
  int32_t density;         /* REGEN_DENSITY_SPAN (default) or REGEN_DENSITY_MEMBERS */
} regen_pack_params;

/* SR network (D11): EDSR-baseline, or the tiny 2-conv model when n_resblocks == 0. */
typedef struct {
  int32_t scale;        /* 2, 3 or 4 */
  int32_t channels;     /* C: 8..64, multiple of 8 (tiny model: 8..64) */
  int32_t n_resblocks;  /* 0 => tiny model: conv 3->C, ReLU, conv C->3s^2, PixelShuffle(s) */
  int32_t dtype;        /* REGEN_DTYPE_BF16 (tcgen05, bf16 storage, fp32 accumulate) or REGEN_DTYPE_FP32 */
  float res_scale;      /* residual scaling, 1.0 */
  int32_t bin_w;        /* bin width the handle is planned for (BF16: every conv's tcgen05 plan and B
                           image are built by regen_sr_create for it; enhance calls with another
                           bin_w return REGEN_E_INVALID). BF16 requires channels % 16 == 0,
                           bin_w % 128 == 0 and n_resblocks > 0: there is no silent fallback to a
                           CUDA-core kernel, other BF16 configs return REGEN_E_UNSUPPORTED. FP32 runs
                           every conv on the fp32 CUDA-core kernel (the C1 model). */
} regen_sr_config;

/* Region record (Alg. 1 l.3): id order = (stream, frame, smallest raster index) (D3). 32 bytes. */
typedef struct {
  int32_t stream, frame;
  int32_t root;                 /* smallest raster index gy*GW+gx of the region in its frame */
  int32_t mx0, my0, mx1, my1;   /* MB bounding span, half-open */
  int32_t n_members;
} regen_region;

/* Box record (Alg. 1 l.4-6 + the packing plan, l.12). Index = creation order (region id, then
 * partition pieces in raster order). 80 bytes. */
typedef struct {
  int32_t stream, frame;
  int32_t mx0, my0, mx1, my1;   /* MB span after partition and re-bounding (D5), half-open */
  int32_t x0, y0, w, h;         /* LR pixel box after 3-px expansion, clamped to the frame */
  int32_t n_members;            /* member MBs (selected MBs of its region inside the span) */
  int32_t region;               /* region id */
  double density;               /* mean importance over the MB span, fp64 raster-order sum (D4) */
  int32_t bin, bx, by;          /* placement: bin index and top-left in the bin; bin = -1: unplaced */
  int32_t rotated;              /* 1: stored rotated 90 deg clockwise in the bin (D7) */
  int32_t rank;                 /* position in the packing order */
  int32_t reserved;
} regen_box;

/* ---------------------------------------------------------------------------------------------
 * a1+a2. Select MBs and grow regions. §3.3.1; Alg. 1 l.3 P:688.
 *   d_importance  [S][F][GH][GW] fp32 scores (in)
 *   d_sel_bitmap  [S][F][GH][ceil(GW/32)] u32; bit gx%32 of word gx/32 = MB selected (out)
 *   d_labels      [S][F][GH][GW] int32 region id of each selected MB, -1 otherwise (out)
 *   d_regions     [max_regions] region records (out); d_num_regions: int64 count (out, may exceed
 *                 max_regions => REGEN_ST_REGION_OVERFLOW and records truncated)
 *   d_status      reset to 0 on `stream` first (this is the first call of a batch; the later calls
 *                 of the batch OR their overflow bits into it)
 * ------------------------------------------------------------------------------------------- */
REGEN_API regen_status regen_select_mbs(const regen_geom* geom, const regen_select_params* params,
                              const float* d_importance, uint32_t* d_sel_bitmap, int32_t* d_labels,
                              regen_region* d_regions, int64_t max_regions, int64_t* d_num_regions,
                              int32_t* d_status, void* d_ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------------------
 * a3-a5. Bound + expand + partition + density, sort, pack. Alg. 1 l.4-21 P:689-717, Alg. 2.
 *   in : d_importance, d_labels, d_regions, d_num_regions (from regen_select_mbs)
 *   out: d_boxes [max_boxes] (creation order, placement filled in), d_num_boxes (int64),
 *        d_order [max_boxes] int32 box indices in packing order, d_num_bins (int32, 1 + highest
 *        bin used), d_mb_owner [S][F][GH][GW] int32: index of the placed box owning each selected
 *        MB, -1 if unselected or its box is unplaced (D9).
 * ------------------------------------------------------------------------------------------- */
REGEN_API regen_status regen_pack_regions(const regen_geom* geom, const regen_pack_params* params,
                                const float* d_importance, const int32_t* d_labels,
                                const regen_region* d_regions, const int64_t* d_num_regions,
                                regen_box* d_boxes, int64_t max_boxes, int64_t* d_num_boxes,
                                int32_t* d_order, int32_t* d_num_bins, int32_t* d_mb_owner,
                                int32_t* d_status, void* d_ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------------------
 * SR network handle. h_weights: host fp32, per conv W[Cout][Cin][3][3] then bias[Cout], in
 * network order (D11): head, 2 per resblock, body, upsampler conv(s), tail; tiny: conv0, conv1.
 * n_weights must equal the sum. Weights are repacked once (bf16 per-tap tensor-core layout for
 * BF16, planned for cfg->bin_w) and copied to the device with synchronous copies; the caller's
 * buffer may be freed afterwards. Not stream-ordered: call it before capturing or launching work.
 * After create, every enhance call is free of host synchronisation and allocation, and a handle may
 * be used from several host threads (it is read-only after create).
 * ------------------------------------------------------------------------------------------- */
REGEN_API regen_status regen_sr_create(const regen_sr_config* cfg, const float* h_weights, size_t n_weights,
                             void** out_handle);
REGEN_API regen_status regen_sr_destroy(void* handle);

/* ---------------------------------------------------------------------------------------------
 * a6. Stitch regions into bins, the first stage of regen_enhance_packed, exposed alone.
 *   d_frames  [S][F][frame_h][frame_w][3] u8 RGB (in)
 *   d_lr_bins [max_bins][bin_h][bin_w][4] (dtype: bf16 or fp32): channels 0..2 = bf16(u8/255) or
 *             fp32(u8/255) (D9) inside placed boxes (rotated per D7), 0 elsewhere; channel 3 = 0.
 * Bins >= *d_num_bins are not written. max_boxes = capacity of d_boxes (as given to
 * regen_pack_regions). Workspace: regen_workspace_size(REGEN_CALL_ENHANCE, ...) suffices.
 * ------------------------------------------------------------------------------------------- */
REGEN_API regen_status regen_stitch_bins(const regen_geom* geom, const regen_pack_params* params, int32_t dtype,
                               const uint8_t* d_frames, const regen_box* d_boxes, int64_t max_boxes,
                               const int64_t* d_num_boxes, const int32_t* d_num_bins, void* d_lr_bins,
                               void* d_ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------------------
 * a6+a7. Gather the placed boxes into packed bins and run the SR network over the packed batch.
 *   d_hr_bins [max_bins][scale*bin_h][scale*bin_w][4] (bf16 for BF16, fp32 for FP32): channels
 *             0..2 = SR output, each box equal to SR of the box alone with zero padding (D8);
 *             0 outside boxes; channel 3 = 0. Bins >= *d_num_bins are not written.
 * ------------------------------------------------------------------------------------------- */
REGEN_API regen_status regen_enhance_packed(void* sr, const regen_geom* geom, const regen_pack_params* params,
                                  const uint8_t* d_frames, const regen_box* d_boxes, int64_t max_boxes,
                                  const int64_t* d_num_boxes, const int32_t* d_num_bins, void* d_hr_bins,
                                  int32_t* d_status, void* d_ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------------------
 * a8. Scatter-and-blend (eq. P:461-464): d_out [S][F][scale*frame_h][scale*frame_w][3]
 * (out_dtype bf16, fp32 or u8 (D20)) = bilinear x scale of u8/255 (D10), overwritten on the HR
 * square of every MB with d_mb_owner >= 0 by that box's HR bin pixels (un-rotated).
 * ------------------------------------------------------------------------------------------- */
REGEN_API regen_status regen_scatter_blend(const regen_geom* geom, const regen_pack_params* params, int32_t scale,
                                 const uint8_t* d_frames, const regen_box* d_boxes,
                                 const int32_t* d_mb_owner, const void* d_hr_bins, int32_t hr_dtype,
                                 void* d_out, int32_t out_dtype, void* stream);

/* ---------------------------------------------------------------------------------------------
 * a6+a7+a8 in one call: the HR frames d_out (as regen_scatter_blend) from the packed boxes, equal
 * bit for bit to regen_enhance_packed followed by regen_scatter_blend with hr_dtype = the model
 * dtype. When the network's last upsampler + tail run folded (BF16 tensor-core path)
 * the HR bins are never formed: the fold's combine pass writes each owned selected MB's HR pixels
 * straight into d_out and the scatter pass writes the bilinear pixels only (the paper's paste-back,
 * P:771, without the HR-bin round trip). Otherwise the two calls run back to back with the HR bins
 * in the workspace. Workspace: regen_workspace_size(REGEN_CALL_ENHANCE_SCATTER, geom, &pack_params,
 * sr, &bytes). Argument errors as regen_enhance_packed / regen_scatter_blend.
 * ------------------------------------------------------------------------------------------- */
REGEN_API regen_status regen_enhance_scatter(void* sr, const regen_geom* geom, const regen_pack_params* params,
                                   const uint8_t* d_frames, const regen_box* d_boxes, int64_t max_boxes,
                                   const int64_t* d_num_boxes, const int32_t* d_num_bins,
                                   const int32_t* d_mb_owner, void* d_out, int32_t out_dtype,
                                   int32_t* d_status, void* d_ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------------------
 * The two halves of regen_enhance_scatter, for callers that schedule them on different streams
 * (the bilinear half needs only the frames and the MB owners, so it can run while the previous
 * batch's SR still occupies the tensor cores). Together they write every HR pixel of d_out exactly
 * once, bit-identical to regen_enhance_scatter (eq. P:461-464: SR(MB_s) + IN(rest)).
 *   regen_enhance_owned: a6+a7 and the paste-back of the HR square of every MB with
 *     d_mb_owner >= 0; pixels of the other MBs are not touched. Same arguments, workspace and
 *     errors as regen_enhance_scatter.
 *   regen_scatter_bilinear: a8's bilinear x scale of u8/255 (D10) on the HR square of every
 *     MB with d_mb_owner < 0; owned squares are not touched. d_frames [S][F][frame_h][frame_w][3]
 *     u8, d_mb_owner [S][F][GH][GW] int32, d_out as regen_scatter_blend. No workspace.
 *     REGEN_E_INVALID on null pointers, scale outside {2,3,4}, a bad out_dtype or geometry.
 * ------------------------------------------------------------------------------------------- */
REGEN_API regen_status regen_enhance_owned(void* sr, const regen_geom* geom, const regen_pack_params* params,
                                 const uint8_t* d_frames, const regen_box* d_boxes, int64_t max_boxes,
                                 const int64_t* d_num_boxes, const int32_t* d_num_bins,
                                 const int32_t* d_mb_owner, void* d_out, int32_t out_dtype,
                                 int32_t* d_status, void* d_ws, size_t ws_bytes, void* stream);
REGEN_API regen_status regen_scatter_bilinear(const regen_geom* geom, int32_t scale, const uint8_t* d_frames,
                                    const int32_t* d_mb_owner, void* d_out, int32_t out_dtype, void* stream);

/* ---------------------------------------------------------------------------------------------
 * exact cross-rank global top-N. The paper's queue "aggregates and sorts MBs from all
 * streams" (§3.3.1); when the streams are sharded over ranks (one process per GPU),
 * the top-N must be taken over every rank's MBs. Reading D2 with a GLOBAL MB id: key = ord(score)
 * << 32 | (0xFFFFFFFF - gid), gid = ((stream0 + s) * F + f) * GH * GW + y * GW + x (stream0 = the
 * global index of this call's first stream; ids must fit 32 bits); the N largest keys are selected,
 * i.e. every key >= the N-th largest. Protocol, identical on every rank (D17):
 *   regen_topk_init(N, state)                                  N = the job-wide k
 *   for round in 0..3:
 *     zero hist; regen_topk_histogram(geom_i, stream0_i, imp_i, state, hist) for each of the rank's
 *       calls (it ADDS the 16-bit digit `round` of the keys matching the prefix into hist[65536]);
 *     all-reduce(hist, SUM) over the ranks (the caller's collective, e.g. NCCL over NVLink);
 *     regen_topk_pick(hist, state)                             same sums -> same digit everywhere
 *   regen_select_mbs_global(geom_i, params, stream0_i, imp_i, state, ...) for each call: the bitmap
 *     of the MBs with key >= the N-th key, then regions exactly as regen_select_mbs (a2).
 * d_state: 24-byte device struct; d_hist: 65536 uint32 counts. N >= total MBs selects every MB, N =
 * 0 none. params: only `connectivity` is used. Errors as regen_select_mbs; selecting before the 4
 * rounds sets REGEN_ST_TOPK_INCOMPLETE. All calls stream-ordered, graph-capturable.
 * ------------------------------------------------------------------------------------------- */
enum { REGEN_TOPK_SEARCH = 0, REGEN_TOPK_ALL = 1, REGEN_TOPK_NONE = 2 };
typedef struct {
  uint64_t prefix;   /* digits found so far (after round 4: the N-th largest key) */
  int64_t k_rem;     /* rank of the N-th key among the keys matching the prefix */
  int32_t round;     /* digits found, 0..4 */
  int32_t flag;      /* REGEN_TOPK_SEARCH / ALL (N >= every MB) / NONE (N == 0) */
} regen_topk_state;
REGEN_API regen_status regen_topk_init(int64_t k, regen_topk_state* d_state, void* stream);
REGEN_API regen_status regen_topk_histogram(const regen_geom* geom, int64_t stream0, const float* d_importance,
                                  const regen_topk_state* d_state, uint32_t* d_hist, void* stream);
REGEN_API regen_status regen_topk_pick(const uint32_t* d_hist, regen_topk_state* d_state, void* stream);
REGEN_API regen_status regen_select_mbs_global(const regen_geom* geom, const regen_select_params* params,
                                     int64_t stream0, const float* d_importance,
                                     const regen_topk_state* d_state, uint32_t* d_sel_bitmap, int32_t* d_labels,
                                     regen_region* d_regions, int64_t max_regions, int64_t* d_num_regions,
                                     int32_t* d_status, void* d_ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------------------
 * temporal MB-importance reuse, §3.2.2 P:584-609 (the step before a1: which frames of
 * a chunk get a fresh importance prediction). One call = one chunk of F frames of S streams.
 *   d_residual_y   [S][F][frame_h][frame_w] int16: the Y-channel residual of each frame
 *   threshold      foreground = |residual| > threshold (D18)
 *   budget         frames to predict over the S streams (from the execution plan); every
 *                  stream keeps its anchor frame 0, the rest is shared by the ratio
 *                  sum_i |dPhi_ij| / sum_j sum_i |dPhi_ij| with the largest-remainder rule
 *                  (ties: lower stream), capped at F per stream (D18)
 *   d_phi          [S][F] fp64 out: Phi = sum over the 4-connected foreground components of 1/area
 *                  (the 1/Area operator), the exact sum of the correctly rounded terms
 *   d_selected     [S][F] uint8 out: 1 = predict this frame: frame 0, and for N = budget_j - 1 even
 *                  intervals of the y axis of the CDF of S = Norm(|dPhi|) (L1) the smallest
 *                  frame k >= 1 whose CDF sum_{i<k} S_i reaches the interval's midpoint (t+0.5)/N
 *                  (dPhi_i = Phi_{i+1} - Phi_i belongs to frame i+1)
 *   d_reuse        [S][F] int32 out: the selected frame whose prediction frame f reuses (the nearest
 *                  selected frame at or before f)
 *   d_frames_per_stream [S] int32 out: each stream's budget
 * Workspace: regen_workspace_size(REGEN_CALL_TEMPORAL, geom, NULL, NULL, &bytes). Frames must have
 * fewer than 2^28 pixels, S <= 1024. fp64 decisions are taken in the oracle's order (bit-exact).
 * regen_reuse_importance: d_out[s][f] = d_pred[s][d_reuse[s][f]] for the [S][F][GH][GW] fp32 maps
 * (the predictor ran on the selected frames only); d_out must not alias d_pred.
 * ------------------------------------------------------------------------------------------- */
REGEN_API regen_status regen_temporal_select(const regen_geom* geom, const int16_t* d_residual_y, int32_t threshold,
                                   int64_t budget, double* d_phi, uint8_t* d_selected, int32_t* d_reuse,
                                   int32_t* d_frames_per_stream, void* d_ws, size_t ws_bytes, void* stream);
REGEN_API regen_status regen_reuse_importance(const regen_geom* geom, const float* d_pred, const int32_t* d_reuse,
                                    float* d_out, void* stream);

/* ---------------------------------------------------------------------------------------------
 * NV12 input (the hardware decoder's output format; decode stage P:424 §3.1).
 *   d_nv12  [S][F] frames of frame_w*frame_h*3/2 bytes: Y plane [frame_h][frame_w] then the
 *           interleaved U,V plane [frame_h/2][frame_w/2][2]
 *   d_rgb8  [S][F][frame_h][frame_w][3] out, the d_frames of every other call
 * BT.601 limited range, 8-bit integer form, nearest chroma (D19, bit-exact vs the oracle).
 * REGEN_E_INVALID unless frame_w % 4 == 0, frame_h % 2 == 0 and both buffers are 4-byte aligned.
 * ------------------------------------------------------------------------------------------- */
REGEN_API regen_status regen_nv12_to_rgb8(const regen_geom* geom, const uint8_t* d_nv12, uint8_t* d_rgb8, void* stream);

/* ---------------------------------------------------------------------------------------------
 * regen_enhance_owned split into two stream-ordered halves, for schedules that run the partial-sum
 * combine of batch k on another stream beside batch k+1's convolutions (BF16 tensor-core path with the
 * UP∘TAIL fold; REGEN_E_UNSUPPORTED otherwise):
 *   regen_enhance_partials: a6 + a7 up to the fold conv; its partial sums stay in d_ws.
 *   regen_fold_combine_frames: the combine of those partials into the owned MBs' HR pixels of d_out.
 * Both take the same d_ws (sized by regen_workspace_size(REGEN_CALL_ENHANCE, ...)); the pair is
 * bit-identical to regen_enhance_owned. The combine must complete before the next partials call on
 * the same workspace.
 * ------------------------------------------------------------------------------------------- */
REGEN_API regen_status regen_enhance_partials(void* sr, const regen_geom* geom, const regen_pack_params* params,
                                    const uint8_t* d_frames, const regen_box* d_boxes, int64_t max_boxes,
                                    const int64_t* d_num_boxes, const int32_t* d_num_bins,
                                    const int32_t* d_mb_owner, int32_t* d_status, void* d_ws, size_t ws_bytes,
                                    void* stream);
REGEN_API regen_status regen_fold_combine_frames(void* sr, const regen_geom* geom, const regen_pack_params* params,
                                       const regen_box* d_boxes, const int32_t* d_num_bins,
                                       const int32_t* d_mb_owner, void* d_out, int32_t out_dtype, void* d_ws,
                                       size_t ws_bytes, void* stream);

/* Workspace bytes for a call (which = REGEN_CALL_*; params = the call's params struct — for PACK,
 * NULL sizes the default guillotine packer, the pack params add a placement policy's per-bin state;
 * sr = SR handle for ENHANCE, else NULL). */
REGEN_API regen_status regen_workspace_size(int32_t which, const regen_geom* geom, const void* params, const void* sr,
                                  size_t* bytes);

/* Number of kernels one regen_enhance_packed call launches for this SR handle and bin geometry
 * (clear + paint + gather + one per conv launch + the fold combine; memsets excluded). Host-only, no device
 * work; lets benchmarks count launches without a profiler. Returns REGEN_E_INVALID on null args. */
REGEN_API regen_status regen_enhance_kernel_count(const void* sr, const regen_pack_params* params, int32_t* count);

/* Launch tracing (measurement aid). When enabled, every kernel libregen launches is bracketed by
 * two CUDA events recorded on its stream. regen_trace_read waits for the recorded launches and
 * returns, in launch order, up to `cap` names (REGEN_TRACE_NAME_LEN bytes each, NUL-terminated)
 * and device durations in ms; *n = number of launches recorded (may exceed cap); the record is then
 * cleared. Host-thread-safe; adds two event records per launch while on. */
#define REGEN_TRACE_NAME_LEN 32
REGEN_API regen_status regen_trace_enable(int32_t on);
/* Trace only kernels whose name starts with `prefix` (NULL or "" = all). */
REGEN_API regen_status regen_trace_filter(const char* prefix);
REGEN_API regen_status regen_trace_read(char* names, float* ms, int32_t cap, int32_t* n);

/* Helpers. */
REGEN_API int64_t regen_capacity_mbs(int32_t bin_w, int32_t bin_h, int32_t n_bins, int32_t mb);  /* floor(H*W*B/mb^2) */
REGEN_API const char* regen_status_string(regen_status s);
REGEN_API const char* regen_last_error(void);
REGEN_API int32_t regen_abi_version(void);   /* 2 */

#ifdef __cplusplus
}
#endif
#endif /* REGEN_H_ */
