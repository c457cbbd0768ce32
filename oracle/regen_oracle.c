/*
 * regen_oracle.c — CPU ORACLE for the RegenHance region-aware enhancement hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library. The product path (paper_2407_16990_b200/) never
 * links, imports or calls it, and shares no header, helper, table or constant generator with it.
 *
 * Plain, slow, written from the paper (arXiv 2407.16990, /root/reference/PAPER.md,
 * cited as P:<line>) in the paper's order. Floating point is fp64 except where a stated reading
 * fixes a lower precision (input quantisation to bf16, bf16-rounded conv weights).
 * Readings of the paper's gaps are D1..D12 in DESIGN.md §3; each function names the ones it uses.
 *
 * Parity status: every function below is pinned by tests/test_oracle_*.py (not-gpu). The SR pixels
 * of a random-init EDSR have no paper-printed values; the conv/pixel-shuffle/bilinear steps are
 * pinned to torch fp64 library routines and closed forms, the end-to-end SR is pinned only through
 * those steps plus the isolation invariant ("parity pinned via steps").
 *
 * Every step is a single-threaded function; ref_enhance_mt / ref_scatter_mt only distribute the same
 * per-box / per-frame functions over POSIX threads (bit-identical results, for the all-box parity
 * checks and the all-cores CPU baseline).
 *
 * Build: gcc -O2 -std=c11 -fPIC -shared -pthread -ffp-contract=off -o liboracle.so regen_oracle.c
 * (no -ffast-math: fp64 sums in the stated order; no FMA contraction).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <pthread.h>

/* ------------------------------------------------------------------------------------------ */
/* Geometry. P:454 "frames are divided into an array of 16x16-pixel MBs"; P:535 1920x1080 ->   */
/* 120x68 labels, i.e. partial MBs at the bottom/right are real grid cells (reading D1: ceil). */
/* ------------------------------------------------------------------------------------------ */
static int grid_w(int W, int mb) { return (W + mb - 1) / mb; }
static int grid_h(int H, int mb) { return (H + mb - 1) / mb; }

/* ------------------------------------------------------------------------------------------ */
/* O2. Cross-stream MB selection, P:638-667 (§3.3.1).                                          */
/* "constructs a global queue that aggregates and sorts MBs from all streams in order of the    */
/* importance" and "selects the top N MBs". Reading D2: the queue order is      */
/* importance descending, ties by linear MB id ascending, id = ((s*F+f)*GH+y)*GW+x; the         */
/* importance order is IEEE order with -0 == +0 and NaN lowest. cap >= 0: the capacity N of     */
/* P:663 ("max N: MB_size * N <= H * W * B") bounds every scope segment's selection as well.    */
/* mode 0 = TOPK (k largest), mode 1 = THRESHOLD (score >= tau, P:1352 baseline; if k >= 0 the  */
/* result is capped to its k first queue entries). scope 0 = GLOBAL (the whole call),    */
/* 1 = PER_STREAM (Uniform baseline P:1352: k per stream), 2 = PER_FRAME (k per frame).         */
/* ------------------------------------------------------------------------------------------ */
typedef struct { uint32_t ord; uint32_t id; } sel_item;

static uint32_t score_order(float s) {
  uint32_t b;
  if (s != s) return 0u;            /* NaN: lowest */
  if (s == 0.0f) s = 0.0f;          /* -0 == +0 */
  memcpy(&b, &s, 4);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

static int cmp_queue(const void* a, const void* b) {
  const sel_item* x = (const sel_item*)a;
  const sel_item* y = (const sel_item*)b;
  if (x->ord != y->ord) return x->ord > y->ord ? -1 : 1;   /* importance descending */
  if (x->id != y->id) return x->id < y->id ? -1 : 1;       /* id ascending */
  return 0;
}

int ref_select(int S, int F, int W, int H, int mb, int mode, int64_t k, float tau, int scope, int64_t cap,
               const float* score, uint8_t* sel) {
  const int GW = grid_w(W, mb), GH = grid_h(H, mb);
  const int64_t per_frame = (int64_t)GH * GW;
  const int64_t M = (int64_t)S * F * per_frame;
  int64_t seg_len = scope == 0 ? M : scope == 1 ? (int64_t)F * per_frame : per_frame;
  if (M == 0) return 0;
  sel_item* q = (sel_item*)malloc(sizeof(sel_item) * (size_t)seg_len);
  if (!q) return -1;
  memset(sel, 0, (size_t)M);
  for (int64_t seg0 = 0; seg0 < M; seg0 += seg_len) {
    int64_t n = 0;
    for (int64_t id = seg0; id < seg0 + seg_len; ++id) {
      if (mode == 1 && !(score[id] >= tau)) continue;          /* threshold filter */
      q[n].ord = score_order(score[id]);
      q[n].id = (uint32_t)id;
      ++n;
    }
    qsort(q, (size_t)n, sizeof(sel_item), cmp_queue);          /* the global queue */
    int64_t take = n;
    if (mode == 0 || k >= 0) take = k < n ? k : n;            /* top-N / threshold cap */
    if (cap >= 0 && take > cap) take = cap;                   /* capacity N */
    if (take < 0) take = 0;
    for (int64_t i = 0; i < take; ++i) sel[q[i].id] = 1;
  }
  free(q);
  return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* O3. RegionProps, Alg. 1 line 3, "constructs regions by calculating the        */
/* connected components of selected MB". Reading D3: 8-connectivity (4 optional). Regions are   */
/* numbered in (stream, frame, smallest raster index) order: a raster scan of each frame starts */
/* a breadth-first flood fill at every not-yet-labelled selected MB.                           */
/* region record (int32 x8): stream, frame, root(raster idx), mx0, my0, mx1, my1 (half-open),   */
/* n_members. labels: region id per MB, -1 if unselected.                                      */
/* ------------------------------------------------------------------------------------------ */
int ref_regions(int S, int F, int W, int H, int mb, int conn, const uint8_t* sel,
                int32_t* labels, int32_t* regions, int64_t max_regions, int64_t* num_regions) {
  const int GW = grid_w(W, mb), GH = grid_h(H, mb);
  const int per_frame = GH * GW;
  static const int dx8[8] = {-1, 0, 1, -1, 1, -1, 0, 1};
  static const int dy8[8] = {-1, -1, -1, 0, 0, 1, 1, 1};
  static const int dx4[4] = {0, -1, 1, 0};
  static const int dy4[4] = {-1, 0, 0, 1};
  const int nn = conn == 4 ? 4 : 8;
  const int* dx = conn == 4 ? dx4 : dx8;
  const int* dy = conn == 4 ? dy4 : dy8;
  int* queue = (int*)malloc(sizeof(int) * (size_t)(per_frame > 0 ? per_frame : 1));
  int64_t nreg = 0;
  int overflow = 0;
  for (int64_t i = 0; i < (int64_t)S * F * per_frame; ++i) labels[i] = -1;
  for (int s = 0; s < S; ++s)
    for (int f = 0; f < F; ++f) {
      const int64_t base = ((int64_t)s * F + f) * per_frame;
      for (int start = 0; start < per_frame; ++start) {
        if (!sel[base + start] || labels[base + start] >= 0) continue;
        const int64_t r = nreg++;
        int head = 0, tail = 0;
        int mx0 = GW, my0 = GH, mx1 = 0, my1 = 0, cnt = 0;
        labels[base + start] = (int32_t)r;
        queue[tail++] = start;
        while (head < tail) {
          const int c = queue[head++];
          const int cx = c % GW, cy = c / GW;
          ++cnt;
          if (cx < mx0) mx0 = cx;
          if (cy < my0) my0 = cy;
          if (cx + 1 > mx1) mx1 = cx + 1;
          if (cy + 1 > my1) my1 = cy + 1;
          for (int d = 0; d < nn; ++d) {
            const int nx = cx + dx[d], ny = cy + dy[d];
            if (nx < 0 || ny < 0 || nx >= GW || ny >= GH) continue;
            const int nc = ny * GW + nx;
            if (sel[base + nc] && labels[base + nc] < 0) {
              labels[base + nc] = (int32_t)r;
              queue[tail++] = nc;
            }
          }
        }
        if (r < max_regions) {
          int32_t* rec = regions + 8 * r;
          rec[0] = s; rec[1] = f; rec[2] = start;
          rec[3] = mx0; rec[4] = my0; rec[5] = mx1; rec[6] = my1; rec[7] = cnt;
        } else {
          overflow = 1;
        }
      }
    }
  free(queue);
  *num_regions = nreg;
  return overflow ? 2 : 0;
}

/* ------------------------------------------------------------------------------------------ */
/* O4. Bound + Partition + density, Alg. 1 lines 4-6, footnote P:735    */
/* (3-pixel expansion). Readings: D4 density = mean importance of ALL MBs in the box's  */
/* MB span ("average importance of all MBs in it"), fp64, raster order (density_mode 1:  */
/* the mean over the box's member MBs only, P:691's set notation); D5 partition:                */
/* a region whose MB span is wider/taller than P MBs is cut into ceil(n/P) near-equal           */
/* MB-aligned pieces per axis (the first n mod pieces get one extra MB), pieces are visited in  */
/* raster order, each piece keeps only the region's member MBs and is re-bounded to them; empty */
/* pieces are dropped. Pixel box = [16*mx0-e, min(W,16*mx1+e)) x [...] clamped at 0.            */
/* box record (int32 x12): stream, frame, mx0, my0, mx1, my1, x0, y0, w, h, n_members, region.  */
/* box_of_mb: index of the box owning each member MB (every selected MB has exactly one).       */
/* ------------------------------------------------------------------------------------------ */
static int piece_start(int n, int pieces, int i) {
  /* start offset of piece i when n cells are cut into `pieces` near-equal parts, first ones larger */
  const int base = n / pieces, rem = n % pieces;
  return i * base + (i < rem ? i : rem);
}

int ref_boxes(int S, int F, int W, int H, int mb, int expand, int partition_mb, int density_mode,
              const float* score, const int32_t* labels, const int32_t* regions, int64_t num_regions,
              int32_t* boxes, double* density, int64_t max_boxes, int64_t* num_boxes, int32_t* box_of_mb) {
  const int GW = grid_w(W, mb), GH = grid_h(H, mb);
  const int per_frame = GH * GW;
  int64_t nb = 0;
  int overflow = 0;
  for (int64_t i = 0; i < (int64_t)S * F * per_frame; ++i) box_of_mb[i] = -1;
  for (int64_t r = 0; r < num_regions; ++r) {
    const int32_t* rec = regions + 8 * r;
    const int s = rec[0], f = rec[1];
    const int64_t base = ((int64_t)s * F + f) * per_frame;
    const int rx0 = rec[3], ry0 = rec[4], rx1 = rec[5], ry1 = rec[6];
    const int wm = rx1 - rx0, hm = ry1 - ry0;
    const int nx = (wm + partition_mb - 1) / partition_mb;   /* Partition (line 5) */
    const int ny = (hm + partition_mb - 1) / partition_mb;
    for (int py = 0; py < ny; ++py)
      for (int px = 0; px < nx; ++px) {
        const int sx0 = rx0 + piece_start(wm, nx, px), sx1 = rx0 + piece_start(wm, nx, px + 1);
        const int sy0 = ry0 + piece_start(hm, ny, py), sy1 = ry0 + piece_start(hm, ny, py + 1);
        int mx0 = GW, my0 = GH, mx1 = 0, my1 = 0, cnt = 0;
        for (int y = sy0; y < sy1; ++y)
          for (int x = sx0; x < sx1; ++x)
            if (labels[base + y * GW + x] == (int32_t)r) {
              ++cnt;
              if (x < mx0) mx0 = x;
              if (y < my0) my0 = y;
              if (x + 1 > mx1) mx1 = x + 1;
              if (y + 1 > my1) my1 = y + 1;
            }
        if (cnt == 0) continue;                                  /* empty piece dropped */
        const int64_t b = nb++;
        if (b >= max_boxes) { overflow = 1; continue; }
        /* Bound (line 4) with the 3-pixel expansion, clamped to the frame */
        int x0 = mb * mx0 - expand, y0 = mb * my0 - expand;
        int x1 = mb * mx1 + expand, y1 = mb * my1 + expand;
        if (x0 < 0) x0 = 0;
        if (y0 < 0) y0 = 0;
        if (x1 > W) x1 = W;
        if (y1 > H) y1 = H;
        /* importance density (line 6 order key) over the full MB span, raster order */
        double sum = 0.0;
        for (int y = my0; y < my1; ++y)
          for (int x = mx0; x < mx1; ++x)
            if (density_mode == 0 || labels[base + y * GW + x] == (int32_t)r) sum += (double)score[base + y * GW + x];
        density[b] = sum / (double)(density_mode == 0 ? (mx1 - mx0) * (my1 - my0) : cnt);
        int32_t* bx = boxes + 12 * b;
        bx[0] = s; bx[1] = f; bx[2] = mx0; bx[3] = my0; bx[4] = mx1; bx[5] = my1;
        bx[6] = x0; bx[7] = y0; bx[8] = x1 - x0; bx[9] = y1 - y0; bx[10] = cnt; bx[11] = (int32_t)r;
        for (int y = my0; y < my1; ++y)
          for (int x = mx0; x < mx1; ++x)
            if (labels[base + y * GW + x] == (int32_t)r) box_of_mb[base + y * GW + x] = (int32_t)b;
      }
  }
  *num_boxes = nb;
  return overflow ? 2 : 0;
}

/* ------------------------------------------------------------------------------------------ */
/* O5a. Sort, Alg. 1 line 6: boxes in descending importance density; ties   */
/* by creation index (reading D2 applied to boxes). order 1 = max-area-first baseline (P:753,   */
/* `fig:Puzzle`): area w*h descending, ties by index; order 2 = box height h descending (shelf  */
/* packing's usual order), ties by index. NaN densities sort last.                              */
/* ------------------------------------------------------------------------------------------ */
static const double* g_sort_density;
static const int32_t* g_sort_boxes;
static int g_sort_policy;

static int cmp_boxes(const void* a, const void* b) {
  const int32_t i = *(const int32_t*)a, j = *(const int32_t*)b;
  if (g_sort_policy == 1) {
    const int64_t ai = (int64_t)g_sort_boxes[12 * i + 8] * g_sort_boxes[12 * i + 9];
    const int64_t aj = (int64_t)g_sort_boxes[12 * j + 8] * g_sort_boxes[12 * j + 9];
    if (ai != aj) return ai > aj ? -1 : 1;
  } else if (g_sort_policy == 2) {
    const int32_t hi = g_sort_boxes[12 * i + 9], hj = g_sort_boxes[12 * j + 9];
    if (hi != hj) return hi > hj ? -1 : 1;
  } else {
    const double di = g_sort_density[i], dj = g_sort_density[j];
    const int ni = di != di, nj = dj != dj;
    if (ni != nj) return ni ? 1 : -1;
    if (!ni && di != dj) return di > dj ? -1 : 1;
  }
  return i < j ? -1 : (i > j ? 1 : 0);
}

int ref_sort(int64_t num_boxes, const int32_t* boxes, const double* density, int policy, int32_t* order) {
  for (int64_t i = 0; i < num_boxes; ++i) order[i] = (int32_t)i;
  g_sort_density = density;
  g_sort_boxes = boxes;
  g_sort_policy = policy;
  qsort(order, (size_t)num_boxes, sizeof(int32_t), cmp_boxes);
  return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* O5b. Packing, Alg. 1 lines 7-13 + RotatePacking + Update/InnerFree (P:711-717,  */
/* Alg. 2). Readings: D6 InnerFree = guillotine split of the used free area into    */
/* <= 2 remainders (vertical: right full-height + bottom; horizontal: bottom full-width +       */
/* right), choosing the option whose larger remainder is larger, ties vertical; non-empty       */
/* remainders are appended in that listed order. D12 free-area order: `for farea in freeareas`  */
/* scans free areas in (bin index, creation sequence) order; the box goes to the first one that */
/* admits it unrotated or rotated (RotatePacking), unrotated preferred (P:706 before P:707,     */
/* D7: rotated = 90 deg clockwise), anchored at the area's top-left. D8 bin layout: a box of     */
/* w x h needs a footprint (w+g) x (h+g) (g = 1 zero gutter right/below); bin column 0 is a     */
/* reserved zero column, so every bin starts as one free area (x=1, y=0, W-1, H+g).             */
/* placement record (int32 x4): bin, bx, by, rotated; bin = -1 if the box fits nowhere (its MBs */
/* stay bilinear, "not an error").                                                        */
/* ------------------------------------------------------------------------------------------ */
typedef struct { int bin, seq, x, y, w, h; } free_area;

/* InnerFree (Alg. 2, reading D6): free area fw x fh with a uw x uh footprint at its top-left.
 * Returns the number (0..2) of non-empty remainders written as (dx, dy, w, h) relative to the
 * free area's origin, in listed order. vertical = {right full-height, bottom}, horizontal =
 * {bottom full-width, right}; the option whose larger remainder has the larger area wins, ties
 * vertical. */
int ref_inner_free(int fw, int fh, int uw, int uh, int32_t* out) {
  const int64_t v_a = (int64_t)(fw - uw) * fh, v_b = (int64_t)uw * (fh - uh);
  const int64_t h_a = (int64_t)fw * (fh - uh), h_b = (int64_t)(fw - uw) * uh;
  const int64_t vmax = v_a > v_b ? v_a : v_b, hmax = h_a > h_b ? h_a : h_b;
  int32_t cand[8];
  if (vmax >= hmax) {
    cand[0] = uw; cand[1] = 0;  cand[2] = fw - uw; cand[3] = fh;        /* right, full height */
    cand[4] = 0;  cand[5] = uh; cand[6] = uw;      cand[7] = fh - uh;   /* bottom */
  } else {
    cand[0] = 0;  cand[1] = uh; cand[2] = fw;      cand[3] = fh - uh;   /* bottom, full width */
    cand[4] = uw; cand[5] = 0;  cand[6] = fw - uw; cand[7] = uh;        /* right */
  }
  int n = 0;
  for (int t = 0; t < 2; ++t)
    if (cand[4 * t + 2] > 0 && cand[4 * t + 3] > 0) {
      for (int i = 0; i < 4; ++i) out[4 * n + i] = cand[4 * t + i];
      ++n;
    }
  return n;
}

int ref_pack(int64_t num_boxes, const int32_t* boxes, const int32_t* order, int bin_w, int bin_h,
             int max_bins, int gutter, int32_t* placement, int32_t* num_bins) {
  int64_t cap = (int64_t)max_bins + 2 * num_boxes + 4;
  free_area* fa = (free_area*)malloc(sizeof(free_area) * (size_t)cap);
  if (!fa) return -1;
  int64_t nfa = 0;
  int next_seq = 0;
  int used = 0;
  for (int b = 0; b < max_bins; ++b) {                        /* freeareas = Bins (line 1) */
    fa[nfa].bin = b; fa[nfa].seq = next_seq++;
    fa[nfa].x = 1; fa[nfa].y = 0; fa[nfa].w = bin_w - 1; fa[nfa].h = bin_h + gutter;
    ++nfa;
  }
  for (int64_t i = 0; i < num_boxes; ++i) placement[4 * i] = -1, placement[4 * i + 1] = 0,
                                          placement[4 * i + 2] = 0, placement[4 * i + 3] = 0;
  for (int64_t oi = 0; oi < num_boxes; ++oi) {                 /* for box in boxes (line 7) */
    const int32_t b = order[oi];
    const int pw = boxes[12 * b + 8] + gutter, ph = boxes[12 * b + 9] + gutter;
    int64_t best = -1;
    for (int64_t j = 0; j < nfa; ++j) {                        /* for farea in freeareas (line 8) */
      const int fits = (fa[j].w >= pw && fa[j].h >= ph) || (fa[j].w >= ph && fa[j].h >= pw);
      if (!fits) continue;
      if (best < 0 || fa[j].bin < fa[best].bin || (fa[j].bin == fa[best].bin && fa[j].seq < fa[best].seq))
        best = j;
    }
    if (best < 0) continue;                                    /* unplaced */
    const free_area r = fa[best];
    const int rot = !(r.w >= pw && r.h >= ph);
    const int uw = rot ? ph : pw, uh = rot ? pw : ph;
    placement[4 * b] = r.bin; placement[4 * b + 1] = r.x; placement[4 * b + 2] = r.y; placement[4 * b + 3] = rot;
    if (r.bin + 1 > used) used = r.bin + 1;
    fa[best] = fa[--nfa];                                      /* freeareas \ {farea} */
    /* InnerFree (guillotine, D6) */
    int32_t rem[8];
    const int nrem = ref_inner_free(r.w, r.h, uw, uh, rem);
    for (int t = 0; t < nrem; ++t) {
      fa[nfa].bin = r.bin; fa[nfa].seq = next_seq++;
      fa[nfa].x = r.x + rem[4 * t]; fa[nfa].y = r.y + rem[4 * t + 1];
      fa[nfa].w = rem[4 * t + 2]; fa[nfa].h = rem[4 * t + 3];
      ++nfa;
    }
  }
  free(fa);
  *num_bins = used;
  return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* O6. Stitch regions into bins, "we stitch the real-content regions into tensors (bins)  */
/* following the packing plan". Bin-local pixel (p,q) of a placed box: unrotated source          */
/* (x0+p, y0+q); rotated 90 deg CW (bin footprint h x w): source (x0+q, y0+h-1-p). Value: D9     */
/* input quantisation v = u8/255 computed in fp32, then rounded to bf16 when bf16 != 0. All other */
/* bin pixels are 0. lr: [num_bins][bin_h][bin_w][3] fp64.                                       */
/* ------------------------------------------------------------------------------------------ */
static float round_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  u &= 0xFFFF0000u;
  memcpy(&f, &u, 4);
  return f;
}

double ref_input_value(uint8_t u, int bf16) {
  float v = (float)u / 255.0f;
  return (double)(bf16 ? round_bf16(v) : v);
}

int ref_gather(int S, int F, int W, int H, const uint8_t* frames, int64_t num_boxes, const int32_t* boxes,
               const int32_t* placement, int bin_w, int bin_h, int num_bins, int bf16, double* lr) {
  (void)S;
  memset(lr, 0, sizeof(double) * (size_t)num_bins * bin_h * bin_w * 3);
  for (int64_t b = 0; b < num_boxes; ++b) {
    const int32_t* bx = boxes + 12 * b;
    const int32_t* pl = placement + 4 * b;
    if (pl[0] < 0) continue;
    const int s = bx[0], f = bx[1], x0 = bx[6], y0 = bx[7], w = bx[8], h = bx[9];
    const int rot = pl[3];
    const int fw = rot ? h : w, fh = rot ? w : h;
    for (int q = 0; q < fh; ++q)
      for (int p = 0; p < fw; ++p) {
        const int sx = rot ? x0 + q : x0 + p;
        const int sy = rot ? y0 + h - 1 - p : y0 + q;
        const uint8_t* src = frames + ((((int64_t)s * F + f) * H + sy) * W + sx) * 3;
        double* dst = lr + (((int64_t)pl[0] * bin_h + pl[2] + q) * bin_w + pl[1] + p) * 3;
        for (int c = 0; c < 3; ++c) dst[c] = ref_input_value(src[c], bf16);
      }
  }
  return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* O7. Super-resolution of one stitched box, "pre-trained EDSR", §3.3.3. Reading D10: the */
/* network runs on each placed box ALONE (its rotated crop) with zero padding at every layer,   */
/* which is what the packed batch computes under the seam-isolation reading D8. Direct loops in */
/* fp64. Network (EDSR baseline structure, reading D11): head conv 3->C; n x [conv C->C, ReLU,  */
/* conv C->C, x res_scale, + skip]; body conv C->C + global skip; upsampler conv C->C*s^2 +      */
/* PixelShuffle(s) (s=4: two x2 stages); tail conv C->3 at HR. Tiny model (n_resblocks == 0):   */
/* conv 3->C, ReLU, conv C->3*s^2, PixelShuffle(s). All convs 3x3, pad 1, bias.                  */
/* weights: per conv [Cout][Cin][3][3] then bias[Cout], network order (as given; the caller      */
/* rounds them to bf16 for the bf16 path).                                                       */
/* ------------------------------------------------------------------------------------------ */
static void conv3x3(const double* in, int Cin, int Hh, int Ww, const double* w, const double* bias, int Cout,
                    double* out) {
  for (int co = 0; co < Cout; ++co)
    for (int y = 0; y < Hh; ++y)
      for (int x = 0; x < Ww; ++x) {
        double acc = bias[co];
        for (int ci = 0; ci < Cin; ++ci)
          for (int ky = 0; ky < 3; ++ky)
            for (int kx = 0; kx < 3; ++kx) {
              const int iy = y + ky - 1, ix = x + kx - 1;
              if (iy < 0 || ix < 0 || iy >= Hh || ix >= Ww) continue;   /* zero padding */
              acc += w[((co * Cin + ci) * 3 + ky) * 3 + kx] * in[((int64_t)ci * Hh + iy) * Ww + ix];
            }
        out[((int64_t)co * Hh + y) * Ww + x] = acc;
      }
}

/* PixelShuffle: out[c][y*s+i][x*s+j] = in[c*s*s + i*s + j][y][x] */
static void pixel_shuffle(const double* in, int Cin, int Hh, int Ww, int s, double* out) {
  const int C = Cin / (s * s);
  for (int c = 0; c < C; ++c)
    for (int i = 0; i < s; ++i)
      for (int j = 0; j < s; ++j)
        for (int y = 0; y < Hh; ++y)
          for (int x = 0; x < Ww; ++x)
            out[((int64_t)c * Hh * s + y * s + i) * (Ww * s) + x * s + j] =
                in[((int64_t)(c * s * s + i * s + j) * Hh + y) * Ww + x];
}

void ref_conv3x3(const double* in, int Cin, int Hh, int Ww, const double* w, const double* bias, int Cout,
                 double* out) {
  conv3x3(in, Cin, Hh, Ww, w, bias, Cout, out);
}

void ref_pixel_shuffle(const double* in, int Cin, int Hh, int Ww, int s, double* out) {
  pixel_shuffle(in, Cin, Hh, Ww, s, out);
}

/* in: [3][Hh][Ww] planar; out: [3][s*Hh][s*Ww] planar */
int ref_sr_crop(int scale, int C, int n_resblocks, double res_scale, const double* weights,
                const double* in, int Hh, int Ww, double* out) {
  const int64_t P = (int64_t)Hh * Ww;
  const int64_t big = P * scale * scale * (C > 3 ? C : 3);   /* largest intermediate */
  double* a = (double*)calloc((size_t)big, sizeof(double));
  double* b = (double*)calloc((size_t)big, sizeof(double));
  double* t = (double*)calloc((size_t)big, sizeof(double));
  double* h = (double*)calloc((size_t)C * P, sizeof(double));
  if (!a || !b || !t || !h) { free(a); free(b); free(t); free(h); return -1; }
  const double* wp = weights;
#define NEXT_CONV(cin, cout, src, dst, hh, ww)                                   \
  do {                                                                         \
    conv3x3((src), (cin), (hh), (ww), wp, wp + (int64_t)(cout) * (cin) * 9, (cout), (dst)); \
    wp += (int64_t)(cout) * (cin) * 9 + (cout);                                \
  } while (0)
  if (n_resblocks == 0) {
    const int s2 = scale * scale;
    NEXT_CONV(3, C, in, a, Hh, Ww);
    for (int64_t i = 0; i < (int64_t)C * P; ++i) a[i] = a[i] > 0.0 ? a[i] : 0.0;   /* ReLU */
    NEXT_CONV(C, 3 * s2, a, b, Hh, Ww);
    pixel_shuffle(b, 3 * s2, Hh, Ww, scale, out);
  } else {
    NEXT_CONV(3, C, in, h, Hh, Ww);                                  /* head */
    memcpy(a, h, sizeof(double) * (size_t)(C * P));                  /* residual stream */
    for (int r = 0; r < n_resblocks; ++r) {
      NEXT_CONV(C, C, a, t, Hh, Ww);
      for (int64_t i = 0; i < (int64_t)C * P; ++i) t[i] = t[i] > 0.0 ? t[i] : 0.0;
      NEXT_CONV(C, C, t, b, Hh, Ww);
      for (int64_t i = 0; i < (int64_t)C * P; ++i) a[i] = a[i] + res_scale * b[i];
    }
    NEXT_CONV(C, C, a, b, Hh, Ww);                                   /* body conv */
    for (int64_t i = 0; i < (int64_t)C * P; ++i) b[i] += h[i];       /* global skip */
    int hh = Hh, ww = Ww;
    const int stages = scale == 4 ? 2 : 1;
    const int ss = scale == 4 ? 2 : scale;
    for (int st = 0; st < stages; ++st) {                            /* upsampler */
      NEXT_CONV(C, C * ss * ss, b, t, hh, ww);
      pixel_shuffle(t, C * ss * ss, hh, ww, ss, b);
      hh *= ss; ww *= ss;
    }
    NEXT_CONV(C, 3, b, out, hh, ww);                                 /* tail at HR */
  }
#undef NEXT_CONV
  free(a); free(b); free(t); free(h);
  return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* O7b. Enhance every placed box into the HR bins: hr[num_bins][s*bin_h][s*bin_w][3] fp64 gets   */
/* SR(crop) at (s*bx, s*by) for each placed box (crop = its rotated footprint, read back from    */
/* lr), zeros elsewhere. Boxes with index in [box_lo, box_hi) only (sampling for large sizes).   */
/* ------------------------------------------------------------------------------------------ */
static int enhance_box(int scale, int C, int n_resblocks, double res_scale, const double* weights,
                       const double* lr, int bin_w, int bin_h, const int32_t* bx, const int32_t* pl, double* hr) {
  const int HW = scale * bin_w, HH = scale * bin_h;
  const int rot = pl[3];
  const int fw = rot ? bx[9] : bx[8], fh = rot ? bx[8] : bx[9];
  double* in = (double*)malloc(sizeof(double) * 3 * (size_t)fw * fh);
  double* out = (double*)malloc(sizeof(double) * 3 * (size_t)fw * fh * scale * scale);
  if (!in || !out) { free(in); free(out); return -1; }
  for (int c = 0; c < 3; ++c)
    for (int q = 0; q < fh; ++q)
      for (int p = 0; p < fw; ++p)
        in[((int64_t)c * fh + q) * fw + p] = lr[(((int64_t)pl[0] * bin_h + pl[2] + q) * bin_w + pl[1] + p) * 3 + c];
  const int rc = ref_sr_crop(scale, C, n_resblocks, res_scale, weights, in, fh, fw, out);
  for (int c = 0; c < 3; ++c)
    for (int q = 0; q < fh * scale; ++q)
      for (int p = 0; p < fw * scale; ++p)
        hr[(((int64_t)pl[0] * HH + scale * pl[2] + q) * HW + scale * pl[1] + p) * 3 + c] =
            out[((int64_t)c * fh * scale + q) * fw * scale + p];
  free(in);
  free(out);
  return rc;
}

int ref_enhance(int scale, int C, int n_resblocks, double res_scale, const double* weights,
                const double* lr, int bin_w, int bin_h, int num_bins, int64_t num_boxes, const int32_t* boxes,
                const int32_t* placement, int64_t box_lo, int64_t box_hi, double* hr) {
  const int HW = scale * bin_w, HH = scale * bin_h;
  memset(hr, 0, sizeof(double) * (size_t)num_bins * HH * HW * 3);
  for (int64_t b = box_lo; b < box_hi && b < num_boxes; ++b) {
    if (placement[4 * b] < 0) continue;
    if (enhance_box(scale, C, n_resblocks, res_scale, weights, lr, bin_w, bin_h, boxes + 12 * b, placement + 4 * b,
                    hr) != 0)
      return -1;
  }
  return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* Multi-threaded entries (for the all-box parity checks and the all-cores CPU baseline): the   */
/* same per-box / per-frame functions as the single-threaded ones, distributed round-robin over */
/* POSIX threads. Boxes occupy disjoint HR-bin footprints and frames disjoint outputs, so the   */
/* results are bit-identical to ref_enhance / ref_scatter.                                       */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
  int scale, C, n_resblocks, bin_w, bin_h;
  double res_scale;
  const double *weights, *lr;
  const int32_t *boxes, *placement;
  int64_t lo, hi, stride, first;
  double* hr;
  int rc;
} enhance_job;

static void* enhance_worker(void* arg) {
  enhance_job* j = (enhance_job*)arg;
  j->rc = 0;
  for (int64_t b = j->lo + j->first; b < j->hi; b += j->stride) {
    if (j->placement[4 * b] < 0) continue;
    if (enhance_box(j->scale, j->C, j->n_resblocks, j->res_scale, j->weights, j->lr, j->bin_w, j->bin_h,
                    j->boxes + 12 * b, j->placement + 4 * b, j->hr) != 0)
      j->rc = -1;
  }
  return NULL;
}

int ref_enhance_mt(int scale, int C, int n_resblocks, double res_scale, const double* weights,
                   const double* lr, int bin_w, int bin_h, int num_bins, int64_t num_boxes, const int32_t* boxes,
                   const int32_t* placement, int64_t box_lo, int64_t box_hi, double* hr, int nthreads) {
  const int HW = scale * bin_w, HH = scale * bin_h;
  memset(hr, 0, sizeof(double) * (size_t)num_bins * HH * HW * 3);
  if (box_hi > num_boxes) box_hi = num_boxes;
  if (nthreads < 1) nthreads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  enhance_job* jobs = (enhance_job*)malloc(sizeof(enhance_job) * (size_t)nthreads);
  if (!th || !jobs) { free(th); free(jobs); return -1; }
  for (int t = 0; t < nthreads; ++t) {
    enhance_job j = {scale, C, n_resblocks, bin_w, bin_h, res_scale, weights, lr, boxes, placement,
                     box_lo, box_hi, nthreads, t, hr, 0};
    jobs[t] = j;
    pthread_create(&th[t], NULL, enhance_worker, &jobs[t]);
  }
  int rc = 0;
  for (int t = 0; t < nthreads; ++t) {
    pthread_join(th[t], NULL);
    if (jobs[t].rc) rc = -1;
  }
  free(th);
  free(jobs);
  return rc;
}

/* ------------------------------------------------------------------------------------------ */
/* O8. Paste back, P:461-464 output = SR(MB_s) + IN(unselected MBs), IN = bilinear with the same */
/* enlarge factor; "stitching them back to bi-linear-interpolated non-regions". Readings:  */
/* D10 bilinear = half-pixel centres, edge clamp (src = max(0,(d+0.5)/s-0.5)), on u8/255 in fp64; */
/* D9 paste set = the HR square of every selected MB whose box was placed (mb_owner >= 0), taken */
/* from that box's HR bin output, un-rotated: HR box-local (u,v) <- bin HR (s*h-1-v, u) when     */
/* rotated. out: [S][F][s*H][s*W][3] fp64. Frames [f_lo, f_hi) of the flat (s,f) index only.     */
/* ------------------------------------------------------------------------------------------ */
static double lerp_src(int d, int scale, int n, int* i0, int* i1) {
  double src = ((double)d + 0.5) / (double)scale - 0.5;
  if (src < 0.0) src = 0.0;
  int a = (int)floor(src);
  if (a > n - 1) a = n - 1;
  *i0 = a;
  *i1 = a + 1 < n ? a + 1 : n - 1;
  return src - (double)a;
}

static void scatter_frame(int F, int W, int H, int mb, int scale, const uint8_t* frames, const int32_t* boxes,
                          const int32_t* placement, const int32_t* mb_owner, const double* hr_bins, int bin_w,
                          int bin_h, int64_t sf, double* o) {
  (void)F;
  const int GW = grid_w(W, mb), GH = grid_h(H, mb);
  const int OW = W * scale, OH = H * scale;
  const int HW = scale * bin_w, HH = scale * bin_h;
  const uint8_t* img = frames + sf * (int64_t)H * W * 3;
  for (int Y = 0; Y < OH; ++Y) {
    int y0, y1;
    const double ly = lerp_src(Y, scale, H, &y0, &y1);
    for (int X = 0; X < OW; ++X) {
      const int mx = X / (mb * scale), my = Y / (mb * scale);
      const int32_t b = mb_owner[sf * GH * GW + (int64_t)my * GW + mx];
      double* px = o + ((int64_t)Y * OW + X) * 3;
      if (b >= 0) {
        const int32_t* bx = boxes + 12 * b;
        const int32_t* pl = placement + 4 * b;
        const int u = X - scale * bx[6], v = Y - scale * bx[7];
        int bxp, byp;
        if (pl[3]) { bxp = scale * pl[1] + (scale * bx[9] - 1 - v); byp = scale * pl[2] + u; }
        else { bxp = scale * pl[1] + u; byp = scale * pl[2] + v; }
        const double* src = hr_bins + (((int64_t)pl[0] * HH + byp) * HW + bxp) * 3;
        px[0] = src[0]; px[1] = src[1]; px[2] = src[2];
      } else {
        int x0, x1;
        const double lx = lerp_src(X, scale, W, &x0, &x1);
        for (int c = 0; c < 3; ++c) {
          const double p00 = img[((int64_t)y0 * W + x0) * 3 + c] / 255.0;
          const double p01 = img[((int64_t)y0 * W + x1) * 3 + c] / 255.0;
          const double p10 = img[((int64_t)y1 * W + x0) * 3 + c] / 255.0;
          const double p11 = img[((int64_t)y1 * W + x1) * 3 + c] / 255.0;
          px[c] = (1.0 - ly) * ((1.0 - lx) * p00 + lx * p01) + ly * ((1.0 - lx) * p10 + lx * p11);
        }
      }
    }
  }
}

int ref_scatter(int S, int F, int W, int H, int mb, int scale, const uint8_t* frames, const int32_t* boxes,
                const int32_t* placement, const int32_t* mb_owner, const double* hr_bins, int bin_w, int bin_h,
                int64_t f_lo, int64_t f_hi, double* out) {
  const int64_t frame_px = (int64_t)H * scale * W * scale * 3;
  for (int64_t sf = f_lo; sf < f_hi && sf < (int64_t)S * F; ++sf)
    scatter_frame(F, W, H, mb, scale, frames, boxes, placement, mb_owner, hr_bins, bin_w, bin_h, sf,
                  out + (sf - f_lo) * frame_px);
  return 0;
}

typedef struct {
  int F, W, H, mb, scale, bin_w, bin_h;
  const uint8_t* frames;
  const int32_t *boxes, *placement, *mb_owner;
  const double* hr_bins;
  int64_t lo, hi, stride, first;
  double* out;
} scatter_job;

static void* scatter_worker(void* arg) {
  scatter_job* j = (scatter_job*)arg;
  const int64_t frame_px = (int64_t)j->H * j->scale * j->W * j->scale * 3;
  for (int64_t sf = j->lo + j->first; sf < j->hi; sf += j->stride)
    scatter_frame(j->F, j->W, j->H, j->mb, j->scale, j->frames, j->boxes, j->placement, j->mb_owner, j->hr_bins,
                  j->bin_w, j->bin_h, sf, j->out + (sf - j->lo) * frame_px);
  return NULL;
}

int ref_scatter_mt(int S, int F, int W, int H, int mb, int scale, const uint8_t* frames, const int32_t* boxes,
                   const int32_t* placement, const int32_t* mb_owner, const double* hr_bins, int bin_w, int bin_h,
                   int64_t f_lo, int64_t f_hi, double* out, int nthreads) {
  if (f_hi > (int64_t)S * F) f_hi = (int64_t)S * F;
  if (nthreads < 1) nthreads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  scatter_job* jobs = (scatter_job*)malloc(sizeof(scatter_job) * (size_t)nthreads);
  if (!th || !jobs) { free(th); free(jobs); return -1; }
  for (int t = 0; t < nthreads; ++t) {
    scatter_job j = {F, W, H, mb, scale, bin_w, bin_h, frames, boxes, placement, mb_owner, hr_bins,
                     f_lo, f_hi, nthreads, t, out};
    jobs[t] = j;
    pthread_create(&th[t], NULL, scatter_worker, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
  return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* D20 u8 output (SURVEY §8(c) "u8 output (clamp, round-half-even)"): the HR frame of O8 as 8-bit */
/* codes. A pasted pixel (mb_owner >= 0) of fp64 value v: rhe(clamp(v, 0, 1) * 255). A bilinear   */
/* pixel: D10's value times 255, exactly: the source coordinate (d + 0.5)/s - 0.5 = (2d + 1 - s)   */
/* / (2s), clamped at 0, has integer part i0 and fraction a/(2s); the value is N / (2s)^2 with     */
/* N = (2s-b)((2s-a) p00 + a p01) + b((2s-a) p10 + a p11) over the u8 codes, rounded half to even */
/* in integers. hr_frames: the fp64 frames of ref_scatter for [f_lo, f_hi); out likewise, u8.     */
/* ------------------------------------------------------------------------------------------ */
static int rhe_double(double v) {
  double c = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
  double x = c * 255.0, fl = floor(x);
  int q = (int)fl;
  if (x - fl > 0.5 || (x - fl == 0.5 && (q & 1))) ++q;
  return q;
}

static void src_num(int d, int scale, int n, int* i0, int* i1, int* a) {
  int num = 2 * d + 1 - scale; /* source coordinate times 2s */
  if (num < 0) num = 0;
  *i0 = num / (2 * scale);
  *a = num - 2 * scale * *i0;
  if (*i0 > n - 1) { *i0 = n - 1; *a = 0; }
  *i1 = *i0 + 1 < n ? *i0 + 1 : n - 1;
}

int ref_quantize_u8(int S, int F, int W, int H, int mb, int scale, const uint8_t* frames, const int32_t* mb_owner,
                    const double* hr_frames, int64_t f_lo, int64_t f_hi, uint8_t* out) {
  const int GW = grid_w(W, mb), GH = grid_h(H, mb);
  const int OW = W * scale, OH = H * scale, s2 = 2 * scale, D = s2 * s2;
  for (int64_t sf = f_lo; sf < f_hi && sf < (int64_t)S * F; ++sf) {
    const uint8_t* img = frames + sf * (int64_t)H * W * 3;
    const double* fr = hr_frames + (sf - f_lo) * (int64_t)OH * OW * 3;
    uint8_t* o = out + (sf - f_lo) * (int64_t)OH * OW * 3;
    for (int Y = 0; Y < OH; ++Y) {
      int y0, y1, b;
      src_num(Y, scale, H, &y0, &y1, &b);
      for (int X = 0; X < OW; ++X) {
        const int32_t own = mb_owner[sf * GH * GW + (int64_t)(Y / (mb * scale)) * GW + X / (mb * scale)];
        for (int c = 0; c < 3; ++c) {
          const int64_t e = ((int64_t)Y * OW + X) * 3 + c;
          if (own >= 0) {
            o[e] = (uint8_t)rhe_double(fr[e]);
          } else {
            int x0, x1, a;
            src_num(X, scale, W, &x0, &x1, &a);
            const int p00 = img[((int64_t)y0 * W + x0) * 3 + c], p01 = img[((int64_t)y0 * W + x1) * 3 + c];
            const int p10 = img[((int64_t)y1 * W + x0) * 3 + c], p11 = img[((int64_t)y1 * W + x1) * 3 + c];
            const int N = (s2 - b) * ((s2 - a) * p00 + a * p01) + b * ((s2 - a) * p10 + a * p11);
            int q = N / D;
            const int r = N - q * D;
            if (2 * r > D || (2 * r == D && (q & 1))) ++q;
            o[e] = (uint8_t)q;
          }
        }
      }
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* f3. Temporal MB-importance reuse, §3.2.2: the 1/Area operator Phi of one frame's   */
/* Y-channel residual (Appx D.2 P:1625-1628: "1/Area captures the change of small    */
/* objects"). Readings (D18): foreground = |residual| > thr; components are           */
/* 4-connected (BFS flood fill in raster order); Phi = sum over components of 1/area, each term  */
/* the correctly rounded fp64 1.0/area and the sum the exact sum of those terms rounded once to */
/* fp64 (an order-independent definition: terms are multiples of 2^-80 for areas < 2^28, so an  */
/* __int128 accumulator of term * 2^80 is exact). Returns Phi; *ncomp = number of components.   */
/* ------------------------------------------------------------------------------------------ */
double ref_phi_inv_area(int W, int H, const int16_t* res, int thr, int64_t* ncomp) {
  const int64_t n = (int64_t)W * H;
  uint8_t* seen = (uint8_t*)calloc((size_t)(n > 0 ? n : 1), 1);
  int64_t* queue = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  __int128 acc = 0;
  int64_t nc = 0;
  for (int64_t start = 0; start < n; ++start) {
    const int v0 = res[start] < 0 ? -res[start] : res[start];
    if (v0 <= thr || seen[start]) continue;
    int64_t head = 0, tail = 0, area = 0;
    seen[start] = 1;
    queue[tail++] = start;
    while (head < tail) {
      const int64_t c = queue[head++];
      const int cx = (int)(c % W), cy = (int)(c / W);
      ++area;
      const int nx[4] = {cx, cx - 1, cx + 1, cx}, ny[4] = {cy - 1, cy, cy, cy + 1};
      for (int d = 0; d < 4; ++d) {
        if (nx[d] < 0 || ny[d] < 0 || nx[d] >= W || ny[d] >= H) continue;
        const int64_t nb = (int64_t)ny[d] * W + nx[d];
        const int v = res[nb] < 0 ? -res[nb] : res[nb];
        if (v > thr && !seen[nb]) {
          seen[nb] = 1;
          queue[tail++] = nb;
        }
      }
    }
    ++nc;
    const double t = 1.0 / (double)area;            /* correctly rounded term */
    acc += (__int128)ldexp(t, 80);                   /* exact: t is a multiple of 2^-80 */
  }
  free(seen);
  free(queue);
  if (ncomp) *ncomp = nc;
  return ldexp((double)acc, -80);                    /* int128 -> double: round to nearest even */
}

/* ------------------------------------------------------------------------------------------ */
/* f4. NV12 decoder output ("decoded into frames") to the RGB8 frames the path reads.     */
/* Reading D19: ITU-R BT.601 limited range in the common 8-bit integer form                     */
/*   C = Y-16, D = U-128, E = V-128; R = clip((298C + 409E + 128) >> 8),                        */
/*   G = clip((298C - 100D - 208E + 128) >> 8), B = clip((298C + 516D + 128) >> 8),              */
/* chroma of pixel (x, y) = the U/V sample (x/2, y/2) (nearest). NV12 frame = Y plane [H][W]    */
/* then interleaved U,V plane [H/2][W/2][2]; out [frames][H][W][3].                             */
/* ------------------------------------------------------------------------------------------ */
static int clip255(int v) { return v < 0 ? 0 : (v > 255 ? 255 : v); }

int ref_nv12_to_rgb8(int64_t frames, int W, int H, const uint8_t* nv12, uint8_t* rgb) {
  for (int64_t f = 0; f < frames; ++f) {
    const uint8_t* Y = nv12 + f * (int64_t)W * H * 3 / 2;
    const uint8_t* UV = Y + (int64_t)W * H;
    uint8_t* out = rgb + f * (int64_t)W * H * 3;
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x) {
        const int C = Y[(int64_t)y * W + x] - 16;
        const int D = UV[(int64_t)(y / 2) * W + 2 * (x / 2)] - 128;
        const int E = UV[(int64_t)(y / 2) * W + 2 * (x / 2) + 1] - 128;
        uint8_t* px = out + ((int64_t)y * W + x) * 3;
        px[0] = (uint8_t)clip255((298 * C + 409 * E + 128) >> 8);
        px[1] = (uint8_t)clip255((298 * C - 100 * D - 208 * E + 128) >> 8);
        px[2] = (uint8_t)clip255((298 * C + 516 * D + 128) >> 8);
      }
  }
  return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* f1. Placement policies beside the guillotine reading. Common frame: a bin is  */
/* W columns x (H + g) rows, column 0 reserved (D8); a box needs a (w+g) x (h+g) footprint,      */
/* (h+g) x (w+g) when rotated; boxes are taken in the given order; bins are opened lazily in     */
/* index order; RotatePacking prefers the unrotated footprint; placement record as   */
/* ref_pack; a box that fits nowhere is unplaced.                                                */
/* ------------------------------------------------------------------------------------------ */

/* Alg. 2 InnerFree read literally (D14): the maximal empty rectangle of a bin's free cells.     */
/* left[y][x] = free cells ending at (x, y) going left; for each column x (Alg. 2's outer loop   */
/* over j), the largest rectangle under the histogram left[.][x] by the monotone stack (pop      */
/* while left[top] >= left[y]: down[top] = y; up[y] = top); the first maximal area in (x, y)     */
/* order wins. occ: [Hg][W] bytes, 1 = used. out: x, y, w, h (all 0 if the bin is full).         */
void ref_max_empty_rect(const uint8_t* occ, int W, int Hg, int32_t* out) {
  int* left = (int*)malloc(sizeof(int) * (size_t)W * Hg);
  int* up = (int*)malloc(sizeof(int) * (size_t)Hg);
  int* down = (int*)malloc(sizeof(int) * (size_t)Hg);
  int* stk = (int*)malloc(sizeof(int) * (size_t)Hg);
  for (int y = 0; y < Hg; ++y)
    for (int x = 0; x < W; ++x)
      left[y * W + x] = occ[(int64_t)y * W + x] ? 0 : (x > 0 ? left[y * W + x - 1] : 0) + 1;
  int64_t best = 0;
  out[0] = out[1] = out[2] = out[3] = 0;
  for (int x = 0; x < W; ++x) {
    int top = 0;
    for (int y = 0; y < Hg; ++y) {
      up[y] = -1;
      down[y] = Hg;
    }
    for (int y = 0; y < Hg; ++y) {
      while (top > 0 && left[stk[top - 1] * W + x] >= left[y * W + x]) down[stk[--top]] = y;
      up[y] = top > 0 ? stk[top - 1] : -1;
      stk[top++] = y;
    }
    for (int y = 0; y < Hg; ++y) {
      const int l = left[y * W + x];
      const int64_t area = (int64_t)(down[y] - up[y] - 1) * l;
      if (area > best) {
        best = area;
        out[0] = x - l + 1; out[1] = up[y] + 1; out[2] = l; out[3] = down[y] - up[y] - 1;
      }
    }
  }
  free(left); free(up); free(down); free(stk);
}

static void pack_init_placement(int64_t n, int32_t* placement) {
  for (int64_t i = 0; i < n; ++i)
    placement[4 * i] = -1, placement[4 * i + 1] = 0, placement[4 * i + 2] = 0, placement[4 * i + 3] = 0;
}

int ref_pack_maxrect(int64_t num_boxes, const int32_t* boxes, const int32_t* order, int bin_w, int bin_h,
                     int max_bins, int gutter, int32_t* placement, int32_t* num_bins) {
  const int W = bin_w, Hg = bin_h + gutter;
  uint8_t* occ = (uint8_t*)calloc((size_t)(max_bins > 0 ? max_bins : 1) * W * Hg, 1);
  int32_t* mer = (int32_t*)malloc(sizeof(int32_t) * 4 * (size_t)(max_bins > 0 ? max_bins : 1));
  int opened = 0, used = 0;
  pack_init_placement(num_boxes, placement);
  for (int64_t oi = 0; oi < num_boxes; ++oi) {
    const int32_t b = order[oi];
    const int pw = boxes[12 * b + 8] + gutter, ph = boxes[12 * b + 9] + gutter;
    int bin = -1;
    for (int k = 0; k <= opened && k < max_bins; ++k) {   /* freeareas: one MER per bin, bin order */
      if (k == opened) {                                  /* open the next bin lazily */
        uint8_t* o = occ + (size_t)k * W * Hg;
        for (int y = 0; y < Hg; ++y) o[(int64_t)y * W] = 1;   /* reserved column 0 */
        ref_max_empty_rect(o, W, Hg, mer + 4 * k);
      }
      const int fw = mer[4 * k + 2], fh = mer[4 * k + 3];
      if ((fw >= pw && fh >= ph) || (fw >= ph && fh >= pw)) { bin = k; break; }
      if (k == opened) break;                             /* not even a fresh bin admits it */
    }
    if (bin < 0) continue;
    if (bin == opened) ++opened;
    const int32_t* r = mer + 4 * bin;
    const int rot = !(r[2] >= pw && r[3] >= ph);
    const int uw = rot ? ph : pw, uh = rot ? pw : ph;
    placement[4 * b] = bin; placement[4 * b + 1] = r[0]; placement[4 * b + 2] = r[1]; placement[4 * b + 3] = rot;
    if (bin + 1 > used) used = bin + 1;
    uint8_t* o = occ + (size_t)bin * W * Hg;
    for (int y = r[1]; y < r[1] + uh; ++y)
      for (int x = r[0]; x < r[0] + uw; ++x) o[(int64_t)y * W + x] = 1;
    ref_max_empty_rect(o, W, Hg, mer + 4 * bin);            /* Update: the bin's new free area */
  }
  free(occ);
  free(mer);
  *num_bins = used;
  return 0;
}

/* D15 skyline bottom-left: a bin's skyline is the height of the used part of every column      */
/* (column 0 reserved: full). A footprint uw x uh can rest at x (1 <= x, x + uw <= W) at          */
/* y = max height over [x, x+uw), if y + uh <= H + g; the lowest y wins, then the leftmost x. In  */
/* the first bin (index order) that admits the box: the best unrotated position if there is one, */
/* else the best rotated one; the columns under the footprint rise to y + uh.                    */
static int sky_best(const int32_t* hgt, int W, int Hg, int uw, int uh, int* bx, int* by) {
  int found = 0;
  for (int x = 1; x + uw <= W; ++x) {
    int y = 0;
    for (int c = x; c < x + uw; ++c) y = hgt[c] > y ? hgt[c] : y;
    if (y + uh > Hg) continue;
    if (!found || y < *by || (y == *by && x < *bx)) { *bx = x; *by = y; found = 1; }
  }
  return found;
}

int ref_pack_skyline(int64_t num_boxes, const int32_t* boxes, const int32_t* order, int bin_w, int bin_h,
                     int max_bins, int gutter, int32_t* placement, int32_t* num_bins) {
  const int W = bin_w, Hg = bin_h + gutter;
  int32_t* hgt = (int32_t*)calloc((size_t)(max_bins > 0 ? max_bins : 1) * W, sizeof(int32_t));
  int opened = 0, used = 0;
  pack_init_placement(num_boxes, placement);
  for (int64_t oi = 0; oi < num_boxes; ++oi) {
    const int32_t b = order[oi];
    const int pw = boxes[12 * b + 8] + gutter, ph = boxes[12 * b + 9] + gutter;
    for (int k = 0; k <= opened && k < max_bins; ++k) {
      int32_t* h = hgt + (size_t)k * W;
      if (k == opened) h[0] = Hg;                          /* fresh bin: column 0 reserved */
      int x = 0, y = 0, rot = 0;
      if (sky_best(h, W, Hg, pw, ph, &x, &y)) rot = 0;
      else if (sky_best(h, W, Hg, ph, pw, &x, &y)) rot = 1;
      else {
        if (k == opened) break;
        continue;
      }
      if (k == opened) ++opened;
      const int uw = rot ? ph : pw, uh = rot ? pw : ph;
      for (int c = x; c < x + uw; ++c) h[c] = y + uh;
      placement[4 * b] = k; placement[4 * b + 1] = x; placement[4 * b + 2] = y; placement[4 * b + 3] = rot;
      if (k + 1 > used) used = k + 1;
      break;
    }
  }
  free(hgt);
  *num_bins = used;
  return 0;
}

/* D16 first-fit shelves: a bin holds shelves (y0, height, end x) in creation order and the y of   */
/* its next shelf. A box goes on the first shelf (bin order, then shelf order) where it fits      */
/* unrotated (height <= shelf height, end + width <= W), else rotated; otherwise, in the same    */
/* bin, on a new shelf at the bin's next y if the bin has the height (unrotated preferred; the    */
/* new shelf's height is the box's); otherwise the next bin. Shelves start at x = 1 (column 0).  */
#define SHELF_CAP 256
int ref_pack_shelf(int64_t num_boxes, const int32_t* boxes, const int32_t* order, int bin_w, int bin_h,
                   int max_bins, int gutter, int32_t* placement, int32_t* num_bins) {
  const int W = bin_w, Hg = bin_h + gutter;
  const size_t nb = (size_t)(max_bins > 0 ? max_bins : 1);
  int32_t* sy = (int32_t*)malloc(sizeof(int32_t) * nb * SHELF_CAP);
  int32_t* sh = (int32_t*)malloc(sizeof(int32_t) * nb * SHELF_CAP);
  int32_t* sx = (int32_t*)malloc(sizeof(int32_t) * nb * SHELF_CAP);
  int32_t* ns = (int32_t*)calloc(nb, sizeof(int32_t));
  int32_t* top = (int32_t*)calloc(nb, sizeof(int32_t));
  int opened = 0, used = 0, rc = 0;
  pack_init_placement(num_boxes, placement);
  for (int64_t oi = 0; oi < num_boxes; ++oi) {
    const int32_t b = order[oi];
    const int pw = boxes[12 * b + 8] + gutter, ph = boxes[12 * b + 9] + gutter;
    for (int k = 0; k <= opened && k < max_bins; ++k) {
      int px = -1, py = 0, rot = 0;
      for (int s = 0; s < ns[k] && px < 0; ++s) {
        const size_t i = (size_t)k * SHELF_CAP + s;
        if (ph <= sh[i] && sx[i] + pw <= W) { px = sx[i]; py = sy[i]; rot = 0; sx[i] += pw; }
        else if (pw <= sh[i] && sx[i] + ph <= W) { px = sx[i]; py = sy[i]; rot = 1; sx[i] += ph; }
      }
      if (px < 0 && ns[k] < SHELF_CAP) {
        int hh = 0, ww = 0;
        if (top[k] + ph <= Hg && 1 + pw <= W) { hh = ph; ww = pw; rot = 0; }
        else if (top[k] + pw <= Hg && 1 + ph <= W) { hh = pw; ww = ph; rot = 1; }
        if (hh > 0) {
          const size_t i = (size_t)k * SHELF_CAP + ns[k]++;
          sy[i] = top[k]; sh[i] = hh; sx[i] = 1 + ww;
          px = 1; py = top[k];
          top[k] += hh;
        }
      } else if (px < 0) {
        rc = 2;   /* shelf table full */
      }
      if (px < 0) {
        if (k == opened) break;
        continue;
      }
      if (k == opened) ++opened;
      placement[4 * b] = k; placement[4 * b + 1] = px; placement[4 * b + 2] = py; placement[4 * b + 3] = rot;
      if (k + 1 > used) used = k + 1;
      break;
    }
  }
  free(sy); free(sh); free(sx); free(ns); free(top);
  *num_bins = used;
  return rc;
}
