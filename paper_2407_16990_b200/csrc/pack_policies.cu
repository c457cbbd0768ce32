// the packing-policy suite beside the guillotine reading of Alg. 1 (pack.cu).
//
//   MAXRECT  (D14) Alg. 2 InnerFree read literally: each opened bin's free area is the maximal empty
//            rectangle of its free cells (histogram-stack method), recomputed after every
//            placement (one thread per column: the run of free cells ending at (x, y) going left,
//            and a monotone stack over y; the first maximal area in (x, y) order).
//   SKYLINE  (D15) bottom-left on a per-column height profile: the lowest, then leftmost resting place
//            (unrotated preferred within a bin).
//   SHELF    (D16) first-fit shelves (shelf order within the bin, then a new shelf at the bin's top).
//
// All three keep Alg. 1's outer structure (boxes in the given order, bins scanned in index order and
// opened lazily, RotatePacking prefers the unrotated footprint, D7/D8 footprint and reserved column)
// and match the oracle's placements bit for bit. One CTA of PP_THREADS threads per call: the decision
// for one box is taken cooperatively (candidate bins by a per-bin summary filter, then a block-wide
// search inside the first candidate), the boxes one after the other. These are comparison policies
// (the survey's fill study); the hot path's default is the guillotine packer.
#include <algorithm>

#include "common.cuh"

namespace regen {

constexpr int PP_THREADS = 256;
constexpr int PP_MAX_BINS = 8192;
constexpr int SHELF_CAP = 256;   // shelves per bin (as the oracle)
constexpr int SKY_NW = 8;        // SKYLINE summary widths 4, 8, ..., 512
__host__ __device__ constexpr int sky_w(int i) { return 4 << i; }

// SKYLINE filter: a footprint uw x uh can rest in bin k only if, for the widest summary width w <= uw,
// the lowest resting height of a w-wide footprint (<= that of the uw-wide one) leaves uh rows
__device__ __forceinline__ bool sky_may_fit(const int16_t* lw, int uw, int uh, int Hg) {
  if (uw < sky_w(0)) return true;   // narrower than every summary width: no filter
  int i = 0;
  while (i + 1 < SKY_NW && sky_w(i + 1) <= uw) ++i;
  return lw[i] + uh <= Hg;
}

struct PolicyArgs {
  regen_box* boxes;
  const int32_t* order;
  const int64_t* num_boxes;
  int64_t max_boxes;
  int32_t* num_bins;
  int32_t* status;
  int bin_w, bin_h, max_bins, gutter, policy;
  // workspace, per bin
  uint32_t* occ;      // MAXRECT: [max_bins][Hg][W32] occupancy bits
  int4* mer;          // MAXRECT: [max_bins] the bin's free area (x, y, w, h)
  int16_t* hgt;       // SKYLINE: [max_bins][W] column heights
  int16_t* lw;        // SKYLINE: [max_bins][SKY_NW] lowest resting height of a footprint SKY_W(i) wide
  int16_t* sy;        // SHELF: [max_bins][SHELF_CAP] shelf y0, height, end x
  int16_t* sh;
  int16_t* sx;
  int32_t* ns;        // SHELF: [max_bins] shelves, next y
  int32_t* top;
  short2* stack;      // MAXRECT: [PP_THREADS][Hg] per-thread stacks (y, left)
};

__device__ __forceinline__ bool rp_fits(int fw, int fh, int pw, int ph) {   // RotatePacking
  return (fw >= pw && fh >= ph) || (fw >= ph && fh >= pw);
}

// block-wide minimum of a 64-bit key (all threads get it)
__device__ __forceinline__ unsigned long long block_min64(unsigned long long v, unsigned long long* red) {
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  unsigned long long m = red[0];
  for (int i = 1; i < PP_THREADS / 32; ++i) m = red[i] < m ? red[i] : m;
  return m;
}

// ---------------------------------------------------------------------------------- MAXRECT

// free-cell run ending at column x of a row (bits: 1 = used): x - (last used column <= x)
__device__ __forceinline__ int left_run(const uint32_t* row, int x) {
  int w = x >> 5;
  uint32_t m = row[w] & (0xFFFFFFFFu >> (31 - (x & 31)));   // bits 0..x&31
  while (m == 0 && w > 0) m = row[--w];
  if (m == 0) return x + 1;
  return x - (32 * w + 31 - __clz(m));
}

// the maximal empty rectangle of bin b (Alg. 2): every thread takes columns t, t + PP_THREADS, ...
__device__ void mer_recompute(const PolicyArgs& a, int b, unsigned long long* red) {
  const int W = a.bin_w, Hg = a.bin_h + a.gutter, W32 = (W + 31) / 32;
  const uint32_t* occ = a.occ + (size_t)b * Hg * W32;
  short2* stk = a.stack + (size_t)threadIdx.x * Hg;
  // key: area (high), then the smallest x, then the smallest y (the oracle's first strict maximum)
  unsigned long long best = ~0ull;
  int bx = 0, by = 0, bw = 0, bh = 0;
  for (int x = threadIdx.x; x < W; x += PP_THREADS) {
    int top = 0;
    for (int y = 0; y <= Hg; ++y) {
      const int l = y < Hg ? left_run(occ + (size_t)y * W32, x) : -1;   // y == Hg: flush the stack
      while (top > 0 && stk[top - 1].y >= l) {
        const short2 e = stk[--top];
        const int up = top > 0 ? stk[top - 1].x : -1;
        const long long area = (long long)(y - up - 1) * e.y;
        // e was pushed at row e.x: its rectangle spans rows up+1 .. y-1
        const unsigned long long key =
            ((unsigned long long)(0xFFFFFFFFll - area) << 32) | ((unsigned long long)x << 16) | (unsigned)e.x;
        if (area > 0 && key < best) { best = key; bx = x - e.y + 1; by = up + 1; bw = e.y; bh = y - up - 1; }
      }
      if (y < Hg) stk[top++] = make_short2((short)y, (short)l);
    }
  }
  const unsigned long long m = block_min64(best, red);
  if (m != ~0ull && best == m) a.mer[b] = make_int4(bx, by, bw, bh);
  if (m == ~0ull && threadIdx.x == 0) a.mer[b] = make_int4(0, 0, 0, 0);
  __syncthreads();
}

// ---------------------------------------------------------------------------------- kernel

__global__ void __launch_bounds__(PP_THREADS, 1) pack_policy_kernel(PolicyArgs a) {
  __shared__ unsigned long long red[PP_THREADS / 32];
  __shared__ int16_t sum_a[PP_MAX_BINS];   // per bin: a necessary condition for admitting a footprint
  const int W = a.bin_w, Hg = a.bin_h + a.gutter, W32 = (W + 31) / 32;
  const int64_t n = min(*a.num_boxes, a.max_boxes);
  int opened = 0, used = 0;
  bool overflow = false;
  for (int64_t oi = 0; oi < n; ++oi) {
    const int b = a.order[oi];
    const int pw = a.boxes[b].w + a.gutter, ph = a.boxes[b].h + a.gutter;
    const int qa = min(pw, ph);
    int placed_bin = -1, px = 0, py = 0, rot = 0;
    int from = 0;   // next bin to examine
    while (placed_bin < 0) {
      // first candidate bin >= from (summary filter), the fresh bin `opened` always a candidate
      unsigned long long c = ~0ull;
      for (int k = from + threadIdx.x; k < opened; k += PP_THREADS) {
        bool ok = sum_a[k] >= qa;
        if (ok && a.policy == REGEN_POLICY_SKYLINE) {
          const int16_t* lw = a.lw + (size_t)k * SKY_NW;
          ok = sky_may_fit(lw, pw, ph, Hg) || sky_may_fit(lw, ph, pw, Hg);
        }
        if (ok) { c = (unsigned long long)k; break; }
      }
      unsigned long long cand = block_min64(c, red);
      int k = cand == ~0ull ? opened : (int)cand;
      if (k >= a.max_bins) break;
      const bool fresh = k == opened;
      if (fresh) {   // open the next bin lazily (its state initialised; `opened` advances only if used)
        if (a.policy == REGEN_POLICY_MAXRECT) {
          uint32_t* o = a.occ + (size_t)k * Hg * W32;
          for (int i = threadIdx.x; i < Hg * W32; i += PP_THREADS) o[i] = (i % W32 == 0) ? 1u : 0u;
          if (threadIdx.x == 0) a.mer[k] = make_int4(1, 0, W - 1, Hg);
        } else if (a.policy == REGEN_POLICY_SKYLINE) {
          int16_t* h = a.hgt + (size_t)k * W;
          for (int i = threadIdx.x; i < W; i += PP_THREADS) h[i] = i == 0 ? (int16_t)Hg : (int16_t)0;
        } else {
          if (threadIdx.x == 0) { a.ns[k] = 0; a.top[k] = 0; }
        }
        __syncthreads();
      }
      // ---- does bin k admit the box? where?
      if (a.policy == REGEN_POLICY_MAXRECT) {
        const int4 r = a.mer[k];
        if (rp_fits(r.z, r.w, pw, ph)) {
          placed_bin = k;
          rot = !(r.z >= pw && r.w >= ph);
          px = r.x;
          py = r.y;
        }
      } else if (a.policy == REGEN_POLICY_SKYLINE) {
        const int16_t* h = a.hgt + (size_t)k * W;
        for (int o = 0; o < 2 && placed_bin < 0; ++o) {   // unrotated first, within the bin
          const int uw = o ? ph : pw, uh = o ? pw : ph;
          unsigned long long best = ~0ull;
          for (int x = 1 + threadIdx.x; x + uw <= W; x += PP_THREADS) {
            int y = 0;
            for (int cc = x; cc < x + uw; ++cc) y = max(y, (int)h[cc]);
            if (y + uh <= Hg) {
              const unsigned long long key = ((unsigned long long)y << 32) | (unsigned)x;
              best = key < best ? key : best;
            }
          }
          const unsigned long long m = block_min64(best, red);
          if (m != ~0ull) {
            placed_bin = k;
            rot = o;
            px = (int)(m & 0xFFFFFFFFu);
            py = (int)(m >> 32);
          }
        }
      } else {   // SHELF
        const int nsh = a.ns[k];
        unsigned long long best = ~0ull;   // (shelf index << 1 | rotated)
        for (int s = threadIdx.x; s < nsh; s += PP_THREADS) {
          const size_t i = (size_t)k * SHELF_CAP + s;
          const int hh = a.sh[i], xe = a.sx[i];
          unsigned long long key = ~0ull;
          if (ph <= hh && xe + pw <= W) key = (unsigned long long)s << 1;
          else if (pw <= hh && xe + ph <= W) key = ((unsigned long long)s << 1) | 1ull;
          best = key < best ? key : best;
        }
        const unsigned long long m = block_min64(best, red);
        if (m != ~0ull) {
          const int s = (int)(m >> 1);
          const size_t i = (size_t)k * SHELF_CAP + s;
          placed_bin = k;
          rot = (int)(m & 1);
          px = a.sx[i];
          py = a.sy[i];
          __syncthreads();
          if (threadIdx.x == 0) a.sx[i] = (int16_t)(px + (rot ? ph : pw));
        } else if (nsh < SHELF_CAP) {
          const int t = a.top[k];
          int hh = 0, ww = 0;
          if (t + ph <= Hg && 1 + pw <= W) { hh = ph; ww = pw; rot = 0; }
          else if (t + pw <= Hg && 1 + ph <= W) { hh = pw; ww = ph; rot = 1; }
          if (hh > 0) {
            placed_bin = k;
            px = 1;
            py = t;
            __syncthreads();
            if (threadIdx.x == 0) {
              const size_t i = (size_t)k * SHELF_CAP + nsh;
              a.sy[i] = (int16_t)t; a.sh[i] = (int16_t)hh; a.sx[i] = (int16_t)(1 + ww);
              a.ns[k] = nsh + 1;
              a.top[k] = t + hh;
            }
          }
        } else {
          overflow = true;
        }
      }
      __syncthreads();
      if (placed_bin < 0) {
        if (fresh) break;      // not even an empty bin admits it: unplaced
        from = k + 1;
        continue;
      }
      if (fresh) ++opened;
    }
    if (placed_bin < 0) continue;
    used = max(used, placed_bin + 1);
    const int k = placed_bin;
    const int uw = rot ? ph : pw, uh = rot ? pw : ph;
    if (threadIdx.x == 0) {
      int2* pl = reinterpret_cast<int2*>(&a.boxes[b].bin);
      pl[0] = make_int2(k, px);
      pl[1] = make_int2(py, rot);
    }
    // ---- update the bin and its summary (sum_a: a footprint whose shorter side exceeds it never fits)
    if (a.policy == REGEN_POLICY_MAXRECT) {
      uint32_t* o = a.occ + (size_t)k * Hg * W32;
      for (int i = threadIdx.x; i < uh * W32; i += PP_THREADS) {
        const int y = py + i / W32, w = i % W32;
        const int lo = max(px, 32 * w), hi = min(px + uw, 32 * w + 32);
        if (lo < hi) {
          const int nb = hi - lo;
          const uint32_t bits = (nb == 32 ? 0xFFFFFFFFu : ((1u << nb) - 1u)) << (lo - 32 * w);
          o[(size_t)y * W32 + w] |= bits;
        }
      }
      __syncthreads();
      mer_recompute(a, k, red);
      if (threadIdx.x == 0) {
        const int4 r = a.mer[k];
        sum_a[k] = (int16_t)min(r.z, r.w);
      }
    } else if (a.policy == REGEN_POLICY_SKYLINE) {
      int16_t* h = a.hgt + (size_t)k * W;
      for (int cc = px + threadIdx.x; cc < px + uw; cc += PP_THREADS) h[cc] = (int16_t)(py + uh);
      __syncthreads();
      // summary: Hg - (lowest column height); a footprint needs its shorter side below that
      unsigned long long lo = ~0ull;
      for (int cc = 1 + threadIdx.x; cc < W; cc += PP_THREADS) lo = min(lo, (unsigned long long)h[cc]);
      const unsigned long long m = block_min64(lo, red);
      if (threadIdx.x == 0) sum_a[k] = (int16_t)(m == ~0ull ? 0 : Hg - (int)m);
      // per-width lowest resting heights (warp i: width sky_w(i); lanes over the positions)
      const int wi = threadIdx.x >> 5;
      if (wi < SKY_NW) {
        const int w = sky_w(wi);
        int best = Hg + 1;
        for (int x = 1 + (threadIdx.x & 31); x + w <= W; x += 32) {
          int y = 0;
          for (int cc = x; cc < x + w; ++cc) y = max(y, (int)h[cc]);
          best = min(best, y);
        }
        best = __reduce_min_sync(0xffffffffu, best);
        if ((threadIdx.x & 31) == 0) a.lw[(size_t)k * SKY_NW + wi] = (int16_t)best;
      }
      __syncthreads();
    } else {
      __syncthreads();
      // summary: the most width left on a shelf, or the height left above the top shelf
      unsigned long long mx = 0;
      const int nsh = a.ns[k];
      for (int s = threadIdx.x; s < nsh; s += PP_THREADS)
        mx = max(mx, (unsigned long long)(W - a.sx[(size_t)k * SHELF_CAP + s]));
      const unsigned long long m = ~block_min64(~mx, red);
      if (threadIdx.x == 0) sum_a[k] = (int16_t)max((int)m, min(Hg - a.top[k], W - 1));
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *a.num_bins = used;
    if (overflow) atomicOr(a.status, REGEN_ST_FREELIST_OVERFLOW);
  }
}

size_t policy_workspace_bytes(const regen_pack_params& p) {
  const size_t Hg = (size_t)p.bin_h + p.gutter, W32 = ((size_t)p.bin_w + 31) / 32, B = (size_t)p.max_bins;
  Carver c(nullptr);
  switch (p.policy) {
    case REGEN_POLICY_MAXRECT:
      c.take<uint32_t>(B * Hg * W32);
      c.take<int4>(B);
      c.take<short2>((size_t)PP_THREADS * Hg);
      break;
    case REGEN_POLICY_SKYLINE:
      c.take<int16_t>(B * p.bin_w);
      c.take<int16_t>(B * SKY_NW);
      break;
    case REGEN_POLICY_SHELF:
      c.take<int16_t>(3 * B * SHELF_CAP);
      c.take<int32_t>(2 * B);
      break;
    default:
      return 0;
  }
  return c.off + 256;
}

regen_status launch_pack_policy(const regen_pack_params& p, regen_box* d_boxes, const int32_t* d_order,
                                const int64_t* d_num_boxes, int64_t max_boxes, int32_t* d_num_bins,
                                int32_t* d_status, void* ws, cudaStream_t s) {
  REGEN_REQUIRE(p.max_bins <= PP_MAX_BINS, "policy packers take at most %d bins", PP_MAX_BINS);
  REGEN_REQUIRE(p.bin_w <= 4096 && p.bin_h + p.gutter <= 32767, "bin too large for the policy packers");
  PolicyArgs a;
  memset(&a, 0, sizeof(a));
  a.boxes = d_boxes;
  a.order = d_order;
  a.num_boxes = d_num_boxes;
  a.max_boxes = max_boxes;
  a.num_bins = d_num_bins;
  a.status = d_status;
  a.bin_w = p.bin_w;
  a.bin_h = p.bin_h;
  a.max_bins = p.max_bins;
  a.gutter = p.gutter;
  a.policy = p.policy;
  const size_t Hg = (size_t)p.bin_h + p.gutter, W32 = ((size_t)p.bin_w + 31) / 32, B = (size_t)p.max_bins;
  Carver c(ws);
  if (p.policy == REGEN_POLICY_MAXRECT) {
    a.occ = c.take<uint32_t>(B * Hg * W32);
    a.mer = c.take<int4>(B);
    a.stack = c.take<short2>((size_t)PP_THREADS * Hg);
  } else if (p.policy == REGEN_POLICY_SKYLINE) {
    a.hgt = c.take<int16_t>(B * p.bin_w);
    a.lw = c.take<int16_t>(B * SKY_NW);
  } else {
    a.sy = c.take<int16_t>(B * SHELF_CAP);
    a.sh = c.take<int16_t>(B * SHELF_CAP);
    a.sx = c.take<int16_t>(B * SHELF_CAP);
    a.ns = c.take<int32_t>(B);
    a.top = c.take<int32_t>(B);
  }
  REGEN_TRACE("pack_policy", s);
  pack_policy_kernel<<<1, PP_THREADS, 0, s>>>(a);
  REGEN_LAUNCH_CHECK();
  return REGEN_OK;
}

}  // namespace regen
