// a3-a5: Bound + expand + Partition + density (Alg. 1 l.4-6), Sort (l.6), Packing (l.7-21, Alg. 2).
//
// box_count/box_write  one warp per region: enumerate the MB-aligned partition pieces (D5), keep
//                      the region's members (warp ballot over the piece span), re-bound them with
//                      warp min/max, drop empty pieces; a scan over regions gives creation-ordered
//                      box indices. Density = fp64 raster-order sum over the span (one lane, D4).
// sort_rank            rank of every box under (density desc, index asc) or (area desc, index asc):
//                      unique keys => order is the exact inverse permutation (SMEM-tiled count).
// pack_kernel          one warp: per-bin free-area lists (slot l owned by lane l) with per-bin and
//                      per-32-bin dominance summaries in SMEM; the first fitting free area in (bin, seq)
//                      order (D12) is found through the summaries; every lane replays the decision and
//                      the guillotine remainders (D6). Unopened bins are implicit.
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"

namespace regen {

size_t select_workspace_bytes(const regen_geom& g);
size_t policy_workspace_bytes(const regen_pack_params& p);
regen_status launch_pack_policy(const regen_pack_params& p, regen_box* d_boxes, const int32_t* d_order,
                                const int64_t* d_num_boxes, int64_t max_boxes, int32_t* d_num_bins,
                                int32_t* d_status, void* ws, cudaStream_t s);

// ------------------------------------------------------------------------------------ boxes

struct BoxArgs {
  const float* imp;
  const int32_t* labels;
  const regen_region* regions;
  const int64_t* num_regions;
  int64_t max_regions;
  int32_t* region_count;     // [max_regions] non-empty pieces per region
  const int64_t* region_off; // [max_regions]
  regen_box* boxes;
  int64_t max_boxes;
  int32_t* box_of_mb;        // [frames][GH][GW] (d_mb_owner, pre-filled with -1)
  int32_t* status;
  int GW, GH, W, H, F, mb, expand, P;
  int density;   // REGEN_DENSITY_SPAN / REGEN_DENSITY_MEMBERS
};

__device__ __forceinline__ int piece_start(int n, int pieces, int i) {
  const int base = n / pieces, rem = n % pieces;
  return i * base + (i < rem ? i : rem);
}

// Enumerates the non-empty pieces of region r with one warp. WRITE=false: count only.
template <bool WRITE>
__device__ int region_pieces(const BoxArgs& a, int64_t r, int64_t box_base) {
  const int lane = threadIdx.x & 31;
  const regen_region rg = a.regions[r];
  const int64_t frame = (int64_t)rg.stream * a.F + rg.frame;
  const int32_t* lab = a.labels + frame * a.GW * a.GH;
  const int wm = rg.mx1 - rg.mx0, hm = rg.my1 - rg.my0;
  const int nx = (wm + a.P - 1) / a.P, ny = (hm + a.P - 1) / a.P;
  int produced = 0;
  for (int py = 0; py < ny; ++py)
    for (int px = 0; px < nx; ++px) {
      const int sx0 = rg.mx0 + piece_start(wm, nx, px), sx1 = rg.mx0 + piece_start(wm, nx, px + 1);
      const int sy0 = rg.my0 + piece_start(hm, ny, py), sy1 = rg.my0 + piece_start(hm, ny, py + 1);
      const int pw = sx1 - sx0, ncell = pw * (sy1 - sy0);
      int mx0 = 1 << 30, my0 = 1 << 30, mx1 = -1, my1 = -1, cnt = 0;
      for (int c = lane; c < ncell; c += 32) {
        const int x = sx0 + c % pw, y = sy0 + c / pw;
        if (lab[y * a.GW + x] == (int32_t)r) {
          ++cnt;
          mx0 = min(mx0, x); my0 = min(my0, y); mx1 = max(mx1, x + 1); my1 = max(my1, y + 1);
        }
      }
      cnt = warp_sum(cnt);
      if (cnt == 0) continue;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mx0 = min(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
        my0 = min(my0, __shfl_xor_sync(0xffffffffu, my0, o));
        mx1 = max(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
        my1 = max(my1, __shfl_xor_sync(0xffffffffu, my1, o));
      }
      if (WRITE) {
        const int64_t b = box_base + produced;
        if (b < a.max_boxes) {
          if (lane == 0) {
            double sum = 0.0;
            const float* sc = a.imp + frame * a.GW * a.GH;
            const bool members = a.density == REGEN_DENSITY_MEMBERS;
            for (int y = my0; y < my1; ++y)
              for (int x = mx0; x < mx1; ++x)
                if (!members || lab[y * a.GW + x] == (int32_t)r) sum = __dadd_rn(sum, (double)sc[y * a.GW + x]);
            regen_box bx;
            bx.stream = rg.stream;
            bx.frame = rg.frame;
            bx.mx0 = mx0; bx.my0 = my0; bx.mx1 = mx1; bx.my1 = my1;
            const int x0 = max(0, a.mb * mx0 - a.expand), y0 = max(0, a.mb * my0 - a.expand);
            const int x1 = min(a.W, a.mb * mx1 + a.expand), y1 = min(a.H, a.mb * my1 + a.expand);
            bx.x0 = x0; bx.y0 = y0; bx.w = x1 - x0; bx.h = y1 - y0;
            bx.n_members = cnt;
            bx.region = (int32_t)r;
            bx.density = __ddiv_rn(sum, (double)(members ? cnt : (mx1 - mx0) * (my1 - my0)));
            bx.bin = -1; bx.bx = 0; bx.by = 0; bx.rotated = 0; bx.rank = 0; bx.reserved = 0;
            a.boxes[b] = bx;
          }
          int32_t* own = a.box_of_mb + frame * a.GW * a.GH;
          const int bw = mx1 - mx0, bc = bw * (my1 - my0);
          for (int c = lane; c < bc; c += 32) {
            const int x = mx0 + c % bw, y = my0 + c / bw;
            if (lab[y * a.GW + x] == (int32_t)r) own[y * a.GW + x] = (int32_t)b;
          }
        } else if (lane == 0) {
          atomicOr(a.status, REGEN_ST_BOX_OVERFLOW);
        }
      }
      ++produced;
    }
  return produced;
}

// warp-stride over the regions actually found (device-side count; the grid is sized to the GPU, not
// to the region capacity)
__global__ void box_count_kernel(BoxArgs a) {
  const int64_t nr = min(*a.num_regions, a.max_regions);
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < nr; r += nw) {
    const int n = region_pieces<false>(a, r, 0);
    if ((threadIdx.x & 31) == 0) a.region_count[r] = n;
  }
}

__global__ void box_write_kernel(BoxArgs a) {
  const int64_t nr = min(*a.num_regions, a.max_regions);
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < nr; r += nw)
    region_pieces<true>(a, r, a.region_off[r]);
}

__global__ void clamp_count_kernel(const int64_t* num_regions, int64_t max_regions, int32_t* region_count,
                                   int64_t* n_out) {
  // regions beyond the (truncated) record count contribute nothing to the scan
  (void)region_count;
  *n_out = min(*num_regions, max_regions);
}

__global__ void scan_counts64_kernel(const int32_t* counts, const int64_t* n_ptr, int64_t* offsets, int64_t* total) {
  __shared__ int scratch[33];
  const int64_t n = *n_ptr;
  int64_t carry = 0;
  for (int64_t base = 0; base < n; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const int c = i < n ? counts[i] : 0;
    int tot;
    const int ex = block_exclusive_scan(c, scratch, &tot);
    if (i < n) offsets[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) *total = carry;
}

// ------------------------------------------------------------------------------------ sort

__device__ __forceinline__ uint64_t box_key(const regen_box& b, int order) {
  return order == REGEN_ORDER_AREA ? (uint64_t)((int64_t)b.w * b.h)
         : order == REGEN_ORDER_HEIGHT ? (uint64_t)b.h : density_ord(b.density);
}

// n <= SORT_SMEM: one CTA bitonic-sorts (key, index) pairs in SMEM (the order is total: keys tie-broken by
// the unique index), else every box counts the boxes ahead of it (O(n^2) tiles, large n only)
constexpr int SORT_SMEM = 4096;   // 48 KB of SMEM: fits beside a resident SR CTA

__device__ __forceinline__ bool sort_before(uint64_t ka, uint32_t ia, uint64_t kb, uint32_t ib) {
  return ka > kb || (ka == kb && ia < ib);   // density (or area) descending, index ascending
}

__global__ void __launch_bounds__(1024) sort_bitonic_kernel(regen_box* boxes, const int64_t* num_boxes,
                                                            int64_t max_boxes, int order, int32_t* out_order) {
  extern __shared__ __align__(16) uint64_t sk[];
  uint32_t* si = reinterpret_cast<uint32_t*>(sk + SORT_SMEM);
  const int64_t n64 = min(*num_boxes, max_boxes);
  if (n64 <= 0 || n64 > SORT_SMEM) return;
  const int n = (int)n64;
  int N = 2;
  while (N < n) N <<= 1;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    sk[i] = i < n ? box_key(boxes[i], order) : 0ull;          // padding sorts last (key 0, index max)
    si[i] = i < n ? (uint32_t)i : 0xFFFFFFFFu;
  }
  __syncthreads();
  for (int k = 2; k <= N; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const uint64_t ka = sk[i], kb = sk[l];
          const uint32_t ia = si[i], ib = si[l];
          const bool sw = (i & k) == 0 ? sort_before(kb, ib, ka, ia) : sort_before(ka, ia, kb, ib);
          if (sw) { sk[i] = kb; sk[l] = ka; si[i] = ib; si[l] = ia; }
        }
      }
      __syncthreads();
    }
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    const uint32_t i = si[p];
    out_order[p] = (int32_t)i;
    boxes[i].rank = p;
  }
}

__global__ void __launch_bounds__(256) sort_rank_kernel(regen_box* boxes, const int64_t* num_boxes, int64_t max_boxes,
                                                        int order, int32_t* out_order) {
  __shared__ uint64_t tile[1024];
  const int64_t n = min(*num_boxes, max_boxes);
  if (n <= SORT_SMEM) return;   // sort_bitonic_kernel
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if ((int64_t)blockIdx.x * blockDim.x >= n) return;
  const uint64_t ki = i < n ? box_key(boxes[i], order) : 0;
  int64_t rank = 0;
  for (int64_t base = 0; base < n; base += 1024) {
    for (int t = threadIdx.x; t < 1024; t += blockDim.x) {
      const int64_t j = base + t;
      tile[t] = j < n ? box_key(boxes[j], order) : 0;
    }
    __syncthreads();
    const int lim = (int)min((int64_t)1024, n - base);
    for (int t = 0; t < lim; ++t) {
      const uint64_t kj = tile[t];
      const int64_t j = base + t;
      rank += (kj > ki) || (kj == ki && j < i);
    }
    __syncthreads();
  }
  if (i < n) {
    out_order[rank] = (int32_t)i;
    boxes[i].rank = (int32_t)rank;
  }
}

// ------------------------------------------------------------------------------------ pack

constexpr int PACK_MAX_BINS = 8192;   // bins one pack call can open (per-bin summaries live in SMEM)
constexpr int PACK_SLOTS = 32;        // live free areas per bin (one per lane; measured <= 10 on every config)

struct PackArgs {
  regen_box* boxes;
  uint64_t* rect;           // [PACK_MAX_BINS][PACK_SLOTS] free areas: x | y<<16 | w<<32 | h<<48 (workspace)
  uint32_t* seqv;           // [PACK_MAX_BINS][PACK_SLOTS] creation sequence of each free area
  uint64_t* pool;           // [2][PACK_POOL] pool path: keys then rects of the slots beyond the registers
  const int32_t* order;
  const int64_t* num_boxes;
  int64_t max_boxes;
  int32_t* num_bins;
  int32_t* status;
  int bin_w, bin_h, max_bins, gutter;
  int prof;         // REGEN_PACK_PROF=1: print per-phase cycle counts
  int slot_limit;   // bins path: live free areas per bin (PACK_SLOTS)
  int pool_limit;   // pool path: live free areas (PACK_POOL + 32). REGEN_PACK_POOL_LIMIT=n lowers both: a
                    // test aid that makes REGEN_ST_FREELIST_OVERFLOW reachable on small inputs
};

// Two data structures for the same sequential Alg. 1 loop (identical placements, both bit-exact
// against the oracle): up to PACK_BINS_FROM boxes a single pool of live areas held in registers (one
// per lane) + SMEM/global overflow (pack_pool: a short dependent chain per box while the pool stays
// small); beyond, per-bin area lists with dominance summaries (pack_bins: per-box cost independent
// of the total number of live areas, which reaches thousands on the 720p 50% and 8-stream groups).
constexpr int PACK_BINS_FROM = 5000;
constexpr int PACK_SMEM = 48 * 1024;   // dynamic SMEM of either path: fits beside a resident SR CTA

constexpr int PACK_POOL = 8192;   // live free areas beyond the register slots (global workspace, L1/L2)
constexpr int PACK_DIMS = 4096;   // box footprints + indices staged in SMEM in packing order (32 KB)
constexpr int PACK_SOV = 1024;    // overflow slots 32 .. 32+PACK_SOV-1 in SMEM (16 KB; 48 KB total so the CTA fits beside a resident SR CTA), the rest global


// One warp. The live free areas of the opened bins form a compact pool: key = bin << 32 | creation
// sequence (unique; its minimum is the first area in (bin, seq) order, D12), rect = x | y<<16 | w<<32
// | h<<48. Slot s < 32 lives in a REGISTER of lane s (the pool holds ~15 areas on the paper's maps
// after pruning), slots >= 32 in a global overflow array (L1-resident). Per box: lanes test their
// areas (fit unrotated or rotated), a warp min-reduction picks the first fit, every lane
// replays the placement and the guillotine remainders (D6) on identical state: the consumed area's
// slot takes the first kept remainder (or the pool's last entry), the second is appended. Unopened
// bins are implicit (opened lazily in order). The packer is one dependent chain per box, so it is
// written for the fewest instructions on that chain: the next footprint is prefetched, a register
// slot update is one predicated move, the clock probes run only under REGEN_PACK_PROF=1.
__device__ __forceinline__ bool fits(uint64_t r, int pw, int ph) {
  const int fw = (int)((r >> 32) & 0xFFFF), fh = (int)(r >> 48);
  return (fw >= pw && fh >= ph) || (fw >= ph && fh >= pw);
}

// Large pools (thousands of live areas on noisy maps / Block mode / 8-stream groups): when the overflow
// part of the pool exceeds PACK_BIG slots, warp 0 hands the fit test of that box to all PACK_WARPS warps
// (named barrier 1: publish the box, each warp scans a strided share of the overflow slots and posts its
// first fit, warp 0 merges the candidates); small pools keep the single-warp path and the helper warps
// sleep on the barrier.
constexpr int PACK_WARPS = 8;
constexpr int PACK_BIG = 192;

// non-.aligned named barrier, entered by whole warps after a __syncwarp (lane-0 branches precede it)
__device__ __forceinline__ void pack_bar() {
  __syncwarp();
  asm volatile("barrier.sync 1, %0;" ::"r"(32 * PACK_WARPS) : "memory");
}

// warp-wide first fit: min key over the lanes' candidates, with the holder's rect and slot
__device__ __forceinline__ void warp_first_fit(uint64_t best, uint64_t brect, int bslot, uint64_t& wkey,
                                               uint64_t& wrect, int& wslot) {
  const uint32_t bhi = (uint32_t)(best >> 32);
  const uint32_t mhi = __reduce_min_sync(0xffffffffu, bhi);
  const uint32_t mlo = __reduce_min_sync(0xffffffffu, bhi == mhi ? (uint32_t)best : 0xFFFFFFFFu);
  wkey = ((uint64_t)mhi << 32) | mlo;
  const uint32_t hold = __ballot_sync(0xffffffffu, best == wkey);
  const int hl = hold ? __ffs(hold) - 1 : 0;
  wrect = __shfl_sync(0xffffffffu, brect, hl);
  wslot = __shfl_sync(0xffffffffu, bslot, hl);
}

__device__ void pack_pool(const PackArgs& a, uint8_t* psm) {
  __shared__ int task_hw, task_pw, task_ph;   // the box whose fit test the helper warps join (hw < 0: done)
  __shared__ uint64_t cand_key[PACK_WARPS], cand_rect[PACK_WARPS];
  __shared__ int cand_slot[PACK_WARPS];
  uint32_t* dims = (uint32_t*)psm;                      // (w+g) | (h+g)<<16 of the oi-th box in order
  int32_t* ords = (int32_t*)(dims + PACK_DIMS);         // box index of the oi-th box in order
  uint64_t* skey = (uint64_t*)(ords + PACK_DIMS);       // overflow slots 32 .. 32+PACK_SOV-1 (SMEM)
  uint64_t* srect = skey + PACK_SOV;
  uint64_t* gkey = a.pool;                              // overflow slots beyond (global, L1-resident)
  uint64_t* grect = a.pool + PACK_POOL;
  // overflow slot i (= pool slot 32 + i)
  auto ov_key = [&](int i) -> uint64_t& { return i < PACK_SOV ? skey[i] : gkey[i - PACK_SOV]; };
  auto ov_rect = [&](int i) -> uint64_t& { return i < PACK_SOV ? srect[i] : grect[i - PACK_SOV]; };
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = min(*a.num_boxes, a.max_boxes);
  if (warp > 0) {
    // =========== helper warps: join the fit test of large-pool boxes ===========
    for (;;) {
      pack_bar();   // B1: a task (or the end) is published
      const int hw = task_hw, pw = task_pw, ph = task_ph;
      if (hw < 0) return;
      uint64_t best = ~0ull, brect = 0;
      int bslot = -1;
      for (int s0 = 32 + 32 * warp + lane; s0 < hw; s0 += 128 * PACK_WARPS) {
        uint64_t kk[4], rq[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int sl = s0 + 32 * PACK_WARPS * u;
          kk[u] = sl < hw ? ov_key(sl - 32) : ~0ull;
          rq[u] = sl < hw ? ov_rect(sl - 32) : 0ull;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (fits(rq[u], pw, ph) && kk[u] < best) { best = kk[u]; brect = rq[u]; bslot = s0 + 32 * PACK_WARPS * u; }
      }
      uint64_t wk, wr;
      int ws;
      warp_first_fit(best, brect, bslot, wk, wr, ws);
      if (lane == 0) { cand_key[warp] = wk; cand_rect[warp] = wr; cand_slot[warp] = ws; }
      pack_bar();   // B2: candidates posted
    }
  }
  // placement-invariant pruning bounds: a free area no box fits in (either orientation) is never stored
  int mA = 1 << 30, mB = 1 << 30;
  for (int64_t i = lane; i < n; i += 32) {
    const int bi = a.order[i];
    const regen_box& bx = a.boxes[bi];
    const int pw = bx.w + a.gutter, ph = bx.h + a.gutter;
    mA = min(mA, min(pw, ph));
    mB = min(mB, max(pw, ph));
    if (i < PACK_DIMS) {
      dims[i] = (uint32_t)pw | ((uint32_t)ph << 16);
      ords[i] = bi;
    }
  }
  mA = __reduce_min_sync(0xffffffffu, mA);
  mB = __reduce_min_sync(0xffffffffu, mB);
  __syncwarp();
  uint64_t rk = ~0ull, rr = 0ull;   // this lane's register slot: empty never fits, never wins
  const int FW = a.bin_w - 1, FH = a.bin_h + a.gutter;   // a fresh bin's free area (x=1, y=0)
  int hw = 0;        // live areas: slots [0, hw)
  int opened = 0;    // bins opened (lazily, in index order)
  uint32_t seq = 0;
  int used = 0;
  bool overflow = false;
  long long c_scan = 0, c_dec = 0, c_upd = 0, hw_sum = 0;
  int npw = 0, nph = 0, nb = 0;
  auto fetch = [&](int64_t oi) {
    if (oi >= n) return;
    if (oi < PACK_DIMS) {
      const uint32_t d = dims[oi];
      npw = (int)(d & 0xFFFF);
      nph = (int)(d >> 16);
      nb = ords[oi];
    } else {
      nb = a.order[oi];
      npw = a.boxes[nb].w + a.gutter;
      nph = a.boxes[nb].h + a.gutter;
    }
  };
  fetch(0);
  for (int64_t oi = 0; oi < n; ++oi) {
    long long t0 = 0;
    if (a.prof) t0 = clock64();
    const int pw = npw, ph = nph, b = nb;
    fetch(oi + 1);   // prefetch: off the dependent chain
    uint64_t best = fits(rr, pw, ph) ? rk : ~0ull;
    uint64_t brect = rr;
    int bslot = lane;
    const bool big = hw - 32 > PACK_BIG;   // warp-uniform
    if (big) {
      if (lane == 0) { task_hw = hw; task_pw = pw; task_ph = ph; }
      pack_bar();   // B1
    }
    // overflow slots: this warp's share (all of them on the single-warp path), 4 loads per lane in flight
    const int ostride = big ? 32 * PACK_WARPS : 32;
    for (int s0 = 32 + lane; s0 < hw; s0 += 4 * ostride) {
      uint64_t kk[4], rq[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int sl = s0 + ostride * u;
        kk[u] = sl < hw ? ov_key(sl - 32) : ~0ull;
        rq[u] = sl < hw ? ov_rect(sl - 32) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (fits(rq[u], pw, ph) && kk[u] < best) { best = kk[u]; brect = rq[u]; bslot = s0 + ostride * u; }
    }
    long long t1 = 0;
    if (a.prof) { t1 = clock64(); hw_sum += hw; }
    // 64-bit warp min as two 32-bit REDUX (bin in the high word, sequence in the low word)
    uint64_t wkey, wrect;
    int wslot;
    warp_first_fit(best, brect, bslot, wkey, wrect, wslot);
    if (big) {
      pack_bar();   // B2: the helpers' candidates are posted
      uint64_t ck = ~0ull, cr = 0;
      int cs = -1;
      if (lane == 0) { ck = wkey; cr = wrect; cs = wslot; }
      else if (lane < PACK_WARPS) { ck = cand_key[lane]; cr = cand_rect[lane]; cs = cand_slot[lane]; }
      warp_first_fit(ck, cr, cs, wkey, wrect, wslot);
    }
    __syncwarp();   // every lane's overflow-slot reads of this box's scan precede lane 0's writes below
    int fx, fy, fw, fh, bin, slot = -1;
    bool place = true;
    if (wkey != ~0ull) {
      slot = wslot;
      fx = (int)(wrect & 0xFFFF); fy = (int)((wrect >> 16) & 0xFFFF);
      fw = (int)((wrect >> 32) & 0xFFFF); fh = (int)(wrect >> 48);
      bin = (int)(wkey >> 32);
    } else if (opened < a.max_bins && ((FW >= pw && FH >= ph) || (FW >= ph && FH >= pw))) {
      bin = opened++;
      fx = 1; fy = 0; fw = FW; fh = FH;
    } else {
      place = false;
      fx = fy = fw = fh = bin = 0;
    }
    long long t2 = 0;
    if (a.prof) {
      t2 = clock64();
      c_scan += t1 - t0;
      c_dec += t2 - t1;
    }
    if (place) {
      const bool rot = !(fw >= pw && fh >= ph);
      const int uw = rot ? ph : pw, uh = rot ? pw : ph;
      used = max(used, bin + 1);
      if (lane == 0) {   // bin, bx / by, rotated: two 8-B stores
        int2* pl = reinterpret_cast<int2*>(&a.boxes[b].bin);
        pl[0] = make_int2(bin, fx);
        pl[1] = make_int2(fy, rot ? 1 : 0);
      }
      // InnerFree (D6): guillotine remainders; vertical = {right full height, bottom}, horizontal =
      // {bottom full width, right}; the option whose larger remainder is larger wins, ties vertical
      const int dw = fw - uw, dh = fh - uh;
      const int64_t v_a = (int64_t)dw * fh, v_b = (int64_t)uw * dh;
      const int64_t h_a = (int64_t)fw * dh, h_b = (int64_t)dw * uh;
      const bool vert = max(v_a, v_b) >= max(h_a, h_b);
      const int rx0 = vert ? fx + uw : fx, ry0 = vert ? fy : fy + uh;
      const int rw0 = vert ? dw : fw, rh0 = vert ? fh : dh;
      const int rx1 = vert ? fx : fx + uw, ry1 = vert ? fy + uh : fy;
      const int rw1 = vert ? uw : dw, rh1 = vert ? dh : uh;
      int free_slot = slot;   // the consumed area's slot, to be refilled
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int rx = t ? rx1 : rx0, ry = t ? ry1 : ry0, rw = t ? rw1 : rw0, rh = t ? rh1 : rh0;
        if (rw <= 0 || rh <= 0) continue;
        const uint32_t sq = seq++;   // sequence numbers follow the oracle's creation order
        if (min(rw, rh) < mA || max(rw, rh) < mB) continue;   // unusable: never stored
        int dst;
        if (free_slot >= 0) { dst = free_slot; free_slot = -1; }
        else if (hw < a.pool_limit) dst = hw++;
        else { overflow = true; continue; }
        const uint64_t nk = ((uint64_t)bin << 32) | sq;
        const uint64_t nr = (uint64_t)(uint32_t)(rx | (ry << 16)) | ((uint64_t)(uint32_t)(rw | (rh << 16)) << 32);
        if (dst < 32) {
          if (lane == dst) { rk = nk; rr = nr; }
        } else if (lane == 0) {
          ov_key(dst - 32) = nk;
          ov_rect(dst - 32) = nr;
        }
      }
      if (free_slot >= 0) {   // nothing refilled the consumed slot: move the last live area into it
        --hw;
        if (free_slot != hw) {
          uint64_t lk, lq;
          if (hw < 32) {
            lk = __shfl_sync(0xffffffffu, rk, hw);
            lq = __shfl_sync(0xffffffffu, rr, hw);
          } else {
            lk = ov_key(hw - 32);
            lq = ov_rect(hw - 32);
          }
          if (free_slot < 32) {
            if (lane == free_slot) { rk = lk; rr = lq; }
          } else if (lane == 0) {
            ov_key(free_slot - 32) = lk;
            ov_rect(free_slot - 32) = lq;
          }
        }
        if (hw < 32 && lane == hw) { rk = ~0ull; rr = 0ull; }   // the vacated register slot is empty
      }
    }
    __syncwarp();   // lane 0's overflow-slot writes are visible to every lane before the next scan
    if (a.prof) c_upd += clock64() - t2;
  }
  if (lane == 0) task_hw = -1;
  pack_bar();   // release the helper warps
  if (a.prof && lane == 0)
    printf("[pack-prof] boxes %lld scan %lld dec %lld upd %lld cycles, mean live areas %.1f, bins %d\n", (long long)n,
           c_scan, c_dec, c_upd, n ? (double)hw_sum / n : 0.0, used);
  if (lane == 0) {
    *a.num_bins = used;
    if (overflow) atomicOr(a.status, REGEN_ST_FREELIST_OVERFLOW);
  }
}


// One warp; lane l owns slot l of every bin's free-area list (it alone reads and writes that slot, so
// the lists need no cross-lane memory ordering). An area fits a box in some orientation iff its
// sorted sides dominate the footprint's (min(w,h) >= min(pw,ph) and max(w,h) >= max(pw,ph): the
// RotatePacking test). Each opened bin keeps a summary (max min-side, max max-side over
// its areas) and every 32 bins a group summary, both in SMEM; summaries are necessary conditions,
// so the first fit in (bin, seq) order (D12) is found by scanning group summaries in order, the
// passing group's bin summaries in order, and the first passing bin's slots (min seq among the
// fitting ones); a false positive just continues the scan. Placement and the guillotine remainders
// (D6) are replayed by every lane; only the used bin's list and summaries change. Bins are opened
// lazily in index order; a box that fits nowhere stays unplaced.
__device__ __forceinline__ uint32_t area_sum(uint64_t r) {   // (min side << 16) | max side, 0 if empty
  const uint32_t w = (uint32_t)((r >> 32) & 0xFFFF), h = (uint32_t)(r >> 48);
  return (min(w, h) << 16) | max(w, h);
}

__device__ __forceinline__ bool sum_ok(uint32_t sm, uint32_t qa, uint32_t qb) {
  return (sm >> 16) >= qa && (sm & 0xFFFF) >= qb;
}

__device__ __forceinline__ uint32_t warp_max2(uint32_t v) {   // per-half maxima of (a << 16 | b)
  const uint32_t a = __reduce_max_sync(0xffffffffu, v >> 16), b = __reduce_max_sync(0xffffffffu, v & 0xFFFF);
  return (a << 16) | b;
}

__device__ void pack_bins(const PackArgs& a, uint8_t* psm) {
  uint32_t* bsum = (uint32_t*)psm;                    // [PACK_MAX_BINS] per opened bin
  uint32_t* gsum = bsum + PACK_MAX_BINS;              // [PACK_MAX_BINS / 32] per 32 bins
  uint8_t* bcnt = (uint8_t*)(gsum + PACK_MAX_BINS / 32);   // [PACK_MAX_BINS] live areas per bin
  const int lane = threadIdx.x;
  const int64_t n = min(*a.num_boxes, a.max_boxes);
  // placement-invariant pruning bounds: a free area no box fits in (either orientation) is never stored
  int mA = 1 << 30, mB = 1 << 30;
  for (int64_t i = lane; i < n; i += 32) {
    const regen_box& bx = a.boxes[a.order[i]];
    const int pw = bx.w + a.gutter, ph = bx.h + a.gutter;
    mA = min(mA, min(pw, ph));
    mB = min(mB, max(pw, ph));
  }
  mA = __reduce_min_sync(0xffffffffu, mA);
  mB = __reduce_min_sync(0xffffffffu, mB);
  const int FW = a.bin_w - 1, FH = a.bin_h + a.gutter;   // a fresh bin's free area (x=1, y=0)
  int opened = 0;    // bins opened (lazily, in index order)
  uint32_t seq = 0;
  int used = 0;
  bool overflow = false;
  long long c_scan = 0, c_upd = 0, n_fp = 0;
  int npw = 0, nph = 0, nb = 0;
  auto fetch = [&](int64_t oi) {
    if (oi >= n) return;
    nb = a.order[oi];
    npw = a.boxes[nb].w + a.gutter;
    nph = a.boxes[nb].h + a.gutter;
  };
  fetch(0);
  for (int64_t oi = 0; oi < n; ++oi) {
    long long t0 = 0;
    if (a.prof) t0 = clock64();
    const int pw = npw, ph = nph, b = nb;
    fetch(oi + 1);   // prefetch: off the dependent chain
    const uint32_t qa = (uint32_t)min(pw, ph), qb = (uint32_t)max(pw, ph);
    // ---- first fit in (bin, seq) order over the opened bins
    int bin = -1, slot = -1;
    uint64_t myr = 0;        // this lane's slot of the chosen bin
    uint32_t mys = 0xFFFFFFFFu;
    const int G = (opened + 31) >> 5;
    for (int g0 = 0; g0 < G && bin < 0; g0 += 32) {
      const int g = g0 + lane;
      uint32_t gm = __ballot_sync(0xffffffffu, g < G && sum_ok(gsum[g], qa, qb));
      while (gm && bin < 0) {
        const int gg = g0 + __ffs(gm) - 1;
        gm &= gm - 1;
        const int bb = 32 * gg + lane;
        uint32_t bm = __ballot_sync(0xffffffffu, bb < opened && sum_ok(bsum[bb], qa, qb));
        while (bm) {
          const int cb = 32 * gg + __ffs(bm) - 1;
          bm &= bm - 1;
          const bool live = lane < bcnt[cb];
          const uint64_t r = live ? a.rect[(size_t)cb * PACK_SLOTS + lane] : 0ull;
          const uint32_t sq = live ? a.seqv[(size_t)cb * PACK_SLOTS + lane] : 0xFFFFFFFFu;
          const bool fit = live && sum_ok(area_sum(r), qa, qb);
          const uint32_t best = __reduce_min_sync(0xffffffffu, fit ? sq : 0xFFFFFFFFu);
          if (best != 0xFFFFFFFFu) {
            bin = cb;
            slot = __ffs(__ballot_sync(0xffffffffu, fit && sq == best)) - 1;
            myr = r;
            mys = sq;
            break;
          }
          if (a.prof) ++n_fp;
        }
      }
    }
    int fx, fy, fw, fh;
    bool place = true;
    if (bin >= 0) {
      const uint64_t wr = __shfl_sync(0xffffffffu, myr, slot);
      fx = (int)(wr & 0xFFFF); fy = (int)((wr >> 16) & 0xFFFF);
      fw = (int)((wr >> 32) & 0xFFFF); fh = (int)(wr >> 48);
    } else if (opened < a.max_bins && ((FW >= pw && FH >= ph) || (FW >= ph && FH >= pw))) {
      bin = opened++;
      fx = 1; fy = 0; fw = FW; fh = FH;
      myr = 0ull;
      mys = 0xFFFFFFFFu;
    } else {
      place = false;
      fx = fy = fw = fh = 0;
    }
    long long t1 = 0;
    if (a.prof) { t1 = clock64(); c_scan += t1 - t0; }
    if (place) {
      const bool rot = !(fw >= pw && fh >= ph);
      const int uw = rot ? ph : pw, uh = rot ? pw : ph;
      used = max(used, bin + 1);
      if (lane == 0) {   // bin, bx / by, rotated: two 8-B stores
        int2* pl = reinterpret_cast<int2*>(&a.boxes[b].bin);
        pl[0] = make_int2(bin, fx);
        pl[1] = make_int2(fy, rot ? 1 : 0);
      }
      // this bin's list: remove the used slot (the last slot moves into it), then append the kept
      // guillotine remainders (D6): vertical = {right full height, bottom}, horizontal = {bottom full
      // width, right}; the option whose larger remainder is larger wins, ties vertical
      int cnt = slot >= 0 ? (int)bcnt[bin] : 0;   // a freshly opened bin has no listed areas yet
      if (slot >= 0) {
        const uint64_t lr = __shfl_sync(0xffffffffu, myr, cnt - 1);
        const uint32_t ls = __shfl_sync(0xffffffffu, mys, cnt - 1);
        if (lane == slot) { myr = lr; mys = ls; }
        --cnt;
        if (lane == cnt) { myr = 0ull; mys = 0xFFFFFFFFu; }
      }
      const int dw = fw - uw, dh = fh - uh;
      const int64_t v_a = (int64_t)dw * fh, v_b = (int64_t)uw * dh;
      const int64_t h_a = (int64_t)fw * dh, h_b = (int64_t)dw * uh;
      const bool vert = max(v_a, v_b) >= max(h_a, h_b);
      const int rx0 = vert ? fx + uw : fx, ry0 = vert ? fy : fy + uh;
      const int rw0 = vert ? dw : fw, rh0 = vert ? fh : dh;
      const int rx1 = vert ? fx : fx + uw, ry1 = vert ? fy + uh : fy;
      const int rw1 = vert ? uw : dw, rh1 = vert ? dh : uh;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int rx = t ? rx1 : rx0, ry = t ? ry1 : ry0, rw = t ? rw1 : rw0, rh = t ? rh1 : rh0;
        if (rw <= 0 || rh <= 0) continue;
        const uint32_t sq = seq++;   // sequence numbers follow the oracle's creation order
        if (min(rw, rh) < mA || max(rw, rh) < mB) continue;   // unusable: never stored
        if (cnt >= a.slot_limit) { overflow = true; continue; }
        if (lane == cnt) {
          myr = (uint64_t)(uint32_t)(rx | (ry << 16)) | ((uint64_t)(uint32_t)(rw | (rh << 16)) << 32);
          mys = sq;
        }
        ++cnt;
      }
      // write back this lane's slot of the bin and refresh the bin's and its group's summaries
      if (lane < cnt) {
        a.rect[(size_t)bin * PACK_SLOTS + lane] = myr;
        a.seqv[(size_t)bin * PACK_SLOTS + lane] = mys;
      }
      const uint32_t bs = warp_max2(lane < cnt ? area_sum(myr) : 0u);
      __syncwarp();   // every lane's read of bcnt[bin] above precedes lane 0's write
      if (lane == 0) { bsum[bin] = bs; bcnt[bin] = (uint8_t)cnt; }
      __syncwarp();
      const int gb = (bin >> 5) << 5;
      const uint32_t gs = warp_max2(gb + lane < opened ? bsum[gb + lane] : 0u);
      if (lane == 0) gsum[bin >> 5] = gs;
      __syncwarp();
    }
    if (a.prof) c_upd += clock64() - t1;
  }
  if (a.prof && lane == 0)
    printf("[pack-prof] boxes %lld scan %lld upd %lld cycles, false-positive bins %lld, bins %d\n", (long long)n,
           c_scan, c_upd, n_fp, used);
  if (lane == 0) {
    *a.num_bins = used;
    if (overflow) atomicOr(a.status, REGEN_ST_FREELIST_OVERFLOW);
  }
}

__global__ void __launch_bounds__(32 * PACK_WARPS, 1) pack_kernel(PackArgs a) {
  extern __shared__ __align__(16) uint8_t psm[];
  if (min(*a.num_boxes, a.max_boxes) > PACK_BINS_FROM) {
    if (threadIdx.x < 32) pack_bins(a, psm);
  } else {
    pack_pool(a, psm);
  }
}

__global__ void owner_fix_kernel(int32_t* owner, int64_t n_mbs, const regen_box* boxes, const int64_t* num_boxes,
                                 int64_t max_boxes) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_mbs) return;
  const int32_t o = owner[i];
  if (o < 0) return;
  const int64_t nb = min(*num_boxes, max_boxes);
  if (o >= nb || boxes[o].bin < 0) owner[i] = -1;
}

static size_t pack_ws(const regen_geom& g, int64_t max_regions, void* base, int32_t** rcount, int64_t** roff,
                      int64_t** nreg, uint64_t** rect = nullptr, uint32_t** seqv = nullptr) {
  Carver c(base);
  int32_t* rc = c.take<int32_t>((size_t)max_regions + 1);
  int64_t* ro = c.take<int64_t>((size_t)max_regions + 1);
  int64_t* nr = c.take<int64_t>(4);
  uint64_t* rt = c.take<uint64_t>((size_t)PACK_MAX_BINS * PACK_SLOTS + 2 * (size_t)PACK_POOL);
  uint32_t* sq = c.take<uint32_t>((size_t)PACK_MAX_BINS * PACK_SLOTS);
  if (rcount) *rcount = rc;
  if (roff) *roff = ro;
  if (nreg) *nreg = nr;
  if (rect) *rect = rt;
  if (seqv) *seqv = sq;
  (void)g;
  return c.off + 256;
}

// the guillotine packer's state, plus a placement policy's per-bin state when params name one
size_t pack_workspace_bytes(const regen_geom& g, int64_t max_regions, const regen_pack_params* p) {
  const size_t base = (pack_ws(g, max_regions, nullptr, nullptr, nullptr, nullptr) + 255) / 256 * 256;
  return p && p->policy != REGEN_POLICY_GUILLOTINE ? base + policy_workspace_bytes(*p) : base;
}

}  // namespace regen

using namespace regen;

extern "C" regen_status regen_pack_regions(const regen_geom* geom, const regen_pack_params* p,
                                           const float* d_importance, const int32_t* d_labels,
                                           const regen_region* d_regions, const int64_t* d_num_regions,
                                           regen_box* d_boxes, int64_t max_boxes, int64_t* d_num_boxes,
                                           int32_t* d_order, int32_t* d_num_bins, int32_t* d_mb_owner,
                                           int32_t* d_status, void* d_ws, size_t ws_bytes, void* stream) {
  REGEN_NVTX("regen_pack_regions");
  regen_status st = validate_geom(geom);
  if (st != REGEN_OK) return st;
  REGEN_REQUIRE(p != nullptr, "params is null");
  REGEN_REQUIRE(p->bin_w >= 4 && p->bin_h >= 1 && p->bin_w <= 4096 && p->bin_h <= 4096, "bad bin size");
  REGEN_REQUIRE(p->max_bins >= 0 && p->max_bins <= PACK_MAX_BINS, "max_bins must be in [0, %d]", PACK_MAX_BINS);
  REGEN_REQUIRE(p->expand >= 0 && p->expand <= 64, "bad expand");
  REGEN_REQUIRE(p->partition_mb >= 1 && p->partition_mb <= 64, "bad partition_mb");
  REGEN_REQUIRE(p->gutter >= 0 && p->gutter <= 8, "bad gutter");
  REGEN_REQUIRE(p->order == REGEN_ORDER_DENSITY || p->order == REGEN_ORDER_AREA || p->order == REGEN_ORDER_HEIGHT,
                "bad order");
  REGEN_REQUIRE(p->density == REGEN_DENSITY_SPAN || p->density == REGEN_DENSITY_MEMBERS, "bad density mode");
  REGEN_REQUIRE(p->policy >= REGEN_POLICY_GUILLOTINE && p->policy <= REGEN_POLICY_SHELF, "bad policy %d", p->policy);
  REGEN_REQUIRE(d_importance && d_labels && d_num_regions && d_num_boxes && d_num_bins && d_mb_owner && d_status,
                "null device pointer");
  REGEN_REQUIRE(max_boxes >= 1 && max_boxes < (1ll << 31) && d_boxes && d_order, "bad boxes buffer");
  const regen_geom g = *geom;
  // the region capacity is implied by the labels: at most one region per MB
  const int64_t max_regions = n_mbs(g);
  REGEN_REQUIRE(ws_bytes >= pack_workspace_bytes(g, max_regions, p) && d_ws, "workspace too small (%zu < %zu)",
                ws_bytes, pack_workspace_bytes(g, max_regions, p));
  cudaStream_t s = (cudaStream_t)stream;
  int32_t* rcount;
  int64_t *roff, *nreg;
  uint64_t* rect;
  uint32_t* seqv;
  pack_ws(g, max_regions, d_ws, &rcount, &roff, &nreg, &rect, &seqv);
  REGEN_CUDA(cudaMemsetAsync(d_mb_owner, 0xFF, sizeof(int32_t) * (size_t)n_mbs(g), s));

  BoxArgs a;
  a.imp = d_importance;
  a.labels = d_labels;
  a.regions = d_regions;
  a.num_regions = d_num_regions;
  a.max_regions = max_regions;
  a.region_count = rcount;
  a.region_off = roff;
  a.boxes = d_boxes;
  a.max_boxes = max_boxes;
  a.box_of_mb = d_mb_owner;
  a.status = d_status;
  a.GW = grid_w(g);
  a.GH = grid_h(g);
  a.W = g.frame_w;
  a.H = g.frame_h;
  a.F = g.F;
  a.mb = g.mb;
  a.expand = p->expand;
  a.P = p->partition_mb;
  a.density = p->density;
  const int warps_per_block = 4;   // 128 threads x <= 56 registers: fits beside a resident SR conv CTA
  const unsigned nblk = (unsigned)std::min<int64_t>((max_regions + warps_per_block - 1) / warps_per_block, 148 * 4);
  {
    REGEN_TRACE("clamp_count", s);
    clamp_count_kernel<<<1, 1, 0, s>>>(d_num_regions, max_regions, rcount, nreg);
  }
  REGEN_LAUNCH_CHECK();
  {
    REGEN_TRACE("box_count", s);
    box_count_kernel<<<nblk, 32 * warps_per_block, 0, s>>>(a);
  }
  REGEN_LAUNCH_CHECK();
  {
    REGEN_TRACE("scan_boxes", s);
    scan_counts64_kernel<<<1, 256, 0, s>>>(rcount, nreg, roff, d_num_boxes);
  }
  REGEN_LAUNCH_CHECK();
  {
    REGEN_TRACE("box_write", s);
    box_write_kernel<<<nblk, 32 * warps_per_block, 0, s>>>(a);
  }
  REGEN_LAUNCH_CHECK();
  {
    REGEN_TRACE("sort_rank", s);
    const size_t ssm = (size_t)SORT_SMEM * 12;
    REGEN_CUDA(cudaFuncSetAttribute(sort_bitonic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm));
    sort_bitonic_kernel<<<1, 1024, ssm, s>>>(d_boxes, d_num_boxes, max_boxes, p->order, d_order);
    if (max_boxes > SORT_SMEM)
      sort_rank_kernel<<<(unsigned)((max_boxes + 255) / 256), 256, 0, s>>>(d_boxes, d_num_boxes, max_boxes, p->order,
                                                                           d_order);
  }
  REGEN_LAUNCH_CHECK();
  PackArgs k;
  k.boxes = d_boxes;
  k.rect = rect;
  k.seqv = seqv;
  k.pool = rect + (size_t)PACK_MAX_BINS * PACK_SLOTS;
  k.order = d_order;
  k.num_boxes = d_num_boxes;
  k.max_boxes = max_boxes;
  k.num_bins = d_num_bins;
  k.status = d_status;
  k.bin_w = p->bin_w;
  k.bin_h = p->bin_h;
  k.max_bins = p->max_bins;
  k.gutter = p->gutter;
  {
    const char* e = getenv("REGEN_PACK_PROF");
    k.prof = (e && e[0] == '1') ? 1 : 0;
    const char* lim = getenv("REGEN_PACK_POOL_LIMIT");
    k.slot_limit = PACK_SLOTS;
    k.pool_limit = PACK_POOL + 32;
    if (lim && atoi(lim) > 0) {
      k.slot_limit = std::min(atoi(lim), PACK_SLOTS);
      k.pool_limit = std::min(atoi(lim), PACK_POOL + 32);
    }
  }
  if (p->policy != REGEN_POLICY_GUILLOTINE) {   // SURVEY §8(f)1 comparison policies (pack_policies.cu)
    void* pws = (uint8_t*)d_ws + (pack_ws(g, max_regions, nullptr, nullptr, nullptr, nullptr) + 255) / 256 * 256;
    regen_status ps = launch_pack_policy(*p, d_boxes, d_order, d_num_boxes, max_boxes, d_num_bins, d_status, pws, s);
    if (ps != REGEN_OK) return ps;
  } else {
    REGEN_CUDA(cudaFuncSetAttribute(pack_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, PACK_SMEM));
    REGEN_TRACE("pack", s);
    pack_kernel<<<1, 32 * PACK_WARPS, PACK_SMEM, s>>>(k);
  }
  REGEN_LAUNCH_CHECK();
  if (k.prof) {
    cudaStreamSynchronize(s);
    fflush(stdout);
  }
  {
    REGEN_TRACE("owner_fix", s);
    owner_fix_kernel<<<(unsigned)((n_mbs(g) + 255) / 256), 256, 0, s>>>(d_mb_owner, n_mbs(g), d_boxes, d_num_boxes,
                                                                         max_boxes);
  }
  REGEN_LAUNCH_CHECK();
  return REGEN_OK;
}
