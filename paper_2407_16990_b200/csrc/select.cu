// a1 + a2: cross-stream MB selection (§3.3.1) and region growth (Alg. 1 line 3).
//
// select_kernel   one CTA per scope segment. Exact top-k by a 3-pass radix select on the 32-bit
//                 importance order (11/11/10-bit digits, SMEM histograms), then an id-ordered
//                 block scan ranks the ties of the k-th value so the lowest ids win (D2).
//                 Selected MBs are OR-ed into the per-row u32 bitmap.
// ccl_kernel      one CTA per frame: concurrent union-find on the MB grid in SMEM (links always
//                 point to the smaller raster index, so every root is its component's minimum),
//                 regions ranked by root in raster order, SMEM atomics for bbox/count.
// region_write    globalises frame-local region ids with the scanned per-frame offsets.
#include <algorithm>

#include "common.cuh"

namespace regen {

// ------------------------------------------------------------------------------------ select

struct SelArgs {
  const float* imp;
  uint32_t* bitmap;
  int64_t seg_len;
  int per_frame, GW, W32, GH;
  int mode;
  int64_t k;
  float tau;
};

__device__ __forceinline__ bool sel_eligible(const SelArgs& a, float s) {
  return a.mode == REGEN_MODE_TOPK || s >= a.tau;
}

__device__ __forceinline__ void set_bit(const SelArgs& a, int64_t id) {
  const int64_t frame = id / a.per_frame;
  const int cell = (int)(id - frame * a.per_frame);
  const int y = cell / a.GW, x = cell - y * a.GW;
  atomicOr(a.bitmap + (frame * a.GH + y) * a.W32 + (x >> 5), 1u << (x & 31));
}

// Find digit d (scanning from the highest) with above(d) < kk <= above(d) + hist[d].
// hist has nb bins in SMEM; returns d and sets *above. All threads get the result.
__device__ int find_digit(const int* hist, int nb, int64_t kk, int64_t* above, int* scratch, int64_t* sh64) {
  // suffix sums: process bins from high to low in chunks of blockDim
  __shared__ int s_found;
  __shared__ int64_t s_above;
  if (threadIdx.x == 0) { s_found = -1; s_above = 0; }
  __syncthreads();
  int64_t carry = 0;
  for (int base = 0; base < nb; base += blockDim.x) {
    const int t = base + threadIdx.x;           // t-th bin from the top
    const int d = nb - 1 - t;
    const int h = t < nb ? hist[d] : 0;
    int tot;
    const int ex = block_exclusive_scan(h, scratch, &tot);
    const int64_t ab = carry + ex;              // count strictly above digit d
    if (t < nb && h > 0 && ab < kk && kk <= ab + h) { s_found = d; s_above = ab; }
    carry += tot;
    __syncthreads();
    if (s_found >= 0) break;
  }
  (void)sh64;
  *above = s_above;
  return s_found;
}

__global__ void __launch_bounds__(1024) select_kernel(SelArgs a) {
  __shared__ int hist[2048];
  __shared__ int scratch[33];
  __shared__ int64_t sh64;
  const int64_t seg0 = (int64_t)blockIdx.x * a.seg_len;
  const float* sc = a.imp + seg0;
  const int64_t n = a.seg_len;

  // count eligible (and handle the trivial cases)
  int64_t cnt_local = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) cnt_local += sel_eligible(a, sc[i]) ? 1 : 0;
  __shared__ unsigned long long s_cnt;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  cnt_local = warp_sum(cnt_local);
  if ((threadIdx.x & 31) == 0) atomicAdd(&s_cnt, (unsigned long long)cnt_local);
  __syncthreads();
  const int64_t n_elig = (int64_t)s_cnt;
  const bool take_all = (a.mode == REGEN_MODE_THRESHOLD && a.k < 0) || a.k >= n_elig;
  if (a.k == 0 && !(a.mode == REGEN_MODE_THRESHOLD && a.k < 0)) return;
  if (take_all) {
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
      if (sel_eligible(a, sc[i])) set_bit(a, seg0 + i);
    return;
  }
  // 3-pass radix select of the kk-th largest order value among eligible elements
  int64_t kk = a.k;
  uint32_t prefix = 0;
  int64_t above_total = 0;
  const int shifts[3] = {21, 10, 0};
  const int bits[3] = {11, 11, 10};
  for (int pass = 0; pass < 3; ++pass) {
    const int nb = 1 << bits[pass];
    for (int i = threadIdx.x; i < nb; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const int hs = shifts[pass] + bits[pass];   // bits above this digit must equal prefix
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const float s = sc[i];
      if (!sel_eligible(a, s)) continue;
      const uint32_t o = score_ord(s);
      if (hs < 32 && (o >> hs) != prefix) continue;
      atomicAdd(&hist[(o >> shifts[pass]) & (nb - 1)], 1);
    }
    __syncthreads();
    int64_t above;
    const int d = find_digit(hist, nb, kk, &above, scratch, &sh64);
    prefix = (prefix << bits[pass]) | (uint32_t)d;
    kk -= above;
    above_total += above;
    __syncthreads();
  }
  const uint32_t v = prefix;   // the k-th largest order value
  const int64_t r = kk;        // how many elements equal to v are selected (lowest ids first)
  // final pass in id order: ord > v, or ord == v with tie rank < r
  int64_t running = 0;
  for (int64_t base = 0; base < n; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    bool gt = false, eq = false;
    if (i < n) {
      const float s = sc[i];
      if (sel_eligible(a, s)) {
        const uint32_t o = score_ord(s);
        gt = o > v;
        eq = o == v;
      }
    }
    int tot;
    const int ex = block_exclusive_scan(eq ? 1 : 0, scratch, &tot);
    if (gt || (eq && running + ex < r)) set_bit(a, seg0 + i);
    running += tot;
    if (running >= r && base + blockDim.x < n) {
      // remaining elements can only be selected through gt; continue without tie accounting
      for (int64_t j = base + blockDim.x + threadIdx.x; j < n; j += blockDim.x) {
        const float s = sc[j];
        if (sel_eligible(a, s) && score_ord(s) > v) set_bit(a, seg0 + j);
      }
      break;
    }
  }
  (void)above_total;
}

// ------------------------------------------------------------------------------------ CCL

struct CclArgs {
  const uint32_t* bitmap;
  int32_t* labels;          // [frames][GH][GW] out: frame-local region index or -1
  int32_t* stage;           // [frames][per_frame][6]: root, mx0, my0, mx1, my1, count
  int32_t* frame_count;     // [frames]
  int GW, GH, W32, per_frame, conn;
};

__device__ __forceinline__ int uf_find(volatile int* parent, int x) {
  int p = parent[x];
  while (p != x) { x = p; p = parent[x]; }
  return x;
}

__device__ __forceinline__ void uf_unite(int* parent, int a, int b) {
  volatile int* vp = parent;
  while (true) {
    a = uf_find(vp, a);
    b = uf_find(vp, b);
    if (a == b) return;
    if (a > b) { int t = a; a = b; b = t; }   // a < b: link b -> a
    const int old = atomicCAS(&parent[b], b, a);
    if (old == b) return;
    b = old;
  }
}

__global__ void __launch_bounds__(512) ccl_kernel(CclArgs a) {
  extern __shared__ int sm[];
  const int pf = a.per_frame;
  int* parent = sm;              // pf
  int* rank = sm + pf;           // pf (root -> local region index)
  int* rmx0 = sm + 2 * pf;       // per region stats, pf each
  int* rmy0 = sm + 3 * pf;
  int* rmx1 = sm + 4 * pf;
  int* rmy1 = sm + 5 * pf;
  int* rcnt = sm + 6 * pf;
  __shared__ int scratch[33];
  const int64_t frame = blockIdx.x;
  const uint32_t* bm = a.bitmap + frame * a.GH * a.W32;
  for (int i = threadIdx.x; i < pf; i += blockDim.x) {
    const int y = i / a.GW, x = i - y * a.GW;
    const bool s = (bm[y * a.W32 + (x >> 5)] >> (x & 31)) & 1u;
    parent[i] = s ? i : -1;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < pf; i += blockDim.x) {
    if (parent[i] < 0) continue;
    const int y = i / a.GW, x = i - y * a.GW;
    // backward neighbours: left, up; and for 8-conn up-left, up-right
    if (x > 0 && parent[i - 1] >= 0) uf_unite(parent, i, i - 1);
    if (y > 0) {
      const int u = i - a.GW;
      if (parent[u] >= 0) uf_unite(parent, i, u);
      if (a.conn == 8) {
        if (x > 0 && parent[u - 1] >= 0) uf_unite(parent, i, u - 1);
        if (x + 1 < a.GW && parent[u + 1] >= 0) uf_unite(parent, i, u + 1);
      }
    }
  }
  __syncthreads();
  // roots, ranked in raster order
  int carry = 0;
  for (int base = 0; base < pf; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const bool root = i < pf && parent[i] == i;
    int tot;
    const int ex = block_exclusive_scan(root ? 1 : 0, scratch, &tot);
    if (root) rank[i] = carry + ex;
    carry += tot;
  }
  const int nreg = carry;
  for (int r = threadIdx.x; r < nreg; r += blockDim.x) {
    rmx0[r] = a.GW; rmy0[r] = a.GH; rmx1[r] = 0; rmy1[r] = 0; rcnt[r] = 0;
  }
  __syncthreads();
  int32_t* lab = a.labels + frame * pf;
  for (int i = threadIdx.x; i < pf; i += blockDim.x) {
    if (parent[i] < 0) { lab[i] = -1; continue; }
    const int root = uf_find(parent, i);
    const int r = rank[root];
    lab[i] = r;
    const int y = i / a.GW, x = i - y * a.GW;
    atomicMin(&rmx0[r], x);
    atomicMin(&rmy0[r], y);
    atomicMax(&rmx1[r], x + 1);
    atomicMax(&rmy1[r], y + 1);
    atomicAdd(&rcnt[r], 1);
  }
  __syncthreads();
  int32_t* st = a.stage + frame * pf * 6;
  for (int i = threadIdx.x; i < pf; i += blockDim.x) {
    if (parent[i] == i) {
      const int r = rank[i];
      st[r * 6 + 0] = i;
      st[r * 6 + 1] = rmx0[r];
      st[r * 6 + 2] = rmy0[r];
      st[r * 6 + 3] = rmx1[r];
      st[r * 6 + 4] = rmy1[r];
      st[r * 6 + 5] = rcnt[r];
    }
  }
  if (threadIdx.x == 0) a.frame_count[frame] = nreg;
}

// Exclusive scan of n int32 counts (single CTA) -> int64 offsets, total into *total.
__global__ void __launch_bounds__(1024) scan_counts_kernel(const int32_t* counts, int64_t n, int64_t* offsets,
                                                           int64_t* total) {
  __shared__ int scratch[33];
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

struct RegWriteArgs {
  int32_t* labels;
  const int32_t* stage;
  const int32_t* frame_count;
  const int64_t* frame_off;
  regen_region* regions;
  int64_t max_regions;
  int32_t* status;
  int per_frame, F;
};

__global__ void region_write_kernel(RegWriteArgs a) {
  const int64_t frame = blockIdx.x;
  const int64_t off = a.frame_off[frame];
  const int n = a.frame_count[frame];
  int32_t* lab = a.labels + frame * a.per_frame;
  for (int i = threadIdx.x; i < a.per_frame; i += blockDim.x) {
    const int l = lab[i];
    if (l >= 0) lab[i] = (int32_t)(off + l);
  }
  const int32_t* st = a.stage + frame * a.per_frame * 6;
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    const int64_t g = off + r;
    if (g >= a.max_regions) { atomicOr(a.status, REGEN_ST_REGION_OVERFLOW); continue; }
    regen_region rec;
    rec.stream = (int32_t)(frame / a.F);
    rec.frame = (int32_t)(frame % a.F);
    rec.root = st[r * 6 + 0];
    rec.mx0 = st[r * 6 + 1];
    rec.my0 = st[r * 6 + 2];
    rec.mx1 = st[r * 6 + 3];
    rec.my1 = st[r * 6 + 4];
    rec.n_members = st[r * 6 + 5];
    a.regions[g] = rec;
  }
}

// ------------------------------------------------------------------------------------ host

static size_t select_ws(const regen_geom& g, void* base, int32_t** stage, int32_t** fcount, int64_t** foff) {
  Carver c(base);
  const int64_t nf = n_frames(g);
  const int pf = grid_w(g) * grid_h(g);
  int32_t* s = c.take<int32_t>((size_t)nf * pf * 6);
  int32_t* fc = c.take<int32_t>((size_t)nf);
  int64_t* fo = c.take<int64_t>((size_t)nf);
  if (stage) *stage = s;
  if (fcount) *fcount = fc;
  if (foff) *foff = fo;
  return c.off + 256;
}

size_t select_workspace_bytes(const regen_geom& g) { return select_ws(g, nullptr, nullptr, nullptr, nullptr); }

// a2: regions of the selected-MB bitmap (CCL per frame, region table in (s, f, min raster) order);
// shared by regen_select_mbs and regen_select_mbs_global
regen_status launch_regions(const regen_geom& g, int connectivity, const uint32_t* d_sel_bitmap, int32_t* d_labels,
                            regen_region* d_regions, int64_t max_regions, int64_t* d_num_regions, int32_t* d_status,
                            void* d_ws, cudaStream_t s) {
  const int GW = grid_w(g), GH = grid_h(g), W32 = words_per_row(g);
  const int pf = GW * GH;
  const int64_t nf = n_frames(g);
  int32_t *stage, *fcount;
  int64_t* foff;
  select_ws(g, d_ws, &stage, &fcount, &foff);
  CclArgs c;
  c.bitmap = d_sel_bitmap;
  c.labels = d_labels;
  c.stage = stage;
  c.frame_count = fcount;
  c.GW = GW;
  c.GH = GH;
  c.W32 = W32;
  c.per_frame = pf;
  c.conn = connectivity;
  const size_t smem = sizeof(int) * 7 * (size_t)pf;
  REGEN_REQUIRE(smem <= 227 * 1024, "frame MB grid too large for the CCL kernel (%d MBs)", pf);
  REGEN_CUDA(cudaFuncSetAttribute(ccl_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  {
    REGEN_TRACE("ccl", s);
    ccl_kernel<<<(unsigned)nf, 512, smem, s>>>(c);
  }
  REGEN_LAUNCH_CHECK();
  {
    REGEN_TRACE("scan_regions", s);
    scan_counts_kernel<<<1, 1024, 0, s>>>(fcount, nf, foff, d_num_regions);
  }
  REGEN_LAUNCH_CHECK();
  RegWriteArgs w;
  w.labels = d_labels;
  w.stage = stage;
  w.frame_count = fcount;
  w.frame_off = foff;
  w.regions = d_regions;
  w.max_regions = max_regions;
  w.status = d_status;
  w.per_frame = pf;
  w.F = g.F;
  {
    REGEN_TRACE("region_write", s);
    region_write_kernel<<<(unsigned)nf, 256, 0, s>>>(w);
  }
  REGEN_LAUNCH_CHECK();
  return REGEN_OK;
}

}  // namespace regen

using namespace regen;

extern "C" regen_status regen_select_mbs(const regen_geom* geom, const regen_select_params* p,
                                         const float* d_importance, uint32_t* d_sel_bitmap, int32_t* d_labels,
                                         regen_region* d_regions, int64_t max_regions, int64_t* d_num_regions,
                                         int32_t* d_status, void* d_ws, size_t ws_bytes, void* stream) {
  REGEN_NVTX("regen_select_mbs");
  regen_status st = validate_geom(geom);
  if (st != REGEN_OK) return st;
  REGEN_REQUIRE(p != nullptr, "params is null");
  REGEN_REQUIRE(p->mode == REGEN_MODE_TOPK || p->mode == REGEN_MODE_THRESHOLD, "bad mode %d", p->mode);
  REGEN_REQUIRE(p->scope >= 0 && p->scope <= 2, "bad scope %d", p->scope);
  REGEN_REQUIRE(p->connectivity == 8 || p->connectivity == 4, "connectivity must be 4 or 8");
  REGEN_REQUIRE(p->mode == REGEN_MODE_THRESHOLD || p->k >= 0, "k must be >= 0 for TOPK");
  REGEN_REQUIRE(!(p->tau != p->tau), "tau is NaN");
  REGEN_REQUIRE(p->cap >= -1, "cap must be -1 (none) or >= 0");
  REGEN_REQUIRE(d_importance && d_sel_bitmap && d_labels && d_num_regions && d_status, "null device pointer");
  REGEN_REQUIRE(max_regions >= 0 && (max_regions == 0 || d_regions), "bad regions buffer");
  const regen_geom g = *geom;
  REGEN_REQUIRE(ws_bytes >= select_workspace_bytes(g) && d_ws, "workspace too small (%zu < %zu)", ws_bytes,
                select_workspace_bytes(g));
  cudaStream_t s = (cudaStream_t)stream;
  const int GW = grid_w(g), GH = grid_h(g), W32 = words_per_row(g);
  const int pf = GW * GH;
  const int64_t nf = n_frames(g);
  const int64_t M = nf * pf;
  REGEN_REQUIRE(M < (1ll << 31), "too many MBs in one call");
  REGEN_CUDA(cudaMemsetAsync(d_status, 0, sizeof(int32_t), s));   // a batch starts with a clean status word
  REGEN_CUDA(cudaMemsetAsync(d_sel_bitmap, 0, sizeof(uint32_t) * (size_t)nf * GH * W32, s));
  SelArgs a;
  a.imp = d_importance;
  a.bitmap = d_sel_bitmap;
  a.seg_len = p->scope == REGEN_SCOPE_GLOBAL ? M : (p->scope == REGEN_SCOPE_PER_STREAM ? (int64_t)g.F * pf : pf);
  a.per_frame = pf;
  a.GW = GW;
  a.W32 = W32;
  a.GH = GH;
  a.mode = p->mode;
  // the capacity cap N applies on top of k in both modes
  a.k = p->cap < 0 ? p->k : ((p->mode == REGEN_MODE_THRESHOLD && p->k < 0) ? p->cap : std::min(p->k, p->cap));
  a.tau = p->tau;
  const int nseg = (int)(M / a.seg_len);
  {
    REGEN_TRACE("select", s);
    select_kernel<<<nseg, 1024, 0, s>>>(a);
  }
  REGEN_LAUNCH_CHECK();

  return launch_regions(g, p->connectivity, d_sel_bitmap, d_labels, d_regions, max_regions, d_num_regions, d_status,
                        d_ws, s);
}
